// Shared device/host helpers for the kvx sm_100a kernels.
#pragma once

#include <cuda.h>
#include <cuda_runtime.h>
#include <stdint.h>

#include <atomic>
#include <mutex>

#include <string>
#include <vector>

#include "kvx.h"

struct kvx_pool {
  uint8_t* base = nullptr;
  uint64_t num_pages = 0;
  uint64_t page_bytes = 0;
  int device = -1;       // -1: host pool
  bool owned = false;    // cudaFree / cudaFreeHost on destroy
  bool ipc = false;      // opened from a peer's IPC handle
  bool host = false;
  int fd = -1;           // file pool (DISK tier): pages at offset page * page_bytes
  bool direct = false;   // fd opened with O_DIRECT
  std::atomic<int> io_errno{0};  // first failed read/write (sticky)
  // K4's TMA view of a DEVICE pool (kvx_attn.cu): built on first use for a
  // kv-head count, then reused by every launch over this pool.
  std::mutex tmap_mu;
  int tmap_heads = -1;  // -1: not built; -2: cannot be built for this pool
  alignas(64) CUtensorMap tmap;
};

namespace kvx {

void set_error(const std::string& msg);
int fail_cuda(cudaError_t e, const char* what);
int fail_arg(const char* what);
int sm_count(int device);
// Counts launches of this library's own kernels (kvx_launch_count): the
// bench reports how many ran inside its timed region from this counter.
void note_launch(uint64_t n = 1);
void note_library_launch(uint64_t n = 1);  // cuBLAS calls (kvx_model projections)
// File pools (DISK tier): sticky I/O error check, and stream-ordered page I/O
// between a file pool and host memory (kvx_pool.cu).
int check_io(const kvx_pool* pool, const char* who);
struct FileRun {
  uint8_t* host;     // host bytes (pinned pool page run)
  uint64_t offset;   // byte offset in the file
  uint64_t bytes;
};
int enqueue_file_io(kvx_pool* file, std::vector<FileRun> runs, bool write, cudaStream_t stream, const char* who);

// Makes `device` current for the scope (kernels must launch on the device
// that owns the stream and the pool); no-op for host pools (device < 0).
struct DeviceGuard {
  int prev = -1;
  explicit DeviceGuard(int device) {
    if (device < 0) return;
    int cur = 0;
    if (cudaGetDevice(&cur) == cudaSuccess && cur != device && cudaSetDevice(device) == cudaSuccess) prev = cur;
  }
  ~DeviceGuard() {
    if (prev >= 0) cudaSetDevice(prev);
  }
  DeviceGuard(const DeviceGuard&) = delete;
  DeviceGuard& operator=(const DeviceGuard&) = delete;
};

#define KVX_CUDA_TRY(expr, what)                  \
  do {                                            \
    cudaError_t kvx_e_ = (expr);                  \
    if (kvx_e_ != cudaSuccess) return kvx::fail_cuda(kvx_e_, what); \
  } while (0)

inline cudaStream_t as_stream(void* s) { return reinterpret_cast<cudaStream_t>(s); }

// splitmix64 (Steele, Lea, Flood 2014): the page-content generator shared
// bit-for-bit with the CPU oracle (oracle/kvx_oracle.c).
__host__ __device__ __forceinline__ uint64_t splitmix64(uint64_t x) {
  x += 0x9E3779B97F4A7C15ull;
  uint64_t z = x;
  z = (z ^ (z >> 30)) * 0xBF58476D1CE4E5B9ull;
  z = (z ^ (z >> 27)) * 0x94D049BB133111EBull;
  return z ^ (z >> 31);
}

__host__ __device__ __forceinline__ uint64_t block_base(uint64_t seed, uint32_t session, uint32_t layer,
                                                        uint32_t block) {
  uint64_t h = splitmix64(seed);
  h = splitmix64(h ^ session);
  h = splitmix64(h ^ layer);
  return splitmix64(h ^ block);
}

// Uniform on [-sqrt(3), sqrt(3)) (unit variance), exact and identical on
// CPU/GPU: 24 random bits -> exact [-1,1) -> one IEEE fp32 multiply.
__device__ __forceinline__ float unit_value(uint64_t r) {
  const int32_t u = static_cast<int32_t>(r >> 40) - 8388608;
  return __fmul_rn(static_cast<float>(u) * (1.0f / 8388608.0f), 1.7320508f);
}

// fp32 -> bf16 round-to-nearest-even on the bit pattern (finite inputs).
__host__ __device__ __forceinline__ uint16_t f32_to_bf16_rne(float f) {
  uint32_t bits;
  memcpy(&bits, &f, 4);
  const uint32_t rounding = 0x7FFFu + ((bits >> 16) & 1u);
  return static_cast<uint16_t>((bits + rounding) >> 16);
}

// ---- PTX wrappers ---------------------------------------------------------

__device__ __forceinline__ int4 ld_stream(const int4* p) {
  int4 r;
  asm volatile("ld.global.nc.L1::no_allocate.v4.s32 {%0,%1,%2,%3}, [%4];"
               : "=r"(r.x), "=r"(r.y), "=r"(r.z), "=r"(r.w)
               : "l"(p));
  return r;
}

__device__ __forceinline__ void st_stream(int4* p, const int4& v) {
  asm volatile("st.global.L1::no_allocate.v4.s32 [%0], {%1,%2,%3,%4};" ::"l"(p), "r"(v.x), "r"(v.y), "r"(v.z),
               "r"(v.w)
               : "memory");
}

__device__ __forceinline__ uint32_t smem_u32(const void* p) {
  return static_cast<uint32_t>(__cvta_generic_to_shared(p));
}

__device__ __forceinline__ void mbar_init(uint64_t* bar, uint32_t count) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(bar)), "r"(count) : "memory");
}

__device__ __forceinline__ void fence_mbar_init() {
  asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
}

__device__ __forceinline__ void mbar_arrive_expect_tx(uint64_t* bar, uint32_t bytes) {
  asm volatile("mbarrier.arrive.expect_tx.release.cta.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(bar)),
               "r"(bytes)
               : "memory");
}

__device__ __forceinline__ void mbar_wait(uint64_t* bar, uint32_t phase) {
  asm volatile(
      "{\n\t.reg .pred P;\n"
      "WAIT_%=:\n\t"
      "mbarrier.try_wait.parity.acquire.cta.shared::cta.b64 P, [%0], %1;\n\t"
      "@!P bra WAIT_%=;\n}" ::"r"(smem_u32(bar)),
      "r"(phase)
      : "memory");
}

// TMA 1-D bulk copy global -> shared, completion counted on an mbarrier.
__device__ __forceinline__ void bulk_g2s(void* smem_dst, const void* gmem_src, uint32_t bytes, uint64_t* bar) {
  asm volatile(
      "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(
          smem_u32(smem_dst)),
      "l"(gmem_src), "r"(bytes), "r"(smem_u32(bar))
      : "memory");
}

// TMA 1-D bulk copy shared -> global, tracked by bulk async-groups.
__device__ __forceinline__ void bulk_s2g(void* gmem_dst, const void* smem_src, uint32_t bytes) {
  asm volatile("cp.async.bulk.global.shared::cta.bulk_group [%0], [%1], %2;" ::"l"(gmem_dst),
               "r"(smem_u32(smem_src)), "r"(bytes)
               : "memory");
}
__device__ __forceinline__ void bulk_commit() { asm volatile("cp.async.bulk.commit_group;" ::: "memory"); }
template <int N>
__device__ __forceinline__ void bulk_wait_read() {
  asm volatile("cp.async.bulk.wait_group.read %0;" ::"n"(N) : "memory");
}
template <int N>
__device__ __forceinline__ void bulk_wait() {
  asm volatile("cp.async.bulk.wait_group %0;" ::"n"(N) : "memory");
}

// Ampere-style async copy (LDGSTS), 16 bytes, L2-only caching.
__device__ __forceinline__ void cp_async16(void* smem_dst, const void* gmem_src) {
  asm volatile("cp.async.cg.shared.global [%0], [%1], 16;" ::"r"(smem_u32(smem_dst)), "l"(gmem_src) : "memory");
}
__device__ __forceinline__ void cp_async_commit() { asm volatile("cp.async.commit_group;" ::: "memory"); }
template <int N>
__device__ __forceinline__ void cp_async_wait() {
  asm volatile("cp.async.wait_group %0;" ::"n"(N) : "memory");
}

}  // namespace kvx
