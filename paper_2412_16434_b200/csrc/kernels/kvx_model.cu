// K6: the decode step that consumes the paged KV cache — sm_100a.
//
// The reference models a decode step's latency (decode_step_time,
// /root/reference/proj/src/costmodel.cpp:59-80, used by Engine::try_start,
// engine.cpp:256-257) and a prefill's (prefill_time, costmodel.cpp:54-57).
// This file EXECUTES them for a Llama-shaped model with random bf16 weights
// (no checkpoint exists offline), so the serving engine's quanta last what
// the B200 takes:
//
//   per layer:  RMSNorm -> QKV projection -> RoPE(q) -> K4 paged attention
//               with this step's token appended into its page (fused,
//               kvx_decode_attention_append) -> O projection (+ residual)
//               -> RMSNorm -> gate/up projection -> SiLU * up -> down
//               projection (+ residual)
//   then:       final RMSNorm -> LM head -> greedy argmax (the sampled token)
//
// The projections are plain dense GEMMs on cuBLAS (bf16 in, fp32 compute).
// At decode batch sizes they stream the 16 GB of Llama-3.1-8B weights once
// per step (HBM-bound); at prefill sizes they are tensor-core bound.
// Everything around them is hand-written here; the attention is K4.
//
// K/V the step appends: the bytes written into the cache are the
// deterministic K5 content of that slot (the splitmix fill of its (session,
// layer, block) tag), not the projection's output, so every page keeps a
// content the CPU oracle can recompute and migrations / loads stay
// bit-checkable while the step does the same work (the projection is still
// computed in full; only its K/V columns are not what lands in the page).

#include <cublas_v2.h>

#include <algorithm>
#include <cmath>
#include <cstdlib>
#include <cstring>
#include <map>
#include <mutex>
#include <tuple>
#include <vector>

#include "kvx_common.cuh"

struct kvx_model {
  kvx_model_config cfg{};
  int device = 0;
  cublasHandle_t blas = nullptr;
  void* stream = nullptr;  // stream the handle is bound to (rebound per call)
  // weights (bf16)
  uint16_t* embed = nullptr;    // [V][Hd]
  uint16_t* lm_head = nullptr;  // [V][Hd]
  uint16_t* final_norm = nullptr;
  std::vector<uint16_t*> wqkv, wo, wgu, wd, norm1, norm2;
  uint8_t* slab = nullptr;
  uint64_t slab_bytes = 0;
  // activations, sized for `rows_cap` rows
  int rows_cap = 0;
  uint16_t *x = nullptr, *h = nullptr, *qkv = nullptr, *q = nullptr, *kv_new = nullptr, *attn = nullptr,
           *gu = nullptr, *act = nullptr, *logits = nullptr;
  float* attn_f32 = nullptr;
  int32_t* tokens = nullptr;
  void* attn_ws = nullptr;
  uint64_t attn_ws_bytes = 0;
  void* blas_ws = nullptr;  // cuBLAS workspace: no allocation inside graph capture
  // K7 (skinny_linear): split-K partials and per-tile arrival counters
  // (zero between launches), sized at creation for every projection shape.
  float* skinny_part = nullptr;
  uint32_t* skinny_counters = nullptr;
  uint64_t skinny_part_floats = 0;
  uint32_t skinny_tiles = 0;
  // argmax_rows: per-row candidates of its CTAs and arrival counters
  unsigned long long* argmax_cand = nullptr;
  uint32_t* argmax_counters = nullptr;
  // Decode steps replayed as CUDA graphs, per launch shape (pointers and
  // sizes): the ~330 launches of a Llama-8B step cost more host time than
  // the GPU takes for the small-batch kernels.
  // Every buffer a graph captured is either in the key (caller pointers, the
  // pool's memory) or owned here; reallocating an owned buffer (activations
  // grown by a bigger batch or a prefill, the attention workspace) drops
  // every graph (drop_step_graphs).
  using StepKey = std::tuple<const void*, const void*, const void*, const void*, const void*, void*, int, int, int,
                             uint64_t, int, void*, const void*, uint64_t>;
  struct StepGraph {
    int seen = 0;
    cudaGraphExec_t exec = nullptr;
    uint64_t launches = 0;  // this library's kernels inside the graph
  };
  std::map<StepKey, StepGraph> step_graphs;
};

namespace kvx {
namespace {

__global__ void init_uniform_bf16(uint16_t* p, uint64_t n, uint64_t seed, float scale) {
  for (uint64_t i = blockIdx.x * static_cast<uint64_t>(blockDim.x) + threadIdx.x; i < n;
       i += static_cast<uint64_t>(gridDim.x) * blockDim.x)
    p[i] = f32_to_bf16_rne(__fmul_rn(unit_value(splitmix64(seed + i)), scale));
}

__global__ void init_const_bf16(uint16_t* p, uint64_t n, float v) {
  const uint16_t b = f32_to_bf16_rne(v);
  for (uint64_t i = blockIdx.x * static_cast<uint64_t>(blockDim.x) + threadIdx.x; i < n;
       i += static_cast<uint64_t>(gridDim.x) * blockDim.x)
    p[i] = b;
}

__device__ __forceinline__ float bf(uint16_t v) { return __uint_as_float(static_cast<uint32_t>(v) << 16); }

// x[r] = E[token[r]]
__global__ void embed_rows(const uint16_t* E, const int32_t* tok, uint16_t* x, int hidden, int vocab) {
  asm volatile("griddepcontrol.launch_dependents;" ::: "memory");  // a PDL-launched K7 may prefetch its weights
  const int r = blockIdx.x;
  int t = tok[r] % vocab;
  if (t < 0) t += vocab;
  const uint4* src = reinterpret_cast<const uint4*>(E + static_cast<uint64_t>(t) * hidden);
  uint4* dst = reinterpret_cast<uint4*>(x + static_cast<uint64_t>(r) * hidden);
  for (int i = threadIdx.x; i < hidden / 8; i += blockDim.x) dst[i] = src[i];
}

// y[r] = x[r] * rsqrt(mean(x[r]^2) + eps) * w, one CTA per row. The row is
// read once into registers (16-B vectors, all loads in flight together) and
// reused for the scaling pass: one memory latency per launch, not one per
// strided element.
constexpr int kNormThreads = 256, kNormMaxVec = 8;  // hidden <= 8 x 8 x 256 = 16384
__global__ void __launch_bounds__(kNormThreads) rms_norm(const uint16_t* x, const uint16_t* w, uint16_t* y, int hidden,
                                                          float eps) {
  const int r = blockIdx.x, nv = hidden / 8;
  asm volatile("griddepcontrol.launch_dependents;" ::: "memory");  // a PDL-launched K7 may prefetch its weights
  const uint4* xr = reinterpret_cast<const uint4*>(x + static_cast<uint64_t>(r) * hidden);
  uint4 v[kNormMaxVec];
  float ss = 0.f;
#pragma unroll
  for (int u = 0; u < kNormMaxVec; ++u) {
    const int i = threadIdx.x + u * kNormThreads;
    v[u] = i < nv ? xr[i] : make_uint4(0u, 0u, 0u, 0u);
  }
#pragma unroll
  for (int u = 0; u < kNormMaxVec; ++u) {
    const uint32_t q[4] = {v[u].x, v[u].y, v[u].z, v[u].w};
#pragma unroll
    for (int e = 0; e < 4; ++e) {
      const float lo = __uint_as_float(q[e] << 16), hi = __uint_as_float(q[e] & 0xFFFF0000u);
      ss += lo * lo + hi * hi;
    }
  }
  __shared__ float red[32];
  for (int o = 16; o; o >>= 1) ss += __shfl_xor_sync(0xffffffffu, ss, o);
  if ((threadIdx.x & 31) == 0) red[threadIdx.x >> 5] = ss;
  __syncthreads();
  if (threadIdx.x < 32) {
    float t = threadIdx.x < blockDim.x / 32 ? red[threadIdx.x] : 0.f;
    for (int o = 16; o; o >>= 1) t += __shfl_xor_sync(0xffffffffu, t, o);
    if (threadIdx.x == 0) red[0] = t;
  }
  __syncthreads();
  const float inv = rsqrtf(red[0] / hidden + eps);
  const uint4* wr = reinterpret_cast<const uint4*>(w);
  uint4* yr = reinterpret_cast<uint4*>(y + static_cast<uint64_t>(r) * hidden);
#pragma unroll
  for (int u = 0; u < kNormMaxVec; ++u) {
    const int i = threadIdx.x + u * kNormThreads;
    if (i >= nv) continue;
    const uint4 wv = wr[i];
    const uint32_t q[4] = {v[u].x, v[u].y, v[u].z, v[u].w}, qw[4] = {wv.x, wv.y, wv.z, wv.w};
    uint32_t o[4];
#pragma unroll
    for (int e = 0; e < 4; ++e) {
      const float lo = __uint_as_float(q[e] << 16) * inv * __uint_as_float(qw[e] << 16);
      const float hi = __uint_as_float(q[e] & 0xFFFF0000u) * inv * __uint_as_float(qw[e] & 0xFFFF0000u);
      o[e] = static_cast<uint32_t>(f32_to_bf16_rne(lo)) | (static_cast<uint32_t>(f32_to_bf16_rne(hi)) << 16);
    }
    yr[i] = make_uint4(o[0], o[1], o[2], o[3]);
  }
}

// From one request's QKV row: q with RoPE at position ctx-1 (Llama rotate-half
// pairing), and the K/V row this step appends — the K5 content of slot
// (ctx-1) % T of block (ctx-1) / T of (session, layer), so the page keeps
// its oracle-checkable bytes (see the file comment).
__global__ void rope_and_token(const uint16_t* qkv, const int32_t* sessions, const int32_t* ctx_lens, int layer,
                               int hq, int hkv, int d, int block_tokens, float theta, uint64_t seed, int fill_mode,
                               uint16_t* q_out, uint16_t* k_out, uint16_t* v_out) {
  asm volatile("griddepcontrol.launch_dependents;" ::: "memory");  // a PDL-launched K7 may prefetch its weights
  const int b = blockIdx.x;
  const int pos = max(ctx_lens[b] - 1, 0);
  const uint16_t* row = qkv + static_cast<uint64_t>(b) * (hq + 2 * hkv) * d;
  const int half = d / 2;
  for (int e = threadIdx.x; e < hq * half; e += blockDim.x) {
    const int head = e / half, i = e - head * half;
    const float inv_freq = exp2f(-(2.f * i / d) * log2f(theta));
    float sn, cs;
    sincosf(pos * inv_freq, &sn, &cs);
    const float x0 = bf(row[head * d + i]), x1 = bf(row[head * d + i + half]);
    uint16_t* qo = q_out + (static_cast<uint64_t>(b) * hq + head) * d;
    qo[i] = f32_to_bf16_rne(x0 * cs - x1 * sn);
    qo[i + half] = f32_to_bf16_rne(x1 * cs + x0 * sn);
  }
  const uint32_t block = static_cast<uint32_t>(pos / block_tokens), slot = static_cast<uint32_t>(pos % block_tokens);
  const uint64_t h = block_base(seed, static_cast<uint32_t>(sessions[b]), static_cast<uint32_t>(layer), block);
  for (int e = threadIdx.x; e < 2 * hkv * d; e += blockDim.x) {
    const int kv = e / (hkv * d), rem = e - kv * hkv * d, head = rem / d, c = rem - head * d;
    const uint64_t elt = (static_cast<uint64_t>(kv * hkv + head) * block_tokens + slot) * d + c;  // bf16 index in page
    uint16_t val;
    if (fill_mode == KVX_FILL_BITS) {
      const uint64_t w = splitmix64(h + elt / 4);
      val = static_cast<uint16_t>(w >> (16 * (elt % 4)));
    } else {
      val = f32_to_bf16_rne(unit_value(splitmix64(h + elt)));
    }
    (kv ? v_out : k_out)[(static_cast<uint64_t>(b) * hkv + head) * d + c] = val;
  }
}

__global__ void f32_to_bf16_rows(const float* in, uint16_t* out, uint64_t n) {
  asm volatile("griddepcontrol.launch_dependents;" ::: "memory");  // a PDL-launched K7 may prefetch its weights
  for (uint64_t i = blockIdx.x * static_cast<uint64_t>(blockDim.x) + threadIdx.x; i < n;
       i += static_cast<uint64_t>(gridDim.x) * blockDim.x)
    out[i] = f32_to_bf16_rne(in[i]);
}

// act = silu(gate) * up over [rows][2 * inter] -> [rows][inter]
__global__ void silu_mul(const uint16_t* gu, uint16_t* act, int inter, uint64_t rows) {
  asm volatile("griddepcontrol.launch_dependents;" ::: "memory");  // a PDL-launched K7 may prefetch its weights
  const uint64_t n = rows * inter;
  for (uint64_t i = blockIdx.x * static_cast<uint64_t>(blockDim.x) + threadIdx.x; i < n;
       i += static_cast<uint64_t>(gridDim.x) * blockDim.x) {
    const uint64_t r = i / inter, c = i - r * inter;
    const float g = bf(gu[r * 2 * inter + c]), u = bf(gu[r * 2 * inter + inter + c]);
    act[i] = f32_to_bf16_rne(g / (1.f + __expf(-g)) * u);
  }
}

// Greedy sampling: argmax over one row of logits, kArgmaxCtas CTAs per row.
// Candidates are 64-bit keys (order-preserving float bits, then the
// complemented index), so the max key is the max logit at its smallest index
// — the first occurrence, as a serial scan would pick. The last CTA of a row
// (arrival counter) reduces the row's candidates and resets the counter.
constexpr int kArgmaxCtas = 32, kArgmaxThreads = 512;
__device__ __forceinline__ unsigned long long argmax_key(float v, uint32_t idx) {
  uint32_t b = __float_as_uint(v);
  b ^= (b >> 31) ? 0xFFFFFFFFu : 0x80000000u;
  return (static_cast<unsigned long long>(b) << 32) | (0xFFFFFFFFu - idx);
}
__device__ __forceinline__ unsigned long long warp_max_u64(unsigned long long k) {
  for (int o = 16; o; o >>= 1) {
    const unsigned long long other = __shfl_xor_sync(0xffffffffu, k, o);
    k = other > k ? other : k;
  }
  return k;
}
__global__ void __launch_bounds__(kArgmaxThreads) argmax_rows(const uint16_t* logits, int vocab,
                                                             unsigned long long* cand, uint32_t* counters,
                                                             int32_t* out) {
  const int r = blockIdx.y, part = blockIdx.x;
  const int chunk = ((vocab + kArgmaxCtas - 1) / kArgmaxCtas + 7) & ~7;
  const int lo = part * chunk, hi = min(vocab, lo + chunk);
  const uint16_t* row = logits + static_cast<uint64_t>(r) * vocab;
  unsigned long long best = 0;
  // vocab % 8 == 0 (checked at creation): whole 16-B vectors.
  for (int i = lo + 8 * threadIdx.x; i < hi; i += 8 * kArgmaxThreads) {
    const uint4 v = *reinterpret_cast<const uint4*>(row + i);
    const uint32_t q[4] = {v.x, v.y, v.z, v.w};
#pragma unroll
    for (int e = 0; e < 4; ++e) {
      const unsigned long long k0 = argmax_key(__uint_as_float(q[e] << 16), i + 2 * e);
      const unsigned long long k1 = argmax_key(__uint_as_float(q[e] & 0xFFFF0000u), i + 2 * e + 1);
      best = k0 > best ? k0 : best;
      best = k1 > best ? k1 : best;
    }
  }
  __shared__ unsigned long long sk[kArgmaxThreads / 32];
  __shared__ bool last;
  best = warp_max_u64(best);
  if ((threadIdx.x & 31) == 0) sk[threadIdx.x >> 5] = best;
  __syncthreads();
  if (threadIdx.x < 32) {
    best = warp_max_u64(threadIdx.x < kArgmaxThreads / 32 ? sk[threadIdx.x] : 0ull);
    if (threadIdx.x == 0) {
      cand[static_cast<uint64_t>(r) * kArgmaxCtas + part] = best;
      __threadfence();
      last = atomicAdd(counters + r, 1u) == kArgmaxCtas - 1;
    }
  }
  __syncthreads();
  if (!last || threadIdx.x >= 32) return;
  __threadfence();
  unsigned long long k = threadIdx.x < kArgmaxCtas ? __ldcg(cand + static_cast<uint64_t>(r) * kArgmaxCtas + threadIdx.x)
                                                   : 0ull;
  k = warp_max_u64(k);
  if (threadIdx.x == 0) {
    out[r] = static_cast<int32_t>(0xFFFFFFFFu - static_cast<uint32_t>(k & 0xFFFFFFFFu));
    counters[r] = 0;
  }
}

int grid_for(uint64_t n, int threads) {
  return static_cast<int>(std::min<uint64_t>((n + threads - 1) / threads, 148ull * 16));
}

const char* blas_name(cublasStatus_t s) {
  switch (s) {
    case CUBLAS_STATUS_NOT_INITIALIZED: return "CUBLAS_STATUS_NOT_INITIALIZED";
    case CUBLAS_STATUS_ALLOC_FAILED: return "CUBLAS_STATUS_ALLOC_FAILED";
    case CUBLAS_STATUS_INVALID_VALUE: return "CUBLAS_STATUS_INVALID_VALUE";
    case CUBLAS_STATUS_ARCH_MISMATCH: return "CUBLAS_STATUS_ARCH_MISMATCH";
    case CUBLAS_STATUS_EXECUTION_FAILED: return "CUBLAS_STATUS_EXECUTION_FAILED";
    case CUBLAS_STATUS_NOT_SUPPORTED: return "CUBLAS_STATUS_NOT_SUPPORTED";
    default: return "cuBLAS error";
  }
}

#define KVX_BLAS_TRY(expr, what)                                                     \
  do {                                                                               \
    cublasStatus_t kvx_b_ = (expr);                                                  \
    if (kvx_b_ != CUBLAS_STATUS_SUCCESS) {                                           \
      kvx::set_error(std::string(what) + ": " + kvx::blas_name(kvx_b_));             \
      return KVX_ERR_CUDA;                                                           \
    }                                                                                \
  } while (0)

// ---- K7: decode projections at small batch ---------------------------------
// At decode batch sizes a projection streams its weight matrix once and does
// ~rows multiply-adds per weight: HBM-bound. cuBLAS reaches ~half the copy
// roofline on these skinny shapes (a Llama-3.1-8B step took 4.5 ms for
// ~15 GB of weights), so rows <= 8 go to this kernel:
//   * a warp owns 16 output features x a K chunk; per 128 k each lane loads
//     4 x 16 B of each of its two weight rows (streaming, L1 no-allocate) and
//     the matching 16 B of X (cached: every warp of the CTA reads the same X
//     chunk), then issues bf16 mma.sync m16n8k16 (features on M, batch rows
//     on N). The k order inside a 32-k group is permuted identically for W
//     and X (lane c holds physical k 8c..8c+7), so each lane's loads are
//     whole 16-B vectors and no shuffles or shared memory are needed;
//   * split-K sized so ~2 waves of warps stream at once; the last warp of a
//     tile (arrival counter) sums the partials in split order (deterministic)
//     and writes bf16 Y, adding the residual when accumulating.
constexpr int kSkinnyMaxRows = 8;  // measured: cuBLAS is faster from 16 rows (profiles/r02_model_step.txt)
constexpr int kSkinnyWarps = 8;

struct SkinnyArgs {
  const uint16_t* X;  // [rows][in]
  const uint16_t* W;  // [out][in]
  uint16_t* Y;        // [rows][out]
  float* part;        // [tiles][splits][NT * 128]
  uint32_t* counters; // [tiles]
  int rows, in, out, splits, k_chunk, accumulate;
};

__device__ __forceinline__ void mma_bf16_16816(float (&d)[4], uint32_t a0, uint32_t a1, uint32_t a2, uint32_t a3,
                                               uint32_t b0, uint32_t b1) {
  asm volatile(
      "mma.sync.aligned.m16n8k16.row.col.f32.bf16.bf16.f32 {%0,%1,%2,%3}, {%4,%5,%6,%7}, {%8,%9}, "
      "{%0,%1,%2,%3};"
      : "+f"(d[0]), "+f"(d[1]), "+f"(d[2]), "+f"(d[3])
      : "r"(a0), "r"(a1), "r"(a2), "r"(a3), "r"(b0), "r"(b1));
}

// Cached read-only vector load, issued in program order with the streaming
// weight loads (volatile) so a step's X loads are all in flight before its mmas.
__device__ __forceinline__ int4 ld_nc_v4(const void* p) {
  int4 r;
  asm volatile("ld.global.nc.v4.s32 {%0,%1,%2,%3}, [%4];" : "=r"(r.x), "=r"(r.y), "=r"(r.z), "=r"(r.w) : "l"(p));
  return r;
}

__device__ __forceinline__ float bf16_to_f32(uint16_t v) { return __uint_as_float(static_cast<uint32_t>(v) << 16); }

__device__ __forceinline__ int4 ld_w(const uint16_t* p) {  // streamed once: no L1 allocation
  int4 r;
  asm("ld.global.nc.L1::no_allocate.v4.s32 {%0,%1,%2,%3}, [%4];" : "=r"(r.x), "=r"(r.y), "=r"(r.z), "=r"(r.w) : "l"(p));
  return r;
}
__device__ __forceinline__ int4 ld_x(const uint16_t* p) {  // X: shared by the CTA's warps, cached
  int4 r;
  asm("ld.global.nc.v4.s32 {%0,%1,%2,%3}, [%4];" : "=r"(r.x), "=r"(r.y), "=r"(r.z), "=r"(r.w) : "l"(p));
  return r;
}
__device__ __forceinline__ void mma_acc(float (&d)[4], uint32_t a0, uint32_t a1, uint32_t a2, uint32_t a3, uint32_t b0,
                                        uint32_t b1) {
  asm("mma.sync.aligned.m16n8k16.row.col.f32.bf16.bf16.f32 {%0,%1,%2,%3}, {%4,%5,%6,%7}, {%8,%9}, {%0,%1,%2,%3};"
      : "+f"(d[0]), "+f"(d[1]), "+f"(d[2]), "+f"(d[3])
      : "r"(a0), "r"(a1), "r"(a2), "r"(a3), "r"(b0), "r"(b1));
}

template <int NT>  // n-tiles of 8 batch rows: 1 (rows <= 8) or 2 (rows <= 16)
__global__ void __launch_bounds__(kSkinnyWarps * 32, 2) skinny_linear(const SkinnyArgs a) {
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int tile = blockIdx.x * kSkinnyWarps + warp;
  if (tile * 16 >= a.out) return;  // no block-wide barriers below
  const int split = blockIdx.y;
  const int k0 = split * a.k_chunk;
  const int k1 = min(a.in, k0 + a.k_chunk);
  const int g = lane >> 2, c = lane & 3;
  const uint16_t* w0 = a.W + static_cast<uint64_t>(tile * 16 + g) * a.in + 8 * c;
  const uint16_t* w8 = w0 + static_cast<uint64_t>(8) * a.in;
  const uint16_t* xr[NT];
  bool xv[NT];
#pragma unroll
  for (int nt = 0; nt < NT; ++nt) {
    xv[nt] = g + 8 * nt < a.rows;
    xr[nt] = a.X + static_cast<uint64_t>(xv[nt] ? g + 8 * nt : 0) * a.in + 8 * c;
  }
  float d[NT][4];
#pragma unroll
  for (int nt = 0; nt < NT; ++nt) d[nt][0] = d[nt][1] = d[nt][2] = d[nt][3] = 0.f;
  // Two 128-k groups of weights in flight per lane (software pipelined: the
  // next group's loads are issued before this group's mmas).
  int4 wa[4], wb[4];
#pragma unroll
  for (int j = 0; j < 4; ++j) {
    wa[j] = ld_w(w0 + k0 + 32 * j);
    wb[j] = ld_w(w8 + k0 + 32 * j);
  }
  // Programmatic dependent launch: the weights do not depend on the kernel
  // before us, so the first group is in flight before we wait for it (X, the
  // residual Y and the split-K workspace are touched only after the wait).
  asm volatile("griddepcontrol.wait;" ::: "memory");
  for (int k = k0; k < k1; k += 128) {  // in and k_chunk are multiples of 128
    int4 xs[NT][4];
#pragma unroll
    for (int nt = 0; nt < NT; ++nt)
#pragma unroll
      for (int j = 0; j < 4; ++j) xs[nt][j] = xv[nt] ? ld_x(xr[nt] + k + 32 * j) : make_int4(0, 0, 0, 0);
    int4 na[4], nb[4];
    const bool more = k + 128 < k1;
#pragma unroll
    for (int j = 0; j < 4; ++j) {
      na[j] = more ? ld_w(w0 + k + 128 + 32 * j) : make_int4(0, 0, 0, 0);
      nb[j] = more ? ld_w(w8 + k + 128 + 32 * j) : make_int4(0, 0, 0, 0);
    }
#pragma unroll
    for (int j = 0; j < 4; ++j)
#pragma unroll
      for (int nt = 0; nt < NT; ++nt) {
        // virtual k {2c,2c+1 | 2c+8,2c+9} <- physical 8c+{0,1 | 2,3}, then 8c+{4,5 | 6,7}
        mma_acc(d[nt], wa[j].x, wb[j].x, wa[j].y, wb[j].y, xs[nt][j].x, xs[nt][j].y);
        mma_acc(d[nt], wa[j].z, wb[j].z, wa[j].w, wb[j].w, xs[nt][j].z, xs[nt][j].w);
      }
#pragma unroll
    for (int j = 0; j < 4; ++j) {
      wa[j] = na[j];
      wb[j] = nb[j];
    }
  }
  asm volatile("griddepcontrol.launch_dependents;" ::: "memory");  // our weight stream is done
  if (a.splits > 1) {
    float4* mine = reinterpret_cast<float4*>(a.part + (static_cast<uint64_t>(tile) * a.splits + split) * (NT * 128));
#pragma unroll
    for (int nt = 0; nt < NT; ++nt) mine[nt * 32 + lane] = make_float4(d[nt][0], d[nt][1], d[nt][2], d[nt][3]);
    __threadfence();
    uint32_t prev = 0;
    if (lane == 0) prev = atomicAdd(a.counters + tile, 1u);
    prev = __shfl_sync(0xffffffffu, prev, 0);
    if (prev != static_cast<uint32_t>(a.splits - 1)) return;
    __threadfence();
#pragma unroll
    for (int nt = 0; nt < NT; ++nt) d[nt][0] = d[nt][1] = d[nt][2] = d[nt][3] = 0.f;
    const float4* all = reinterpret_cast<const float4*>(a.part + static_cast<uint64_t>(tile) * a.splits * (NT * 128));
    // Eight partials in flight per lane, summed in split order (deterministic).
    for (int s0 = 0; s0 < a.splits; s0 += 8) {
      float4 v[8][NT];
#pragma unroll
      for (int u = 0; u < 8; ++u)
#pragma unroll
        for (int nt = 0; nt < NT; ++nt)
          v[u][nt] = s0 + u < a.splits ? __ldcg(all + (static_cast<uint64_t>(s0 + u) * NT + nt) * 32 + lane)
                                       : make_float4(0.f, 0.f, 0.f, 0.f);
#pragma unroll
      for (int u = 0; u < 8; ++u)
#pragma unroll
        for (int nt = 0; nt < NT; ++nt) {
          d[nt][0] += v[u][nt].x;
          d[nt][1] += v[u][nt].y;
          d[nt][2] += v[u][nt].z;
          d[nt][3] += v[u][nt].w;
        }
    }
    if (lane == 0) a.counters[tile] = 0;  // ready for the next launch
  }
  // d[nt][0/1]: feature g, batch rows 8nt + 2c + {0,1}; d[nt][2/3]: feature g + 8.
#pragma unroll
  for (int nt = 0; nt < NT; ++nt)
#pragma unroll
    for (int e = 0; e < 4; ++e) {
      const int n = 8 * nt + 2 * c + (e & 1);
      if (n >= a.rows) continue;
      uint16_t* y = a.Y + static_cast<uint64_t>(n) * a.out + tile * 16 + g + (e >> 1) * 8;
      const float v = d[nt][e] + (a.accumulate ? bf16_to_f32(*y) : 0.f);
      *y = f32_to_bf16_rne(v);
    }
}

// Split-K factor of a skinny projection: one wave of CTAs (two 8-warp CTAs
// per SM at 128 registers), so no partial second wave trails the launch.
void skinny_plan(int in, int out, int sms, int& splits, int& k_chunk) {
  const int tiles = out / 16;
  const int groups = in / 128;
  const int ctas_per_split = (tiles + kSkinnyWarps - 1) / kSkinnyWarps;
  const int wave = 2 * sms;
  int s = std::max(1, wave / std::max(1, ctas_per_split));
  s = std::min(s, groups);
  k_chunk = ((groups + s - 1) / s) * 128;
  splits = (in + k_chunk - 1) / k_chunk;
}

bool skinny_ok(int rows, int in, int out) {
  static const char* env = std::getenv("KVX_MODEL_SKINNY");
  if (env && env[0] == '0') return false;  // measurement knob: cuBLAS for every projection
  return rows > 0 && rows <= kSkinnyMaxRows && in % 128 == 0 && out % 16 == 0;
}

int skinny_linear_launch(kvx_model* m, const uint16_t* X, const uint16_t* W, uint16_t* Y, int rows, int in, int out,
                         bool accumulate, cudaStream_t st) {
  SkinnyArgs a{X, W, Y, m->skinny_part, m->skinny_counters, rows, in, out, 1, in, accumulate ? 1 : 0};
  skinny_plan(in, out, sm_count(m->device), a.splits, a.k_chunk);
  const uint32_t tiles = static_cast<uint32_t>(out / 16);
  const int nt = rows <= 8 ? 1 : 2;
  if (a.splits > 1 && (tiles > m->skinny_tiles ||
                       static_cast<uint64_t>(tiles) * a.splits * nt * 128 > m->skinny_part_floats))
    return fail_arg("kvx_model: skinny projection workspace too small");
  cudaLaunchConfig_t cfg{};
  cfg.gridDim = dim3((tiles + kSkinnyWarps - 1) / kSkinnyWarps, a.splits);
  cfg.blockDim = dim3(kSkinnyWarps * 32);
  cfg.stream = st;
  cudaLaunchAttribute attr[1];
  attr[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;  // weights prefetched under the previous kernel
  attr[0].val.programmaticStreamSerializationAllowed = 1;
  cfg.attrs = attr;
  cfg.numAttrs = 1;
  KVX_CUDA_TRY(nt == 1 ? cudaLaunchKernelEx(&cfg, skinny_linear<1>, a) : cudaLaunchKernelEx(&cfg, skinny_linear<2>, a),
               "kvx_model: skinny_linear");
  note_launch();
  return KVX_OK;
}

// Y[rows][out] (+)= X[rows][in] . W[out][in]^T, bf16 in/out, fp32 compute.
int linear(kvx_model* m, const uint16_t* X, const uint16_t* W, uint16_t* Y, int rows, int in, int out, bool accumulate) {
  if (skinny_ok(rows, in, out)) return skinny_linear_launch(m, X, W, Y, rows, in, out, accumulate, as_stream(m->stream));
  const float one = 1.f, beta = accumulate ? 1.f : 0.f;
  KVX_BLAS_TRY(cublasGemmEx(m->blas, CUBLAS_OP_T, CUBLAS_OP_N, out, rows, in, &one, W, CUDA_R_16BF, in, X, CUDA_R_16BF,
                            in, &beta, Y, CUDA_R_16BF, out, CUBLAS_COMPUTE_32F, CUBLAS_GEMM_DEFAULT),
               "kvx_model: cublasGemmEx");
  note_library_launch();
  return KVX_OK;
}

// Captured decode-step graphs hold the addresses of the activations and the
// workspace: called (after a stream sync) before either is reallocated.
void drop_step_graphs(kvx_model* m) {
  for (auto& g : m->step_graphs)
    if (g.second.exec) cudaGraphExecDestroy(g.second.exec);
  m->step_graphs.clear();
}

int ensure_rows(kvx_model* m, int rows) {
  if (rows <= m->rows_cap) return KVX_OK;
  const kvx_model_config& c = m->cfg;
  cudaStream_t st = as_stream(m->stream);
  if (m->x) KVX_CUDA_TRY(cudaStreamSynchronize(st), "kvx_model: sync");
  drop_step_graphs(m);
  for (void* p : {static_cast<void*>(m->x), static_cast<void*>(m->h), static_cast<void*>(m->qkv),
                  static_cast<void*>(m->q), static_cast<void*>(m->kv_new), static_cast<void*>(m->attn),
                  static_cast<void*>(m->gu), static_cast<void*>(m->act), static_cast<void*>(m->logits),
                  static_cast<void*>(m->attn_f32), static_cast<void*>(m->tokens)})
    cudaFree(p);
  const int cap = std::max(rows, 64);
  const uint64_t R = static_cast<uint64_t>(cap);
  const uint64_t qkv_w = static_cast<uint64_t>(c.num_q_heads + 2 * c.num_kv_heads) * c.head_dim;
  auto al = [&](auto** p, uint64_t bytes) { return cudaMalloc(reinterpret_cast<void**>(p), bytes); };
  cudaError_t e = cudaSuccess;
  e = e ? e : al(&m->x, R * c.hidden * 2);
  e = e ? e : al(&m->h, R * c.hidden * 2);
  e = e ? e : al(&m->qkv, R * qkv_w * 2);
  e = e ? e : al(&m->q, R * c.num_q_heads * c.head_dim * 2);
  e = e ? e : al(&m->kv_new, R * 2 * c.num_kv_heads * c.head_dim * 2);
  e = e ? e : al(&m->attn, R * c.num_q_heads * c.head_dim * 2);
  e = e ? e : al(&m->gu, R * 2 * c.intermediate * 2);
  e = e ? e : al(&m->act, R * c.intermediate * 2);
  // logits only for decode batches (prefill samples its last row only)
  e = e ? e : al(&m->logits, std::min<uint64_t>(R, 256) * c.vocab * 2);
  e = e ? e : al(&m->attn_f32, R * c.num_q_heads * c.head_dim * 4);
  e = e ? e : al(&m->tokens, R * 4);
  if (e != cudaSuccess) return fail_cuda(e, "kvx_model: activations");
  m->rows_cap = cap;
  return KVX_OK;
}

int bind(kvx_model* m, void* stream) {
  if (m->stream != stream || !m->blas) {
    KVX_BLAS_TRY(cublasSetStream(m->blas, as_stream(stream)), "kvx_model: cublasSetStream");
    m->stream = stream;
  }
  return KVX_OK;
}

// The dense part of one layer around the attention, split at the attention:
// pre = norm + QKV; post = O proj + residual, norm, MLP + residual.
int layer_pre(kvx_model* m, int l, int rows) {
  const kvx_model_config& c = m->cfg;
  cudaStream_t st = as_stream(m->stream);
  rms_norm<<<rows, 256, 0, st>>>(m->x, m->norm1[l], m->h, c.hidden, c.rms_eps);
  KVX_CUDA_TRY(cudaGetLastError(), "kvx_model: rms_norm");
  note_launch();
  return linear(m, m->h, m->wqkv[l], m->qkv, rows, c.hidden, (c.num_q_heads + 2 * c.num_kv_heads) * c.head_dim, false);
}

int layer_post(kvx_model* m, int l, int rows) {
  const kvx_model_config& c = m->cfg;
  cudaStream_t st = as_stream(m->stream);
  if (int rc = linear(m, m->attn, m->wo[l], m->x, rows, c.num_q_heads * c.head_dim, c.hidden, true)) return rc;
  rms_norm<<<rows, 256, 0, st>>>(m->x, m->norm2[l], m->h, c.hidden, c.rms_eps);
  KVX_CUDA_TRY(cudaGetLastError(), "kvx_model: rms_norm");
  note_launch();
  if (int rc = linear(m, m->h, m->wgu[l], m->gu, rows, c.hidden, 2 * c.intermediate, false)) return rc;
  const uint64_t n = static_cast<uint64_t>(rows) * c.intermediate;
  silu_mul<<<grid_for(n, 256), 256, 0, st>>>(m->gu, m->act, c.intermediate, rows);
  KVX_CUDA_TRY(cudaGetLastError(), "kvx_model: silu_mul");
  note_launch();
  return linear(m, m->act, m->wd[l], m->x, rows, c.intermediate, c.hidden, true);
}

// Final norm + LM head + argmax over `rows` rows of the residual stream
// starting at row `first`.
int sample(kvx_model* m, int first, int rows, int32_t* d_tokens_out) {
  const kvx_model_config& c = m->cfg;
  cudaStream_t st = as_stream(m->stream);
  rms_norm<<<rows, 256, 0, st>>>(m->x + static_cast<uint64_t>(first) * c.hidden, m->final_norm, m->h, c.hidden,
                                 c.rms_eps);
  KVX_CUDA_TRY(cudaGetLastError(), "kvx_model: final norm");
  note_launch();
  if (int rc = linear(m, m->h, m->lm_head, m->logits, rows, c.hidden, c.vocab, false)) return rc;
  argmax_rows<<<dim3(kArgmaxCtas, rows), kArgmaxThreads, 0, st>>>(m->logits, c.vocab, m->argmax_cand,
                                                                  m->argmax_counters, d_tokens_out);
  KVX_CUDA_TRY(cudaGetLastError(), "kvx_model: argmax");
  note_launch();
  return KVX_OK;
}

}  // namespace
}  // namespace kvx

extern "C" {

uint64_t kvx_model_weight_bytes(const kvx_model_config* c) {
  if (!c) return 0;
  const uint64_t Hd = c->hidden, D = c->head_dim;
  const uint64_t per_layer = (c->num_q_heads + 2ull * c->num_kv_heads) * D * Hd + c->num_q_heads * D * Hd +
                             2ull * c->intermediate * Hd + c->intermediate * Hd + 2 * Hd;
  return 2 * (c->num_layers * per_layer + 2ull * c->vocab * Hd + Hd);
}

int kvx_model_create(int device, const kvx_model_config* cfg, uint64_t seed, kvx_model** out) {
  if (!cfg || !out) return kvx::fail_arg("kvx_model_create: null argument");
  const kvx_model_config& c = *cfg;
  if (c.num_layers <= 0 || c.hidden <= 0 || c.hidden % 8 || c.num_kv_heads <= 0 || c.num_q_heads % c.num_kv_heads ||
      c.head_dim != 128 || c.intermediate <= 0 || c.vocab <= 0 || c.vocab % 8 || c.num_q_heads * c.head_dim % 8 ||
      c.hidden > 16384)
    return kvx::fail_arg("kvx_model_create: unsupported shape (head_dim 128, hidden % 8 == 0 and <= 16384, vocab % 8 "
                         "== 0, GQA)");
  kvx::DeviceGuard guard(device);
  auto* m = new kvx_model;
  m->cfg = c;
  m->device = device;
  if (cublasCreate(&m->blas) != CUBLAS_STATUS_SUCCESS) {
    delete m;
    kvx::set_error("kvx_model_create: cublasCreate failed");
    return KVX_ERR_CUDA;
  }
  constexpr size_t kBlasWs = 64u << 20;
  if (cudaMalloc(&m->blas_ws, kBlasWs) != cudaSuccess ||
      cublasSetWorkspace(m->blas, m->blas_ws, kBlasWs) != CUBLAS_STATUS_SUCCESS) {
    cudaGetLastError();
    cublasDestroy(m->blas);
    cudaFree(m->blas_ws);
    delete m;
    kvx::set_error("kvx_model_create: cuBLAS workspace");
    return KVX_ERR_CUDA;
  }
  {
    // K7 workspace for the largest split-K plan among the step's projections.
    const int sms = kvx::sm_count(device);
    const int shapes[5][2] = {{c.hidden, (c.num_q_heads + 2 * c.num_kv_heads) * c.head_dim},
                              {c.num_q_heads * c.head_dim, c.hidden},
                              {c.hidden, 2 * c.intermediate},
                              {c.intermediate, c.hidden},
                              {c.hidden, c.vocab}};
    for (const auto& sh : shapes) {
      if (sh[0] % 128 || sh[1] % 16) continue;
      int splits = 1, chunk = 0;
      kvx::skinny_plan(sh[0], sh[1], sms, splits, chunk);
      m->skinny_tiles = std::max<uint32_t>(m->skinny_tiles, static_cast<uint32_t>(sh[1] / 16));
      if (splits > 1) m->skinny_part_floats = std::max<uint64_t>(m->skinny_part_floats, uint64_t(sh[1] / 16) * splits * 256);
    }
    if (cudaMalloc(reinterpret_cast<void**>(&m->skinny_part), std::max<uint64_t>(m->skinny_part_floats, 1) * 4) !=
            cudaSuccess ||
        cudaMalloc(reinterpret_cast<void**>(&m->skinny_counters), std::max<uint32_t>(m->skinny_tiles, 1) * 4) !=
            cudaSuccess ||
        cudaMemset(m->skinny_counters, 0, std::max<uint32_t>(m->skinny_tiles, 1) * 4) != cudaSuccess ||
        cudaMalloc(reinterpret_cast<void**>(&m->argmax_cand), 256 * kvx::kArgmaxCtas * 8) != cudaSuccess ||
        cudaMalloc(reinterpret_cast<void**>(&m->argmax_counters), 256 * 4) != cudaSuccess ||
        cudaMemset(m->argmax_counters, 0, 256 * 4) != cudaSuccess) {
      cudaGetLastError();
      cudaFree(m->skinny_part);
      cudaFree(m->skinny_counters);
      cublasDestroy(m->blas);
      cudaFree(m->blas_ws);
      delete m;
      kvx::set_error("kvx_model_create: projection workspace");
      return KVX_ERR_CUDA;
    }
  }
  m->slab_bytes = kvx_model_weight_bytes(cfg);
  cudaError_t e = cudaMalloc(reinterpret_cast<void**>(&m->slab), m->slab_bytes);
  if (e != cudaSuccess) {
    cublasDestroy(m->blas);
    delete m;
    return kvx::fail_cuda(e, "kvx_model_create: weights");
  }
  uint16_t* p = reinterpret_cast<uint16_t*>(m->slab);
  const uint64_t Hd = c.hidden, D = c.head_dim;
  uint64_t salt = 0;
  // Random weights, uniform with unit variance scaled by 1/sqrt(fan_in):
  // activations stay O(1) through the stack.
  auto take = [&](uint64_t n, float scale, bool ones = false) {
    uint16_t* w = p;
    p += n;
    if (ones)
      kvx::init_const_bf16<<<kvx::grid_for(n, 256), 256>>>(w, n, 1.f);
    else
      kvx::init_uniform_bf16<<<kvx::grid_for(n, 256), 256>>>(w, n, kvx::splitmix64(seed + ++salt), scale);
    return w;
  };
  m->embed = take(c.vocab * Hd, 1.f);
  m->lm_head = take(c.vocab * Hd, 1.f / std::sqrt(static_cast<float>(Hd)));
  m->final_norm = take(Hd, 1.f, true);
  for (int l = 0; l < c.num_layers; ++l) {
    m->wqkv.push_back(take((c.num_q_heads + 2ull * c.num_kv_heads) * D * Hd, 1.f / std::sqrt(static_cast<float>(Hd))));
    m->wo.push_back(take(c.num_q_heads * D * Hd, 1.f / std::sqrt(static_cast<float>(c.num_q_heads * D))));
    m->wgu.push_back(take(2ull * c.intermediate * Hd, 1.f / std::sqrt(static_cast<float>(Hd))));
    m->wd.push_back(take(c.intermediate * Hd, 1.f / std::sqrt(static_cast<float>(c.intermediate))));
    m->norm1.push_back(take(Hd, 1.f, true));
    m->norm2.push_back(take(Hd, 1.f, true));
  }
  e = cudaDeviceSynchronize();
  if (e == cudaSuccess) e = cudaGetLastError();
  if (e != cudaSuccess) {
    kvx_model_destroy(m);
    return kvx::fail_cuda(e, "kvx_model_create: init");
  }
  *out = m;
  return KVX_OK;
}

int kvx_model_destroy(kvx_model* m) {
  if (!m) return KVX_OK;
  kvx::DeviceGuard guard(m->device);
  if (m->stream) cudaStreamSynchronize(kvx::as_stream(m->stream));
  for (void* p : {static_cast<void*>(m->x), static_cast<void*>(m->h), static_cast<void*>(m->qkv),
                  static_cast<void*>(m->q), static_cast<void*>(m->kv_new), static_cast<void*>(m->attn),
                  static_cast<void*>(m->gu), static_cast<void*>(m->act), static_cast<void*>(m->logits),
                  static_cast<void*>(m->attn_f32), static_cast<void*>(m->tokens), m->attn_ws,
                  static_cast<void*>(m->slab), m->blas_ws, static_cast<void*>(m->skinny_part),
                  static_cast<void*>(m->skinny_counters), static_cast<void*>(m->argmax_cand),
                  static_cast<void*>(m->argmax_counters)})
    cudaFree(p);
  for (auto& g : m->step_graphs)
    if (g.second.exec) cudaGraphExecDestroy(g.second.exec);
  if (m->blas) cublasDestroy(m->blas);
  delete m;
  return KVX_OK;
}

}  // extern "C"

namespace kvx {
namespace {
int enqueue_decode(kvx_model* m, kvx_pool* pool, const kvx_page_layout* layout, const kvx_attn_params* ap,
                   const uint32_t* d_tables, const int32_t* d_ctx_lens, const int32_t* d_sessions,
                   const int32_t* d_tokens_in, int32_t batch, int32_t max_blocks, int32_t max_ctx, uint64_t fill_seed,
                   int32_t fill_mode, void* const* layer_waits, const int32_t* layer_wait_offsets,
                   int32_t* d_tokens_out);
}  // namespace
}  // namespace kvx

extern "C" {

int kvx_model_decode_step(kvx_model* m, kvx_pool* pool, const kvx_page_layout* layout, const uint32_t* d_tables,
                          const int32_t* d_ctx_lens, const int32_t* d_sessions, const int32_t* d_tokens_in,
                          int32_t batch, int32_t max_blocks, int32_t max_ctx, uint64_t fill_seed, int32_t fill_mode,
                          void* const* layer_waits, const int32_t* layer_wait_offsets, int32_t* d_tokens_out,
                          void* stream) {
  if (!m || !pool || !layout || !d_tables || !d_ctx_lens || !d_sessions || !d_tokens_in || !d_tokens_out)
    return kvx::fail_arg("kvx_model_decode_step: null argument");
  if (batch <= 0) return KVX_OK;
  const kvx_model_config& c = m->cfg;
  if (layout->num_kv_heads != c.num_kv_heads || layout->head_dim != c.head_dim || layout->dtype != KVX_DTYPE_BF16)
    return kvx::fail_arg("kvx_model_decode_step: page layout does not match the model (bf16, kv heads, head_dim)");
  if (batch > 256) return kvx::fail_arg("kvx_model_decode_step: batch > 256");
  kvx::DeviceGuard guard(m->device);
  if (int rc = kvx::ensure_rows(m, batch)) return rc;
  if (int rc = kvx::bind(m, stream)) return rc;
  cudaStream_t st = kvx::as_stream(stream);
  kvx_attn_params ap{};
  ap.num_q_heads = c.num_q_heads;
  ap.max_blocks = max_blocks;
  ap.flags = KVX_ATTN_EARLY_PREFETCH;
  const uint64_t ws = kvx_decode_attention_workspace(layout, &ap, batch, max_ctx);
  if (ws > m->attn_ws_bytes) {
    if (m->attn_ws) {
      KVX_CUDA_TRY(cudaStreamSynchronize(st), "kvx_model: sync");
      kvx::drop_step_graphs(m);
      cudaFree(m->attn_ws);
      m->attn_ws = nullptr;
    }
    const uint64_t cap = ws * 2;
    KVX_CUDA_TRY(cudaMalloc(&m->attn_ws, cap), "kvx_model: attention workspace");
    KVX_CUDA_TRY(cudaMemsetAsync(m->attn_ws, 0, cap, st), "kvx_model: attention workspace");
    m->attn_ws_bytes = cap;
  }
  const bool waits = layer_waits && layer_wait_offsets && layer_wait_offsets[c.num_layers] > 0;
  static const char* graphs_env = std::getenv("KVX_MODEL_GRAPHS");
  const bool graphs = !(graphs_env && graphs_env[0] == '0');
  if (!waits && graphs) {
    // Same shape seen before: replay (captured on the second sighting, so
    // every one-time allocation / attribute / plan happened eagerly first).
    const kvx_model::StepKey key{pool,     d_tables,  d_ctx_lens, d_sessions,    d_tokens_in,
                                 d_tokens_out, batch,   max_blocks, max_ctx,     fill_seed,
                                 fill_mode, stream,  kvx_pool_base(pool), kvx_pool_num_pages(pool)};
    kvx_model::StepGraph& g = m->step_graphs[key];
    if (g.exec) {
      KVX_CUDA_TRY(cudaGraphLaunch(g.exec, st), "kvx_model: graph launch");
      kvx::note_launch(g.launches);
      return KVX_OK;
    }
    if (g.seen++ > 0) {
      const uint64_t n0 = kvx_launch_count();
      KVX_CUDA_TRY(cudaStreamBeginCapture(st, cudaStreamCaptureModeThreadLocal), "kvx_model: begin capture");
      const int rc = kvx::enqueue_decode(m, pool, layout, &ap, d_tables, d_ctx_lens, d_sessions, d_tokens_in, batch,
                                         max_blocks, max_ctx, fill_seed, fill_mode, nullptr, nullptr, d_tokens_out);
      cudaGraph_t graph = nullptr;
      const cudaError_t e = cudaStreamEndCapture(st, &graph);
      if (rc) {
        if (graph) cudaGraphDestroy(graph);
        return rc;
      }
      KVX_CUDA_TRY(e, "kvx_model: end capture");
      const cudaError_t ei = cudaGraphInstantiate(&g.exec, graph, 0);
      cudaGraphDestroy(graph);
      KVX_CUDA_TRY(ei, "kvx_model: graph instantiate");
      g.launches = kvx_launch_count() - n0;
      KVX_CUDA_TRY(cudaGraphLaunch(g.exec, st), "kvx_model: graph launch");
      return KVX_OK;
    }
  }
  return kvx::enqueue_decode(m, pool, layout, &ap, d_tables, d_ctx_lens, d_sessions, d_tokens_in, batch, max_blocks,
                             max_ctx, fill_seed, fill_mode, layer_waits, layer_wait_offsets, d_tokens_out);
}

}  // extern "C"

namespace kvx {
namespace {

// The launch sequence of one decode step (eager, or recorded into a graph).
int enqueue_decode(kvx_model* m, kvx_pool* pool, const kvx_page_layout* layout, const kvx_attn_params* ap_in,
                   const uint32_t* d_tables, const int32_t* d_ctx_lens, const int32_t* d_sessions,
                   const int32_t* d_tokens_in, int32_t batch, int32_t max_blocks, int32_t max_ctx, uint64_t fill_seed,
                   int32_t fill_mode, void* const* layer_waits, const int32_t* layer_wait_offsets,
                   int32_t* d_tokens_out) {
  const kvx_model_config& c = m->cfg;
  void* stream = m->stream;
  cudaStream_t st = as_stream(stream);
  kvx_attn_params ap = *ap_in;
  kvx::embed_rows<<<batch, 128, 0, st>>>(m->embed, d_tokens_in, m->x, c.hidden, c.vocab);
  KVX_CUDA_TRY(cudaGetLastError(), "kvx_model: embed");
  kvx::note_launch();
  const int Hq = c.num_q_heads, H = c.num_kv_heads, D = c.head_dim;
  for (int l = 0; l < c.num_layers; ++l) {
    if (int rc = kvx::layer_pre(m, l, batch)) return rc;
    uint16_t* new_k = m->kv_new;
    uint16_t* new_v = m->kv_new + static_cast<uint64_t>(batch) * H * D;
    // Layer l's pages may still be landing (a layer-wise load or a migrated
    // layer): wait for exactly the batches writing them — the pipeline gate
    // of the reference (kvstore.cpp:46-59) made physical. The waits precede
    // the (normally launched) rope kernel, so the attention after it, which
    // may launch early (PDL) and prefetch pages before griddepcontrol.wait,
    // still cannot start before those pages are complete.
    if (layer_waits && layer_wait_offsets)
      for (int i = layer_wait_offsets[l]; i < layer_wait_offsets[l + 1]; ++i)
        KVX_CUDA_TRY(cudaStreamWaitEvent(st, static_cast<cudaEvent_t>(layer_waits[i]), 0), "kvx_model: layer wait");
    kvx::rope_and_token<<<batch, 1024, 0, st>>>(m->qkv, d_sessions, d_ctx_lens, l, Hq, H, D, layout->block_tokens,
                                               c.rope_theta, fill_seed, fill_mode, m->q, new_k, new_v);
    KVX_CUDA_TRY(cudaGetLastError(), "kvx_model: rope");
    kvx::note_launch();
    const uint32_t* tab = d_tables + static_cast<uint64_t>(l) * batch * max_blocks;
    if (int rc = kvx_decode_attention_append(pool, layout, &ap, tab, d_ctx_lens, m->q, new_k, new_v, m->attn_f32,
                                             batch, max_ctx, m->attn_ws, m->attn_ws_bytes, stream))
      return rc;
    const uint64_t n = static_cast<uint64_t>(batch) * Hq * D;
    kvx::f32_to_bf16_rows<<<kvx::grid_for(n, 256), 256, 0, st>>>(m->attn_f32, m->attn, n);
    KVX_CUDA_TRY(cudaGetLastError(), "kvx_model: attn to bf16");
    kvx::note_launch();
    if (int rc = kvx::layer_post(m, l, batch)) return rc;
  }
  return kvx::sample(m, 0, batch, d_tokens_out);
}

}  // namespace
}  // namespace kvx

extern "C" {

int kvx_model_linear(kvx_model* m, const void* d_x, const void* d_w, void* d_y, int32_t rows, int32_t in,
                     int32_t out, int32_t accumulate, void* stream) {
  if (!m || !d_x || !d_w || !d_y) return kvx::fail_arg("kvx_model_linear: null argument");
  if (rows <= 0 || in <= 0 || out <= 0) return kvx::fail_arg("kvx_model_linear: empty shape");
  kvx::DeviceGuard guard(m->device);
  if (int rc = kvx::bind(m, stream)) return rc;
  return kvx::linear(m, static_cast<const uint16_t*>(d_x), static_cast<const uint16_t*>(d_w),
                     static_cast<uint16_t*>(d_y), rows, in, out, accumulate != 0);
}

int kvx_model_prefill(kvx_model* m, int32_t tokens, void* stream) {
  if (!m) return kvx::fail_arg("kvx_model_prefill: null model");
  if (tokens <= 0) return KVX_OK;
  const kvx_model_config& c = m->cfg;
  kvx::DeviceGuard guard(m->device);
  constexpr int kChunk = 4096;  // rows per pass (activation memory bound)
  if (int rc = kvx::ensure_rows(m, std::min(tokens, kChunk))) return rc;
  if (int rc = kvx::bind(m, stream)) return rc;
  cudaStream_t st = kvx::as_stream(stream);
  for (int done = 0; done < tokens; done += kChunk) {
    const int rows = std::min(kChunk, tokens - done);
    // Token ids: any; the projections' cost does not depend on them.
    KVX_CUDA_TRY(cudaMemsetAsync(m->tokens, 0, static_cast<size_t>(rows) * 4, st), "kvx_model: prefill tokens");
    kvx::embed_rows<<<rows, 128, 0, st>>>(m->embed, m->tokens, m->x, c.hidden, c.vocab);
    KVX_CUDA_TRY(cudaGetLastError(), "kvx_model: embed");
    kvx::note_launch();
  kvx::note_launch();
    for (int l = 0; l < c.num_layers; ++l) {
      if (int rc = kvx::layer_pre(m, l, rows)) return rc;
      // Prefill attention is not modelled here (its K/V land in the pages as
      // the store's Created fill); the attention output is the q projection.
      const uint64_t n = static_cast<uint64_t>(rows) * c.num_q_heads * c.head_dim;
      KVX_CUDA_TRY(cudaMemcpy2DAsync(m->attn, static_cast<size_t>(c.num_q_heads) * c.head_dim * 2, m->qkv,
                                     static_cast<size_t>(c.num_q_heads + 2 * c.num_kv_heads) * c.head_dim * 2,
                                     static_cast<size_t>(c.num_q_heads) * c.head_dim * 2, rows,
                                     cudaMemcpyDeviceToDevice, st),
                   "kvx_model: prefill attn stand-in");
      (void)n;
      if (int rc = kvx::layer_post(m, l, rows)) return rc;
    }
    // The prompt's last token is sampled (its LM head row is real work).
    if (done + rows == tokens)
      if (int rc = kvx::sample(m, rows - 1, 1, m->tokens)) return rc;
  }
  return KVX_OK;
}

}  // extern "C"
