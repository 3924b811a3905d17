// K1 pack, K2 unpack, K3 page copy (migration), K5 fill / append — sm_100a.
//
// All three movers are one gather/scatter over (page, chunk) work items:
//   pack    src pages by id      -> dst contiguous   (reference SwapOut /
//           HostCopy source side, kvstore.cpp:230-269, 691-706; migration
//           send side, kvstore.cpp:753-769)
//   unpack  src contiguous       -> dst pages by id  (LoadH2D / NetArrive
//           landing, kvstore.cpp:522-533, 599-611, 914-923)
//   copy    src pages by id      -> dst pages by id  (fused pack+send+unpack;
//           dst may be a peer GPU's pool over NVLink or a mapped host pool)
// The work is pure HBM traffic (2 bytes moved per payload byte), so the
// kernels are built for bandwidth: 16-byte vectors, several loads in flight
// per thread before any store, grid sized to the SM count, or — the TMA
// variant — one issuing thread per SM driving cp.async.bulk through a ring of
// shared-memory stages (no register staging at all).

#include <algorithm>
#include <atomic>
#include <mutex>
#include <cstdlib>
#include <cstring>
#include <vector>

#include "kvx_common.cuh"

namespace kvx {
namespace {

constexpr int kVecThreads = 256;
constexpr int kVecUnroll = 4;
constexpr uint32_t kVecChunk = kVecThreads * kVecUnroll * 16;  // 16 KiB per work item

// TMA mover geometry per access pattern, measured on B200 (1 GiB session of
// 16,384 scattered 64 KiB pages, profiles/r01_mover_geometry_sweep.txt):
//   gather, contiguous destination (pack):      32 KiB x 4 stages, 1 CTA/SM
//     -> 6.60 TB/s (16 KiB x 6 x 2: 6.57)
//   contiguous source, scatter (unpack):        16 KiB x 6 stages, 2 CTAs/SM
//     -> 6.60 TB/s (32 KiB x 4 x 1: 6.49)
//   gather AND scatter (page -> page copy):     16 KiB x 6 stages, 2 CTAs/SM
//     -> 6.41-6.42 TB/s (64 KiB x 3 x 1: 6.09-6.25; 32 KiB x 4 x 1: 6.27)
// Two CTAs per SM give each SM two independent issue loops (more chunks in
// flight) where a scattered destination makes each store's completion slower.
// KVX_BULK_CHUNK / KVX_BULK_STAGES / KVX_BULK_CTAS_PER_SM override all (sweeps).
constexpr int kBulkMaxStages = 16;
struct BulkGeometry {
  uint32_t chunk;
  int stages;
  int ctas_per_sm;
};

BulkGeometry bulk_geometry(bool src_scattered, bool dst_scattered) {
  BulkGeometry b = (src_scattered && !dst_scattered) ? BulkGeometry{32768, 4, 1} : BulkGeometry{16384, 6, 2};
  if (const char* e = std::getenv("KVX_BULK_CHUNK")) b.chunk = static_cast<uint32_t>(std::atoi(e));
  if (const char* e = std::getenv("KVX_BULK_STAGES")) b.stages = std::atoi(e);
  if (const char* e = std::getenv("KVX_BULK_CTAS_PER_SM")) b.ctas_per_sm = std::atoi(e);
  b.chunk = std::max<uint32_t>(1024, std::min<uint32_t>(b.chunk, 65536)) & ~15u;
  b.stages = std::max(2, std::min(b.stages, kBulkMaxStages));
  b.ctas_per_sm = std::max(1, std::min(b.ctas_per_sm, 8));
  return b;
}

struct MoveArgs {
  const uint8_t* src;
  const uint32_t* src_ids;  // null: contiguous
  uint8_t* dst;
  const uint32_t* dst_ids;  // null: contiguous
  uint64_t n_pages;
  uint64_t page_bytes;
  uint32_t chunk_bytes;
  uint32_t chunks_per_page;
  int stages;  // TMA ring depth (bulk mover only)
  uint64_t src_pages, dst_pages;  // pool sizes: page ids are checked against them
};

__device__ __forceinline__ void item_addr(const MoveArgs& a, uint64_t item, const uint8_t*& s, uint8_t*& d,
                                          uint32_t& bytes) {
  const uint64_t page = item / a.chunks_per_page;
  const uint32_t c = static_cast<uint32_t>(item - page * a.chunks_per_page);
  const uint64_t sp = a.src_ids ? __ldg(a.src_ids + page) : page;
  const uint64_t dp = a.dst_ids ? __ldg(a.dst_ids + page) : page;
  if ((a.src_ids && sp >= a.src_pages) || (a.dst_ids && dp >= a.dst_pages)) __trap();  // bad id: fail loudly
  const uint64_t off = static_cast<uint64_t>(c) * a.chunk_bytes;
  s = a.src + sp * a.page_bytes + off;
  d = a.dst + dp * a.page_bytes + off;
  const uint64_t left = a.page_bytes - off;
  bytes = static_cast<uint32_t>(left < a.chunk_bytes ? left : a.chunk_bytes);
}

// LDG.128 / STG.128: every thread issues kVecUnroll independent loads before
// its stores, so one 256-thread CTA keeps 16 KiB in flight.
// The movers can be launched with programmatic dependent launch (launch_pdl,
// KVX_MOVER_PDL=1): the next kernel in the stream may then be scheduled as
// soon as this grid starts (it waits in griddepcontrol.wait for our
// completion before touching memory), and this grid's wait covers whatever
// wrote our sources. Without the attribute both instructions are no-ops.
__device__ __forceinline__ void pdl_enter() {
  asm volatile("griddepcontrol.wait;" ::: "memory");
  asm volatile("griddepcontrol.launch_dependents;" ::: "memory");
}

__global__ void __launch_bounds__(kVecThreads) page_move_vec(MoveArgs a) {
  pdl_enter();
  const uint64_t items = a.n_pages * a.chunks_per_page;
  for (uint64_t item = blockIdx.x; item < items; item += gridDim.x) {
    const uint8_t* s8;
    uint8_t* d8;
    uint32_t bytes;
    item_addr(a, item, s8, d8, bytes);
    const int4* s = reinterpret_cast<const int4*>(s8);
    int4* d = reinterpret_cast<int4*>(d8);
    const uint32_t vecs = bytes / 16;
    if (vecs == kVecThreads * kVecUnroll) {
      int4 r[kVecUnroll];
#pragma unroll
      for (int u = 0; u < kVecUnroll; ++u) r[u] = ld_stream(s + threadIdx.x + u * kVecThreads);
#pragma unroll
      for (int u = 0; u < kVecUnroll; ++u) st_stream(d + threadIdx.x + u * kVecThreads, r[u]);
    } else {
      for (uint32_t v = threadIdx.x; v < vecs; v += kVecThreads) st_stream(d + v, ld_stream(s + v));
    }
  }
}

// Host-listed moves: the id pairs travel in the kernel's parameter block
// (no upload, no device id array): used where the ids come from the host
// per move (the payload's lanes), so a move costs one launch call.
// A launch copies its whole parameter block, so the id arrays come in three
// capacities (2 KiB / 8 KiB / 30 KiB of ids) and a move uses the smallest
// that holds it; 3,840 pairs + header stay under the 32,764-B limit.
constexpr int kListedPairs = 3840;
template <int CAP>
struct ListedBulkArgs {
  const uint8_t* src;
  uint8_t* dst;
  uint64_t n_pages;
  uint64_t page_bytes;
  uint32_t chunk_bytes;
  uint32_t chunks_per_page;
  int stages;
  uint32_t src_ids[CAP];
  uint32_t dst_ids[CAP];
};
template <int CAP>
__device__ __forceinline__ void item_addr(const ListedBulkArgs<CAP>& a, uint64_t item, const uint8_t*& s, uint8_t*& d,
                                          uint32_t& bytes) {
  const uint64_t page = item / a.chunks_per_page;
  const uint32_t c = static_cast<uint32_t>(item - page * a.chunks_per_page);
  const uint64_t off = static_cast<uint64_t>(c) * a.chunk_bytes;
  s = a.src + static_cast<uint64_t>(a.src_ids[page]) * a.page_bytes + off;  // ids range-checked on the host
  d = a.dst + static_cast<uint64_t>(a.dst_ids[page]) * a.page_bytes + off;
  const uint64_t left = a.page_bytes - off;
  bytes = static_cast<uint32_t>(left < a.chunk_bytes ? left : a.chunk_bytes);
}

// TMA bulk variant: lane 0 of a single warp per SM streams chunks through a
// a.stages-deep shared-memory ring. Load k+S-1 is issued as soon as the
// bulk store of chunk k-1 has finished READING its stage.
template <typename Args>
__device__ __forceinline__ void bulk_body(const Args& a) {
  extern __shared__ __align__(128) uint8_t ring[];
  __shared__ __align__(8) uint64_t full[kBulkMaxStages];
  const int S = a.stages;
  const uint32_t slot = a.chunk_bytes;
  if (threadIdx.x != 0) return;
  const uint64_t items = a.n_pages * a.chunks_per_page;
  if (blockIdx.x >= items) return;
  const uint64_t mine = (items - blockIdx.x + gridDim.x - 1) / gridDim.x;
  for (int s = 0; s < S; ++s) mbar_init(&full[s], 1);
  asm volatile("fence.mbarrier_init.release.cluster;\n\tfence.proxy.async.shared::cta;" ::: "memory");

  auto load = [&](uint64_t k) {
    const uint8_t* s;
    uint8_t* d;
    uint32_t bytes;
    item_addr(a, blockIdx.x + k * gridDim.x, s, d, bytes);
    const int st = static_cast<int>(k % S);
    mbar_arrive_expect_tx(&full[st], bytes);
    bulk_g2s(ring + st * slot, s, bytes, &full[st]);
  };
  const uint64_t prologue = mine < static_cast<uint64_t>(S) ? mine : S;
  for (uint64_t k = 0; k < prologue; ++k) load(k);
  for (uint64_t k = 0; k < mine; ++k) {
    const int st = static_cast<int>(k % S);
    mbar_wait(&full[st], static_cast<uint32_t>((k / S) & 1));
    const uint8_t* s;
    uint8_t* d;
    uint32_t bytes;
    item_addr(a, blockIdx.x + k * gridDim.x, s, d, bytes);
    bulk_s2g(d, ring + st * slot, bytes);
    bulk_commit();
    if (k >= 1 && k - 1 + S < mine) {
      bulk_wait_read<1>();  // store k-1 has drained its stage
      load(k - 1 + S);
    }
  }
  bulk_wait<0>();
}

__global__ void __launch_bounds__(32, 1) page_move_bulk(MoveArgs a) {
  pdl_enter();
  bulk_body(a);
}

template <int CAP>
__global__ void __launch_bounds__(32, 1) page_move_bulk_listed(const __grid_constant__ ListedBulkArgs<CAP> a) {
  bulk_body(a);
}

// Launch with programmatic stream serialization (PDL).
template <typename Kernel>
void launch_pdl(Kernel kernel, unsigned grid, unsigned block, uint32_t smem, cudaStream_t stream, const MoveArgs& a) {
  cudaLaunchConfig_t cfg{};
  cfg.gridDim = dim3(grid);
  cfg.blockDim = dim3(block);
  cfg.dynamicSmemBytes = smem;
  cfg.stream = stream;
  cudaLaunchAttribute attr[1];
  attr[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
  // Off by default: an early-resident successor mover holds its SM's shared
  // memory while it waits, which delays decode kernels running beside a
  // migration (event-gated decode of a migrating session: 577-596 -> 718 us)
  // for a 3% gain on back-to-back moves alone. KVX_MOVER_PDL=1 turns it on.
  static const char* env = std::getenv("KVX_MOVER_PDL");
  attr[0].val.programmaticStreamSerializationAllowed = (env && env[0] == '1') ? 1 : 0;
  cfg.attrs = attr;
  cfg.numAttrs = 1;
  cudaLaunchKernelEx(&cfg, kernel, a);
  note_launch();
}

// AUTO picks the TMA bulk mover when both sides are in this GPU's HBM (measured
// faster: ~95% vs ~88% of the copy roofline, profiles/), and the SM vector
// mover for peer (NVLink) or mapped-host (PCIe) endpoints.
int launch_move(MoveArgs a, int mode, int device, cudaStream_t stream, const char* who, bool tma_ok,
                uint32_t max_ctas = 0) {
  if (a.n_pages == 0) return KVX_OK;
  DeviceGuard guard(device);
  if (a.page_bytes % 16 != 0 || reinterpret_cast<uintptr_t>(a.src) % 16 || reinterpret_cast<uintptr_t>(a.dst) % 16)
    return fail_arg("page movers need 16-byte aligned pages");
  const int sms = sm_count(device);
  if (mode == KVX_COPY_AUTO) mode = tma_ok ? KVX_COPY_TMA : KVX_COPY_SM;
  if (mode == KVX_COPY_TMA) {
    const BulkGeometry geo = bulk_geometry(a.src_ids != nullptr, a.dst_ids != nullptr);
    a.chunk_bytes = static_cast<uint32_t>(std::min<uint64_t>(a.page_bytes, geo.chunk));
    a.chunks_per_page = static_cast<uint32_t>((a.page_bytes + a.chunk_bytes - 1) / a.chunk_bytes);
    a.stages = geo.stages;
    const uint32_t smem = static_cast<uint32_t>(geo.stages) * a.chunk_bytes;
    // Largest dynamic smem configured so far per device; raised under a
    // mutex so a smaller request can never lower the attribute after a
    // larger one was recorded.
    static std::atomic<uint32_t> configured[64] = {};
    static std::mutex mu;
    std::atomic<uint32_t>& have = configured[(device < 0 ? 0 : device) % 64];
    if (have.load(std::memory_order_acquire) < smem) {
      std::lock_guard<std::mutex> lock(mu);
      if (have.load(std::memory_order_relaxed) < smem) {
        KVX_CUDA_TRY(cudaFuncSetAttribute(page_move_bulk, cudaFuncAttributeMaxDynamicSharedMemorySize, smem), who);
        have.store(smem, std::memory_order_release);
      }
    }
    const uint64_t items = a.n_pages * a.chunks_per_page;
    unsigned grid =
        static_cast<unsigned>(std::min<uint64_t>(items, static_cast<uint64_t>(sms) * geo.ctas_per_sm));
    if (max_ctas && grid > max_ctas) grid = max_ctas;
    launch_pdl(page_move_bulk, grid, 32, smem, stream, a);
  } else if (mode == KVX_COPY_SM) {
    a.chunk_bytes = kVecChunk;
    a.chunks_per_page = static_cast<uint32_t>((a.page_bytes + kVecChunk - 1) / kVecChunk);
    const uint64_t items = a.n_pages * a.chunks_per_page;
    unsigned grid = static_cast<unsigned>(std::min<uint64_t>(items, static_cast<uint64_t>(sms) * 8));
    if (max_ctas && grid > max_ctas) grid = max_ctas;
    launch_pdl(page_move_vec, grid, kVecThreads, 0, stream, a);
  } else {
    set_error(std::string(who) + ": unsupported copy mode");
    return KVX_ERR_UNSUPPORTED;
  }
  KVX_CUDA_TRY(cudaGetLastError(), who);
  return KVX_OK;
}

// Host-listed page moves (KVX_COPY_CE with fragmented id runs): the id
// pairs travel in the launch's parameter block (no upload, no device id
// array), and a few CTAs of the LDG/STG.128 mover stream the pages. Used for
// PCIe moves between HBM and a pinned, mapped HOST pool when the pages do not
// form long runs: per run a copy-engine submission costs microseconds of
// launch overhead, a 64 KiB page only ~1.2 us of PCIe time. Measured on B200
// (profiles/r01_pcie_movers.json.txt): SM zero-copy moves 51-53 GB/s per
// direction, fragmented or not, against 55-57 for copy engines on long runs.
template <int CAP>
struct ListedMove {
  const uint8_t* src;
  uint8_t* dst;
  uint64_t page_bytes;
  uint32_t n;
  uint32_t chunks_per_page;
  uint32_t src_ids[CAP];
  uint32_t dst_ids[CAP];
};

template <int CAP>
__global__ void __launch_bounds__(kVecThreads) page_move_listed(const __grid_constant__ ListedMove<CAP> a) {
  const uint64_t items = static_cast<uint64_t>(a.n) * a.chunks_per_page;
  for (uint64_t item = blockIdx.x; item < items; item += gridDim.x) {
    const uint32_t i = static_cast<uint32_t>(item / a.chunks_per_page);
    const uint64_t off = (item - static_cast<uint64_t>(i) * a.chunks_per_page) * kVecChunk;
    const int4* s = reinterpret_cast<const int4*>(a.src + static_cast<uint64_t>(a.src_ids[i]) * a.page_bytes + off);
    int4* d = reinterpret_cast<int4*>(a.dst + static_cast<uint64_t>(a.dst_ids[i]) * a.page_bytes + off);
    const uint64_t left = a.page_bytes - off;
    const uint32_t vecs = static_cast<uint32_t>((left < kVecChunk ? left : kVecChunk) / 16);
    if (vecs == kVecThreads * kVecUnroll) {
      int4 r[kVecUnroll];
#pragma unroll
      for (int u = 0; u < kVecUnroll; ++u) r[u] = ld_stream(s + threadIdx.x + u * kVecThreads);
#pragma unroll
      for (int u = 0; u < kVecUnroll; ++u) st_stream(d + threadIdx.x + u * kVecThreads, r[u]);
    } else {
      for (uint32_t v = threadIdx.x; v < vecs; v += kVecThreads) st_stream(d + v, ld_stream(s + v));
    }
  }
}

// ---- K5: contents -----------------------------------------------------------

// 16-byte vector v of a page whose tag hashes to h (K5 content).
__device__ __forceinline__ uint4 fill_vec(uint64_t h, uint32_t v, int mode, int dtype) {
  if (mode == KVX_FILL_BITS) {
    const uint64_t w0 = splitmix64(h + 2ull * v), w1 = splitmix64(h + 2ull * v + 1);
    return make_uint4(static_cast<uint32_t>(w0), static_cast<uint32_t>(w0 >> 32), static_cast<uint32_t>(w1),
                      static_cast<uint32_t>(w1 >> 32));
  }
  uint32_t w[4];
  if (dtype == KVX_DTYPE_F32) {
#pragma unroll
    for (int e = 0; e < 4; ++e) w[e] = __float_as_uint(unit_value(splitmix64(h + 4ull * v + e)));
  } else {
#pragma unroll
    for (int e = 0; e < 4; ++e) {
      const uint32_t lo = f32_to_bf16_rne(unit_value(splitmix64(h + 8ull * v + 2 * e)));
      const uint32_t hi = f32_to_bf16_rne(unit_value(splitmix64(h + 8ull * v + 2 * e + 1)));
      w[e] = lo | (hi << 16);
    }
  }
  return make_uint4(w[0], w[1], w[2], w[3]);
}

__global__ void __launch_bounds__(256) fill_pages_kernel(uint8_t* base, uint64_t page_bytes, const uint32_t* ids,
                                                         const kvx_block_tag* tags, uint64_t n, uint64_t seed,
                                                         int mode, int dtype) {
  const uint32_t vecs = static_cast<uint32_t>(page_bytes / 16);
  for (uint64_t i = blockIdx.x; i < n; i += gridDim.x) {
    const kvx_block_tag t = tags[i];
    const uint64_t h = block_base(seed, t.session, t.layer, t.block);
    uint4* page = reinterpret_cast<uint4*>(base + static_cast<uint64_t>(ids[i]) * page_bytes);
    for (uint32_t v = threadIdx.x; v < vecs; v += blockDim.x) page[v] = fill_vec(h, v, mode, dtype);
  }
}

// Scrub: pages whose bytes differ from the K5 content of their tag. Tags
// come from a list, or from block-table coordinates (layer, request, block)
// when `tags` is null (tables [layers][batch][max_blocks], sessions[batch],
// ctx_lens[batch]: blocks beyond a request's context are skipped).
__global__ void __launch_bounds__(256) verify_pages_kernel(const uint8_t* base, uint64_t page_bytes, uint64_t pool_pages,
                                                           const uint32_t* ids, const kvx_block_tag* tags, uint64_t n,
                                                           const int32_t* sessions, const int32_t* ctx_lens,
                                                           int batch, int max_blocks, int block_tokens, uint64_t seed,
                                                           int mode, int dtype, unsigned long long* mismatches) {
  const uint32_t vecs = static_cast<uint32_t>(page_bytes / 16);
  __shared__ int bad;
  for (uint64_t i = blockIdx.x; i < n; i += gridDim.x) {
    kvx_block_tag t;
    if (tags) {
      t = tags[i];
    } else {
      const uint64_t per_layer = static_cast<uint64_t>(batch) * max_blocks;
      const uint32_t layer = static_cast<uint32_t>(i / per_layer);
      const uint64_t rem = i - layer * per_layer;
      const int b = static_cast<int>(rem / max_blocks), blk = static_cast<int>(rem - static_cast<uint64_t>(b) * max_blocks);
      if (blk * block_tokens >= ctx_lens[b]) continue;  // past this request's context (block-uniform)
      t = kvx_block_tag{static_cast<uint32_t>(sessions[b]), layer, static_cast<uint32_t>(blk)};
    }
    const uint32_t id = ids[i];
    if (threadIdx.x == 0) bad = 0;
    __syncthreads();
    if (id >= pool_pages) {
      if (threadIdx.x == 0) bad = 1;
    } else {
      const uint64_t h = block_base(seed, t.session, t.layer, t.block);
      const uint4* page = reinterpret_cast<const uint4*>(base + static_cast<uint64_t>(id) * page_bytes);
      int mine = 0;
      for (uint32_t v = threadIdx.x; v < vecs; v += blockDim.x) {
        const uint4 want = fill_vec(h, v, mode, dtype), got = page[v];
        mine |= (want.x != got.x) | (want.y != got.y) | (want.z != got.z) | (want.w != got.w);
      }
      if (mine) bad = 1;
    }
    __syncthreads();
    if (threadIdx.x == 0 && bad) atomicAdd(mismatches, 1ull);
    __syncthreads();
  }
}

// One CTA per appended token: K and V of every kv head into the page slot.
__global__ void __launch_bounds__(128) append_kv_kernel(uint8_t* base, uint64_t page_bytes, const uint32_t* ids,
                                                        const int32_t* slots, const uint8_t* k, const uint8_t* v,
                                                        int heads, int tokens, int row_bytes) {
  pdl_enter();  // the attention launched next may prefetch every page but this step's
  const uint64_t i = blockIdx.x;
  uint8_t* page = base + static_cast<uint64_t>(ids[i]) * page_bytes;
  const int slot = slots[i];
  const int row_vecs = row_bytes / 16;
  const int total = 2 * heads * row_vecs;
  for (int e = threadIdx.x; e < total; e += blockDim.x) {
    const int kv = e / (heads * row_vecs);
    const int rem = e - kv * heads * row_vecs;
    const int h = rem / row_vecs, c = rem - h * row_vecs;
    const uint8_t* src = (kv ? v : k) + (i * heads + h) * static_cast<uint64_t>(row_bytes);
    uint8_t* dst = page + (static_cast<uint64_t>(kv * heads + h) * tokens + slot) * row_bytes;
    reinterpret_cast<uint4*>(dst)[c] = reinterpret_cast<const uint4*>(src)[c];
  }
}

}  // namespace
}  // namespace kvx

using kvx::MoveArgs;

namespace kvx {
namespace {
// Host-listed move (ids already range-checked by the caller): chunks of
// kListedPairs pages, ids copied into each launch's parameter block. TMA
// bulk mover for HBM<->HBM on one device, the LDG/STG.128 mover otherwise
// (peer, mapped host) or when asked (mode KVX_COPY_SM); `max_ctas` bounds
// the grid (0: the mover's default).
template <int CAP>
int launch_listed_chunk(const kvx_pool* src, const uint32_t* src_ids, const kvx_pool* dst, const uint32_t* dst_ids,
                        uint32_t n, bool tma, int dev, int sms, uint32_t max_ctas, cudaStream_t st, const char* who) {
  if (tma) {
    static thread_local ListedBulkArgs<CAP> b;
    const BulkGeometry geo = bulk_geometry(true, true);
    b.src = src->base;
    b.dst = dst->base;
    b.page_bytes = src->page_bytes;
    b.chunk_bytes = static_cast<uint32_t>(std::min<uint64_t>(src->page_bytes, geo.chunk));
    b.chunks_per_page = static_cast<uint32_t>((src->page_bytes + b.chunk_bytes - 1) / b.chunk_bytes);
    b.stages = geo.stages;
    const uint32_t smem = static_cast<uint32_t>(geo.stages) * b.chunk_bytes;
    static std::atomic<uint32_t> configured[64] = {};
    std::atomic<uint32_t>& have = configured[(dev < 0 ? 0 : dev) % 64];
    if (have.load(std::memory_order_acquire) < smem) {
      static std::mutex mu;
      std::lock_guard<std::mutex> lock(mu);
      if (have.load(std::memory_order_relaxed) < smem) {
        KVX_CUDA_TRY(
            cudaFuncSetAttribute(page_move_bulk_listed<CAP>, cudaFuncAttributeMaxDynamicSharedMemorySize, smem), who);
        have.store(smem, std::memory_order_release);
      }
    }
    b.n_pages = n;
    std::memcpy(b.src_ids, src_ids, n * sizeof(uint32_t));
    std::memcpy(b.dst_ids, dst_ids, n * sizeof(uint32_t));
    const uint64_t items = b.n_pages * b.chunks_per_page;
    unsigned grid = static_cast<unsigned>(std::min<uint64_t>(items, static_cast<uint64_t>(sms) * geo.ctas_per_sm));
    if (max_ctas && grid > max_ctas) grid = max_ctas;
    page_move_bulk_listed<CAP><<<grid, 32, smem, st>>>(b);
  } else {
    static thread_local ListedMove<CAP> m;
    m.src = src->base;
    m.dst = dst->base;
    m.page_bytes = src->page_bytes;
    m.chunks_per_page = static_cast<uint32_t>((src->page_bytes + kVecChunk - 1) / kVecChunk);
    m.n = n;
    std::memcpy(m.src_ids, src_ids, n * sizeof(uint32_t));
    std::memcpy(m.dst_ids, dst_ids, n * sizeof(uint32_t));
    const uint64_t items = static_cast<uint64_t>(m.n) * m.chunks_per_page;
    unsigned grid = static_cast<unsigned>(std::min<uint64_t>(items, static_cast<uint64_t>(sms) * 8));
    if (max_ctas && grid > max_ctas) grid = max_ctas;
    page_move_listed<CAP><<<grid, kVecThreads, 0, st>>>(m);
  }
  note_launch();
  KVX_CUDA_TRY(cudaGetLastError(), who);
  return KVX_OK;
}

int launch_listed(const kvx_pool* src, const uint32_t* src_ids, const kvx_pool* dst, const uint32_t* dst_ids,
                  uint64_t n, int mode, uint32_t max_ctas, cudaStream_t st, const char* who) {
  const int dev = src->device >= 0 ? src->device : dst->device;
  DeviceGuard guard(dev);
  if (src->page_bytes % 16 || reinterpret_cast<uintptr_t>(src->base) % 16 || reinterpret_cast<uintptr_t>(dst->base) % 16)
    return fail_arg("page movers need 16-byte aligned pages");
  const bool local = !src->host && !dst->host && !src->ipc && !dst->ipc && src->device == dst->device;
  const int sms = sm_count(dev);
  if (mode == KVX_COPY_AUTO) mode = local ? KVX_COPY_TMA : KVX_COPY_SM;
  if (mode != KVX_COPY_TMA && mode != KVX_COPY_SM) {
    set_error(std::string(who) + ": unsupported copy mode");
    return KVX_ERR_UNSUPPORTED;
  }
  const bool tma = mode == KVX_COPY_TMA;
  for (uint64_t at = 0; at < n; at += kListedPairs) {
    const uint32_t k = static_cast<uint32_t>(std::min<uint64_t>(kListedPairs, n - at));
    const int rc = k <= 256    ? launch_listed_chunk<256>(src, src_ids + at, dst, dst_ids + at, k, tma, dev, sms,
                                                          max_ctas, st, who)
                   : k <= 1024 ? launch_listed_chunk<1024>(src, src_ids + at, dst, dst_ids + at, k, tma, dev, sms,
                                                           max_ctas, st, who)
                               : launch_listed_chunk<kListedPairs>(src, src_ids + at, dst, dst_ids + at, k, tma, dev,
                                                                   sms, max_ctas, st, who);
    if (rc) return rc;
  }
  return KVX_OK;
}
}  // namespace
}  // namespace kvx

extern "C" {

int kvx_pack(const kvx_pool* src, const uint32_t* d_page_ids, uint64_t n, void* d_dst, int mode, void* stream) {
  if (!src || (n && (!d_page_ids || !d_dst))) return kvx::fail_arg("kvx_pack: null argument");
  if (src->fd >= 0) return kvx::fail_arg("kvx_pack: file pools move through kvx_copy_pages(KVX_COPY_CE)");
  MoveArgs a{src->base, d_page_ids, static_cast<uint8_t*>(d_dst), nullptr, n, src->page_bytes, 0, 0, 0,
             src->num_pages, 0};
  return kvx::launch_move(a, mode, src->device, kvx::as_stream(stream), "kvx_pack", !src->host && !src->ipc);
}

int kvx_unpack(kvx_pool* dst, const uint32_t* d_page_ids, uint64_t n, const void* d_src, int mode, void* stream) {
  if (!dst || (n && (!d_page_ids || !d_src))) return kvx::fail_arg("kvx_unpack: null argument");
  if (dst->fd >= 0) return kvx::fail_arg("kvx_unpack: file pools move through kvx_copy_pages(KVX_COPY_CE)");
  MoveArgs a{static_cast<const uint8_t*>(d_src), nullptr, dst->base, d_page_ids, n, dst->page_bytes, 0, 0, 0,
             0, dst->num_pages};
  return kvx::launch_move(a, mode, dst->device, kvx::as_stream(stream), "kvx_unpack", !dst->host && !dst->ipc);
}

int kvx_copy_pages(const kvx_pool* src, const uint32_t* src_ids, kvx_pool* dst, const uint32_t* dst_ids,
                   uint64_t n, int mode, void* stream) {
  return kvx_copy_pages_capped(src, src_ids, dst, dst_ids, n, mode, 0, stream);
}

int kvx_copy_pages_capped(const kvx_pool* src, const uint32_t* src_ids, kvx_pool* dst, const uint32_t* dst_ids,
                          uint64_t n, int mode, uint32_t max_ctas, void* stream) {
  if (!src || !dst || (n && (!src_ids || !dst_ids))) return kvx::fail_arg("kvx_copy_pages: null argument");
  if (src->page_bytes != dst->page_bytes) return kvx::fail_arg("kvx_copy_pages: page size mismatch");
  if (n == 0) return KVX_OK;
  const cudaStream_t st = kvx::as_stream(stream);
  if (src->fd >= 0 || dst->fd >= 0) {
    // DISK tier: file pool <-> pinned HOST pool, runs of consecutive ids as
    // single preads / pwrites, executed in stream order.
    const kvx_pool* file = src->fd >= 0 ? src : dst;
    const kvx_pool* mem = src->fd >= 0 ? dst : src;
    if (mode != KVX_COPY_CE || mem->fd >= 0 || !mem->host || !mem->base) {
      kvx::set_error("kvx_copy_pages: a file pool exchanges pages only with a HOST pool (KVX_COPY_CE, host ids)");
      return KVX_ERR_UNSUPPORTED;
    }
    const bool write = dst->fd >= 0;
    std::vector<kvx::FileRun> runs;
    for (uint64_t i = 0; i < n;) {
      if (src_ids[i] >= src->num_pages || dst_ids[i] >= dst->num_pages)
        return kvx::fail_arg("kvx_copy_pages: page id out of range");
      uint64_t j = i + 1;
      while (j < n && src_ids[j] == src_ids[j - 1] + 1 && dst_ids[j] == dst_ids[j - 1] + 1) ++j;
      const uint32_t mem_id = write ? src_ids[i] : dst_ids[i];
      const uint32_t file_id = write ? dst_ids[i] : src_ids[i];
      runs.push_back(kvx::FileRun{mem->base + static_cast<uint64_t>(mem_id) * mem->page_bytes,
                                  static_cast<uint64_t>(file_id) * file->page_bytes, (j - i) * file->page_bytes});
      i = j;
    }
    return kvx::enqueue_file_io(const_cast<kvx_pool*>(file), std::move(runs), write, st, "kvx_copy_pages(file)");
  }
  if (mode != KVX_COPY_CE) {
    MoveArgs a{src->base, src_ids, dst->base, dst_ids, n, src->page_bytes, 0, 0, 0, src->num_pages, dst->num_pages};
    const int dev = src->device >= 0 ? src->device : dst->device;
    const bool local = !src->host && !dst->host && !src->ipc && !dst->ipc && src->device == dst->device;
    return kvx::launch_move(a, mode, dev, st, "kvx_copy_pages", local, max_ctas);
  }
  // Host id lists: copy engines, one cudaMemcpyAsync per run of consecutive
  // ids, when the pages form long runs (the payload deals new pages in
  // ascending order); otherwise the listed-id SM mover, ids in the launch
  // parameters. Graph capture records one memcpy node per run / one kernel
  // node per chunk of kListedPairs pages.
  uint64_t runs = 0;
  for (uint64_t i = 0; i < n; ++i) {
    if (src_ids[i] >= src->num_pages || dst_ids[i] >= dst->num_pages)
      return kvx::fail_arg("kvx_copy_pages: page id out of range");
    runs += i == 0 || src_ids[i] != src_ids[i - 1] + 1 || dst_ids[i] != dst_ids[i - 1] + 1;
  }
  const uint64_t run_bytes = n * src->page_bytes / runs;
  static const uint64_t min_run = [] {
    const char* e = std::getenv("KVX_CE_MIN_RUN_BYTES");
    return e ? std::strtoull(e, nullptr, 10) : (uint64_t{1} << 20);
  }();
  // Every pool is device-addressable here: HBM, IPC-opened peer HBM, or
  // pinned host memory allocated mapped (UVA: host pointer == device pointer).
  if (run_bytes < min_run && src->page_bytes % 16 == 0 && (src->device >= 0 || dst->device >= 0)) {
    static const unsigned ctas = [] {
      const char* e = std::getenv("KVX_LISTED_CTAS");
      return e ? static_cast<unsigned>(std::atoi(e)) : 64u;
    }();
    return kvx::launch_listed(src, src_ids, dst, dst_ids, n, KVX_COPY_SM, ctas, st, "kvx_copy_pages(listed)");
  }
  for (uint64_t i = 0; i < n;) {
    uint64_t j = i + 1;
    while (j < n && src_ids[j] == src_ids[j - 1] + 1 && dst_ids[j] == dst_ids[j - 1] + 1) ++j;
    KVX_CUDA_TRY(cudaMemcpyAsync(dst->base + static_cast<uint64_t>(dst_ids[i]) * dst->page_bytes,
                                 src->base + static_cast<uint64_t>(src_ids[i]) * src->page_bytes,
                                 (j - i) * src->page_bytes, cudaMemcpyDefault, st),
                 "kvx_copy_pages(CE)");
    i = j;
  }
  return KVX_OK;
}

int kvx_copy_pages_listed(const kvx_pool* src, const uint32_t* src_ids, kvx_pool* dst, const uint32_t* dst_ids,
                          uint64_t n, int mode, uint32_t max_ctas, void* stream) {
  if (!src || !dst || (n && (!src_ids || !dst_ids))) return kvx::fail_arg("kvx_copy_pages_listed: null argument");
  if (src->page_bytes != dst->page_bytes) return kvx::fail_arg("kvx_copy_pages_listed: page size mismatch");
  if (src->fd >= 0 || dst->fd >= 0) return kvx::fail_arg("kvx_copy_pages_listed: not on a file pool");
  if (src->device < 0 && dst->device < 0) return kvx::fail_arg("kvx_copy_pages_listed: needs a device endpoint");
  if (mode != KVX_COPY_AUTO && mode != KVX_COPY_SM && mode != KVX_COPY_TMA)
    return kvx::fail_arg("kvx_copy_pages_listed: mode must be AUTO, SM or TMA");
  for (uint64_t i = 0; i < n; ++i)
    if (src_ids[i] >= src->num_pages || dst_ids[i] >= dst->num_pages)
      return kvx::fail_arg("kvx_copy_pages_listed: page id out of range");
  if (n == 0) return KVX_OK;
  return kvx::launch_listed(src, src_ids, dst, dst_ids, n, mode, max_ctas, kvx::as_stream(stream),
                            "kvx_copy_pages_listed");
}

int kvx_verify_pages(const kvx_pool* pool, const uint32_t* d_page_ids, const kvx_block_tag* d_tags, uint64_t n,
                     uint64_t seed, const kvx_page_layout* layout, int fill_mode, unsigned long long* d_mismatches,
                     void* stream) {
  if (!pool || !d_mismatches || (n && (!d_page_ids || !d_tags))) return kvx::fail_arg("kvx_verify_pages: null argument");
  if (pool->fd >= 0) return kvx::fail_arg("kvx_verify_pages: not on a file pool");
  if (fill_mode != KVX_FILL_BITS && fill_mode != KVX_FILL_VALUES) return kvx::fail_arg("kvx_verify_pages: bad mode");
  if (fill_mode == KVX_FILL_VALUES && (!layout || kvx_page_bytes(layout) != pool->page_bytes))
    return kvx::fail_arg("kvx_verify_pages: layout does not match the pool's page size");
  if (n == 0) return KVX_OK;
  const int dtype = layout ? layout->dtype : KVX_DTYPE_BF16;
  kvx::DeviceGuard guard(pool->device);
  const unsigned grid = static_cast<unsigned>(std::min<uint64_t>(n, 148ull * 8));
  kvx::verify_pages_kernel<<<grid, 256, 0, kvx::as_stream(stream)>>>(pool->base, pool->page_bytes, pool->num_pages,
                                                                       d_page_ids, d_tags, n, nullptr, nullptr, 0, 1,
                                                                       1, seed, fill_mode, dtype, d_mismatches);
  kvx::note_launch();
  KVX_CUDA_TRY(cudaGetLastError(), "kvx_verify_pages");
  return KVX_OK;
}

int kvx_verify_block_tables(const kvx_pool* pool, const kvx_page_layout* layout, const uint32_t* d_tables,
                            const int32_t* d_ctx_lens, const int32_t* d_sessions, int32_t num_layers, int32_t batch,
                            int32_t max_blocks, uint64_t seed, int fill_mode, unsigned long long* d_mismatches,
                            void* stream) {
  if (!pool || !layout || !d_tables || !d_ctx_lens || !d_sessions || !d_mismatches)
    return kvx::fail_arg("kvx_verify_block_tables: null argument");
  if (kvx_page_bytes(layout) != pool->page_bytes) return kvx::fail_arg("kvx_verify_block_tables: layout/page size");
  if (fill_mode != KVX_FILL_BITS && fill_mode != KVX_FILL_VALUES) return kvx::fail_arg("kvx_verify_block_tables: bad mode");
  const uint64_t n = static_cast<uint64_t>(num_layers) * batch * max_blocks;
  if (n == 0) return KVX_OK;
  kvx::DeviceGuard guard(pool->device);
  const unsigned grid = static_cast<unsigned>(std::min<uint64_t>(n, 148ull * 8));
  kvx::verify_pages_kernel<<<grid, 256, 0, kvx::as_stream(stream)>>>(
      pool->base, pool->page_bytes, pool->num_pages, d_tables, nullptr, n, d_sessions, d_ctx_lens, batch, max_blocks,
      layout->block_tokens, seed, fill_mode, layout->dtype, d_mismatches);
  kvx::note_launch();
  KVX_CUDA_TRY(cudaGetLastError(), "kvx_verify_block_tables");
  return KVX_OK;
}

int kvx_fill_pages(kvx_pool* pool, const uint32_t* d_page_ids, const kvx_block_tag* d_tags, uint64_t n, uint64_t seed,
                   const kvx_page_layout* layout, int fill_mode, void* stream) {
  if (!pool || (n && (!d_page_ids || !d_tags))) return kvx::fail_arg("kvx_fill_pages: null argument");
  if (pool->fd >= 0) return kvx::fail_arg("kvx_fill_pages: not on a file pool");
  if (fill_mode != KVX_FILL_BITS && fill_mode != KVX_FILL_VALUES) return kvx::fail_arg("kvx_fill_pages: bad mode");
  const int dtype = layout ? layout->dtype : KVX_DTYPE_BF16;
  if (fill_mode == KVX_FILL_VALUES && (!layout || kvx_page_bytes(layout) != pool->page_bytes))
    return kvx::fail_arg("kvx_fill_pages: layout does not match the pool's page size");
  if (n == 0) return KVX_OK;
  const unsigned grid = static_cast<unsigned>(std::min<uint64_t>(n, kvx::sm_count(pool->device) * 8ull));
  kvx::DeviceGuard guard(pool->device);
  kvx::fill_pages_kernel<<<grid, 256, 0, kvx::as_stream(stream)>>>(pool->base, pool->page_bytes, d_page_ids, d_tags,
                                                                     n, seed, fill_mode, dtype);
  kvx::note_launch();
  KVX_CUDA_TRY(cudaGetLastError(), "kvx_fill_pages");
  return KVX_OK;
}

int kvx_append_kv(kvx_pool* pool, const kvx_page_layout* layout, const uint32_t* d_page_ids, const int32_t* d_slots,
                  const void* d_k, const void* d_v, uint64_t n, void* stream) {
  if (!pool || !layout || (n && (!d_page_ids || !d_slots || !d_k || !d_v)))
    return kvx::fail_arg("kvx_append_kv: null argument");
  if (pool->fd >= 0) return kvx::fail_arg("kvx_append_kv: not on a file pool");
  if (kvx_page_bytes(layout) != pool->page_bytes) return kvx::fail_arg("kvx_append_kv: layout/page size mismatch");
  const int elt = layout->dtype == KVX_DTYPE_BF16 ? 2 : 4;
  const int row_bytes = layout->head_dim * elt;
  if (row_bytes % 16 != 0) return kvx::fail_arg("kvx_append_kv: head_dim * sizeof(dtype) must be a multiple of 16");
  if (n == 0) return KVX_OK;
  kvx::DeviceGuard guard(pool->device);
  {
    cudaLaunchConfig_t cfg{};
    cfg.gridDim = dim3(static_cast<unsigned>(n));
    cfg.blockDim = dim3(128);
    cfg.stream = kvx::as_stream(stream);
    cudaLaunchAttribute attr[1];
    attr[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;  // PDL, as the movers
    attr[0].val.programmaticStreamSerializationAllowed = 1;
    cfg.attrs = attr;
    cfg.numAttrs = 1;
    cudaLaunchKernelEx(&cfg, kvx::append_kv_kernel, pool->base, pool->page_bytes, d_page_ids, d_slots,
                       static_cast<const uint8_t*>(d_k), static_cast<const uint8_t*>(d_v), layout->num_kv_heads,
                       layout->block_tokens, row_bytes);
    kvx::note_launch();
  }
  KVX_CUDA_TRY(cudaGetLastError(), "kvx_append_kv");
  return KVX_OK;
}

}  // extern "C"
