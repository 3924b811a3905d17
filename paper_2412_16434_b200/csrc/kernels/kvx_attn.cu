// K4: paged decode attention over the KV page pool — sm_100a.
//
// Replaces the reference's modelled decode step (decode_step_time,
// /root/reference/proj/src/costmodel.cpp:59-80, consumed by
// Engine::try_start, engine.cpp:256-257) with the real computation over the
// pages the store holds: out[b][hq] = softmax(scale * q . K^T) V over the
// first ctx_len[b] tokens of request b.
//
// Roofline: every K/V byte is read once; work per byte is g (GQA group)
// multiply-adds for QK plus g for PV, i.e. 2g flop/B — 8 flop/B at g=4,
// ~30x below the bf16 tensor ridge — so the kernel is HBM-bound and is built
// to stream pages: per warp a private 3-stage cp.async ring (8 KiB = one
// page's K+V of one kv head per stage, XOR-swizzled rows so ldmatrix is
// bank-conflict free), split-K over the context so batch 1 still fills 148
// SMs, and a log-sum-exp combine. The GQA group's QK^T and PV tiles
// (g x 16 tokens x 128) are real dense contractions, so they go to the
// tensor cores with mma.sync m16n8k16 (query heads on M, padded to 16;
// tokens on N for QK, on K for PV). tcgen05/TMEM would buy nothing here:
// the tensor pipe is idle >95% of the time even with mma.sync.

#include <algorithm>
#include <atomic>
#include <cfloat>
#include <cstdlib>
#include <cmath>

#include "kvx_common.cuh"

namespace kvx {
namespace {

constexpr int kD = 128;          // head_dim of the fast path
constexpr int kT = 16;           // block_tokens of the fast path
constexpr int kWarps = 4;        // warps per CTA (wide grids); 8 when the grid is one wave
// cp.async ring depth per warp: 3 stages (96 KiB/CTA, 2 CTAs/SM). A 6-stage
// variant (1 CTA/SM, 5 pages in flight per warp) was measured slower at
// batch 1 and 8 (profiles/r01_summary.md): small batches are bound by the
// per-warp instruction latency chain, not by bytes in flight.
constexpr int kStagesWide = 3;
// One-wave (narrow) variant: 8 warps x 3 stages = 192 KiB, one CTA per SM.
#ifndef KVX_NARROW_W
#define KVX_NARROW_W 8
#endif
#ifndef KVX_NARROW_STAGES
#define KVX_NARROW_STAGES 3
#endif
constexpr int kNarrowW = KVX_NARROW_W;
constexpr int kNarrowStages = KVX_NARROW_STAGES;
constexpr int kTileBytes = kT * kD * 2;  // one kv head's K (or V) in a page: 4 KiB
constexpr int kStageBytes = 2 * kTileBytes;
constexpr int smem_bytes(int stages, int warps) { return warps * stages * kStageBytes; }
constexpr int kMaxPagesPerCta = 1024;  // block-table slice staged in smem (4 KiB)
constexpr int kMaxClusterSplits = 16;  // DSMEM split merge: one cluster per (request, kv head)
// Upper bound on split-K (auto and explicit): the GLOBAL merge stages
// splits x 32 + 16 floats of (m, l) in the page ring's shared memory.
constexpr int kMaxSplits = 256;
static_assert(kMaxSplits * 32 + 16 <= 3 * 4 * 8192 / 4, "merge staging must fit the smallest ring");
constexpr float kLog2e = 1.4426950408889634f;

// Per-CTA timeline stamps (%globaltimer) for tools/attn_trace.cu, which
// includes this file with KVX_ATTN_TRACE defined; compiled out otherwise.
#ifdef KVX_ATTN_TRACE
__device__ __forceinline__ void trace_stamp(int slot) {
  uint64_t t;
  asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
  const uint64_t cta = (static_cast<uint64_t>(blockIdx.z) * gridDim.y + blockIdx.y) * gridDim.x + blockIdx.x;
  kvx_attn_trace[cta * 32 + slot] = t;
  if (slot == 0) {
    uint32_t sm;
    asm volatile("mov.u32 %0, %%smid;" : "=r"(sm));
    kvx_attn_trace[cta * 32 + 31] = sm;
  }
}
#define KVX_TRACE(slot) (threadIdx.x == 0 ? trace_stamp(slot) : (void)0)
#define KVX_TRACE_IF(cond, slot) ((cond) ? trace_stamp(slot) : (void)0)
#else
#define KVX_TRACE(slot) ((void)0)
#define KVX_TRACE_IF(cond, slot) ((void)0)
#endif

__device__ __forceinline__ uint32_t pack_bf16(float lo, float hi) {
  uint32_t r;
  asm("cvt.rn.bf16x2.f32 %0, %1, %2;" : "=r"(r) : "f"(hi), "f"(lo));
  return r;
}

__device__ __forceinline__ void ldsm_x4(uint32_t addr, uint32_t& r0, uint32_t& r1, uint32_t& r2, uint32_t& r3) {
  asm volatile("ldmatrix.sync.aligned.m8n8.x4.shared.b16 {%0,%1,%2,%3}, [%4];"
               : "=r"(r0), "=r"(r1), "=r"(r2), "=r"(r3)
               : "r"(addr));
}
__device__ __forceinline__ void ldsm_x4_t(uint32_t addr, uint32_t& r0, uint32_t& r1, uint32_t& r2, uint32_t& r3) {
  asm volatile("ldmatrix.sync.aligned.m8n8.x4.trans.shared.b16 {%0,%1,%2,%3}, [%4];"
               : "=r"(r0), "=r"(r1), "=r"(r2), "=r"(r3)
               : "r"(addr));
}

// D[16x8] += A[16x16] * B[16x8], bf16 in, fp32 accumulate.
__device__ __forceinline__ void mma_bf16(float (&d)[4], const uint32_t (&a)[4], uint32_t b0, uint32_t b1) {
  asm volatile(
      "mma.sync.aligned.m16n8k16.row.col.f32.bf16.bf16.f32 {%0,%1,%2,%3}, {%4,%5,%6,%7}, {%8,%9}, "
      "{%0,%1,%2,%3};"
      : "+f"(d[0]), "+f"(d[1]), "+f"(d[2]), "+f"(d[3])
      : "r"(a[0]), "r"(a[1]), "r"(a[2]), "r"(a[3]), "r"(b0), "r"(b1));
}

// Address of the same shared-memory variable in CTA `rank` of the cluster.
__device__ __forceinline__ uint32_t map_rank(uint32_t smem_addr, uint32_t rank) {
  uint32_t r;
  asm volatile("mapa.shared::cluster.u32 %0, %1, %2;" : "=r"(r) : "r"(smem_addr), "r"(rank));
  return r;
}
// Asynchronous stores into another CTA's shared memory that count their
// bytes on that CTA's mbarrier (complete_tx): no fence, no separate arrive.
__device__ __forceinline__ void st_async_v4(uint32_t cluster_addr, float4 v, uint32_t cluster_bar) {
  asm volatile("st.async.shared::cluster.mbarrier::complete_tx::bytes.v4.f32 [%0], {%1, %2, %3, %4}, [%5];" ::"r"(
                   cluster_addr),
               "f"(v.x), "f"(v.y), "f"(v.z), "f"(v.w), "r"(cluster_bar)
               : "memory");
}
__device__ __forceinline__ void st_async_v2(uint32_t cluster_addr, float x, float y, uint32_t cluster_bar) {
  asm volatile("st.async.shared::cluster.mbarrier::complete_tx::bytes.v2.f32 [%0], {%1, %2}, [%3];" ::"r"(
                   cluster_addr),
               "f"(x), "f"(y), "r"(cluster_bar)
               : "memory");
}
__device__ __forceinline__ void mbar_wait_cluster(uint64_t* bar, uint32_t phase) {
  asm volatile(
      "{\n\t.reg .pred P;\n"
      "WAITC_%=:\n\t"
      "mbarrier.try_wait.parity.acquire.cluster.shared::cta.b64 P, [%0], %1;\n\t"
      "@!P bra WAITC_%=;\n}" ::"r"(smem_u32(bar)),
      "r"(phase)
      : "memory");
}

// Byte offset of 16-B chunk `col16` (0..15) of tile row `row` (0..15): rows
// are 256 B; chunks are XOR-swizzled within each 128-B half by (row & 7).
__device__ __forceinline__ uint32_t swz(int row, int col16) {
  return static_cast<uint32_t>(row * 256 + ((col16 ^ (row & 7)) << 4));
}

// The TMA ring's layout: a 4 KiB tile (16 token rows x 256 B) arrives as two
// 2 KiB boxes (columns 0-63, 64-127) written by the TMA unit with
// SWIZZLE_128B: within a box, row r's 16-B chunk c sits at chunk c ^ (r & 7).
// Same conflict-free property for ldmatrix as swz().
__device__ __forceinline__ uint32_t swz_tma(int row, int col16) {
  return static_cast<uint32_t>(((col16 >> 3) << 11) + row * 128 + (((col16 & 7) ^ (row & 7)) << 4));
}

// 2-D TMA tile load (global -> shared), completion counted on an mbarrier.
__device__ __forceinline__ void tma_load_2d(uint32_t smem_dst, const CUtensorMap* map, int col, int row,
                                            uint32_t bar) {
  asm volatile(
      "cp.async.bulk.tensor.2d.shared::cluster.global.tile.mbarrier::complete_tx::bytes [%0], [%1, {%2, %3}], [%4];"
      ::"r"(smem_dst), "l"(map), "r"(col), "r"(row), "r"(bar)
      : "memory");
}

struct AttnArgs {
  // The pool as a 2-D tensor for TMA (TMA variant): rows of 256 B (one token
  // of one kv head's K or V), row of (page p, K/V kv, head h, token t) =
  // (p * 2H + kv * H + h) * 16 + t; boxes of 64 columns x 16 rows, swizzled.
  CUtensorMap tmap;
  const uint8_t* pool;
  uint64_t page_bytes;
  uint64_t pool_pages;  // block-table entries are checked against it
  const uint32_t* tables;
  const int32_t* ctx_lens;
  const uint16_t* q;  // [B][Hq][128] bf16
  const uint16_t* new_k;  // [B][H][128] bf16: this step's token (position ctx-1), or null
  const uint16_t* new_v;
  float* out;         // [B][Hq][128]
  float* part_o;      // [B][Hq][S][128]
  float* part_ml;     // [B][Hq][S][2]
  uint32_t* arrivals; // [B][H] split counters; zero between launches
  int cluster_merge;  // 1: the splits of a (request, kv head) form clusters; merge over DSMEM
  int csize;          // cluster size (splits per cluster); splits = csize * cgroups
  int cgroups;        // clusters per (request, kv head): > 1 adds a merge of the clusters' results in the workspace
  int early_prefetch; // KVX_ATTN_EARLY_PREFETCH: table + first pages before griddepcontrol.wait
  int signal_at;      // launch_dependents: 0 after the split merge, 1 after the page loop, 2 at kernel start
  int heads;          // kv heads
  int group;          // q heads per kv head
  int max_blocks;
  int spec_pages;     // pages of the host's max_ctx: the slice the table is staged for before ctx_lens[b] arrives
  int splits;
  float scale_log2;
};

// W warps per CTA, each streaming its own pages through a kStages ring.
// kTma: each warp's ring is fed by the TMA unit (lane 0 issues four 2-D box
// loads per page onto the stage's mbarrier) instead of 16 cp.async per lane.
template <int kStages, int W, bool kTma>
__global__ void __launch_bounds__(W * 32, W >= 8 ? 1 : 8 / W) attn_bf16_d128(const __grid_constant__ AttnArgs a) {
  extern __shared__ __align__(128) uint8_t smem_raw[];
  // SWIZZLE_128B boxes need 1024-B aligned destinations (the launch adds the slack).
  uint8_t* smem = kTma ? smem_raw + ((1024 - (smem_u32(smem_raw) & 1023)) & 1023) : smem_raw;
  __shared__ __align__(8) uint64_t s_full[kTma ? W * kStages : 1];  // per (warp, stage): TMA bytes landed
  __shared__ uint32_t s_pages[kMaxPagesPerCta];
  __shared__ int s_last;
  // Cluster merge (push): CTA s of a (request, kv head) cluster owns output
  // slice s; every CTA pushes its partial of each slice into the owner's
  // s_recv_o / s_recv_ml over DSMEM and arrives on the owner's s_merge_bar.
  // Outside the page ring, so pushes may land while the owner still streams.
  __shared__ __align__(16) float s_recv_o[16 * kD + 4 * kMaxClusterSplits];
  __shared__ __align__(16) float s_recv_ml[kMaxClusterSplits * 16 * 2];
  __shared__ __align__(8) uint64_t s_merge_bar;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int split = blockIdx.x, h = blockIdx.y, b = blockIdx.z;
  if (kTma) {  // this warp's stage barriers (one arrival: lane 0's expect_tx; then the TMA bytes)
    if (lane == 0) {
#pragma unroll
      for (int s2 = 0; s2 < kStages; ++s2) mbar_init(&s_full[warp * kStages + s2], 1);
      fence_mbar_init();
    }
    __syncwarp();
  }
  // Output slice per cluster CTA, in float4 units so no vector push straddles
  // two owners.
  const int csize = a.cluster_merge ? a.csize : a.splits;
  const int crank = split % csize;  // rank in this CTA's cluster (clusters tile grid x)
  const int chunk = ((a.group * kD + csize - 1) / csize + 3) & ~3;
  if (a.cluster_merge) {
    if (threadIdx.x == 0) {
      // One arrival (ours, with the byte count) + every partial's bytes.
      const int len = max(0, min(chunk, a.group * kD - crank * chunk));
      mbar_init(&s_merge_bar, 1);
      fence_mbar_init();
      mbar_arrive_expect_tx(&s_merge_bar, static_cast<uint32_t>(csize * (len * 4 + a.group * 8)));
    }
    // Publishes the barrier (and its expected bytes) to the cluster; the
    // matching wait comes after the page loop, long after every CTA arrived.
    asm volatile("barrier.cluster.arrive.release.aligned;" ::: "memory");
  }
  // Programmatic dependent launch: this CTA may be resident before the
  // previous kernel on the stream (e.g. the prior layer, or the append of
  // this step's K/V) has finished; everything we read may be its output, so
  // wait here — what overlaps is launch, rasterisation and CTA setup. With
  // KVX_ATTN_EARLY_PREFETCH the caller promises that the block tables,
  // ctx_lens and every page except the one holding position ctx-1 are not
  // written by that kernel (a decode step only appends its token), so the
  // table and each warp's first pages are fetched before the wait.
  const bool early = a.early_prefetch != 0;
  KVX_TRACE(0);
  if (a.signal_at == 2) asm volatile("griddepcontrol.launch_dependents;" ::: "memory");
  if (!early) asm volatile("griddepcontrol.wait;" ::: "memory");
  KVX_TRACE(1);
  const uint32_t* table = a.tables + static_cast<uint64_t>(b) * a.max_blocks;
  // Stage this CTA's slice of the block table once (one coalesced read
  // instead of a dependent global load in front of every page fetch). The
  // slice depends on ctx_lens[b]; it is staged speculatively for a request
  // of the host's max_ctx (spec_pages <= max_blocks: inside the row), so the
  // table read does not wait for the ctx read — at batch 1, and whenever the
  // request is a longest one, the guess is the slice. Otherwise it is staged
  // again. Entries are checked against the pool when a page is issued.
  const int s_per = (a.spec_pages + a.splits - 1) / a.splits;
  const int s_begin = split * s_per;
  const int s_end = min(a.spec_pages, s_begin + s_per);
  const int ctx = a.ctx_lens[b];
  for (int i = threadIdx.x; i < s_end - s_begin && i < kMaxPagesPerCta; i += blockDim.x)
    s_pages[i] = __ldg(table + s_begin + i);
  // Precondition (kvx.h): 0 <= ctx_lens[b] <= max_ctx <= max_blocks * 16. A
  // longer request would read past its table row and overflow the staged
  // slice below: fail loudly instead of corrupting memory.
  if (ctx < 0 || ctx > a.max_blocks * kT) __trap();
  const int n_pages = (ctx + kT - 1) / kT;
  const int per_split = (n_pages + a.splits - 1) / a.splits;
  const int p_begin = split * per_split;
  const int p_end = min(n_pages, p_begin + per_split);
  if (p_end - p_begin > kMaxPagesPerCta) __trap();
  const int hq0 = h * a.group;
  // Q as mma A fragments. Rows = the group's query heads, zero-padded to 16.
  uint32_t qa[kD / 16][4];
  auto load_q = [&]() {
    const int r0 = lane >> 2, c = (lane & 3) * 2;
    const uint16_t* q0 = a.q + (static_cast<uint64_t>(b) * a.heads * a.group + hq0 + r0) * kD;
    const uint16_t* q8 = q0 + 8 * kD;
    const bool v0 = r0 < a.group, v8 = r0 + 8 < a.group;
#pragma unroll
    for (int kk = 0; kk < kD / 16; ++kk) {
      qa[kk][0] = v0 ? *reinterpret_cast<const uint32_t*>(q0 + kk * 16 + c) : 0u;
      qa[kk][1] = v8 ? *reinterpret_cast<const uint32_t*>(q8 + kk * 16 + c) : 0u;
      qa[kk][2] = v0 ? *reinterpret_cast<const uint32_t*>(q0 + kk * 16 + c + 8) : 0u;
      qa[kk][3] = v8 ? *reinterpret_cast<const uint32_t*>(q8 + kk * 16 + c + 8) : 0u;
    }
  };
  if (!early) load_q();  // issued first: its latency overlaps the table read

  if (p_begin != s_begin || p_end != s_end) {  // a shorter request: its own slice
    __syncthreads();
    for (int i = threadIdx.x; i < p_end - p_begin; i += blockDim.x) s_pages[i] = __ldg(table + p_begin + i);
  }
  __syncthreads();

  uint8_t* ring = smem + warp * (kStages * kStageBytes);
  const uint32_t ring_s = smem_u32(ring);
  // This warp's pages: p_begin + warp, + W, ... — a static deal, so every
  // launch sums each page into the same warp's partial in the same order
  // (bit-identical outputs run to run). A dynamic dealer (CTA-wide counter)
  // was measured at 0-4% faster and gave up that determinism.
  const int my_first = p_begin + warp;
  const int my_count = my_first < p_end ? (p_end - my_first + W - 1) / W : 0;

  auto issue = [&](int i) {  // page i of this warp -> stage i % kStages
    if (kTma) {
      if (i < my_count && lane == 0) {
        const int p = my_first + i * W;
        if (s_pages[p - p_begin] >= a.pool_pages) __trap();  // corrupt block table: fail loudly
        const int row_k = static_cast<int>(s_pages[p - p_begin]) * (2 * a.heads * kT) + h * kT;
        const int row_v = row_k + a.heads * kT;
        const uint32_t st = ring_s + (i % kStages) * kStageBytes;
        const uint32_t bar = smem_u32(&s_full[warp * kStages + (i % kStages)]);
        mbar_arrive_expect_tx(&s_full[warp * kStages + (i % kStages)], kStageBytes);
        tma_load_2d(st, &a.tmap, 0, row_k, bar);
        tma_load_2d(st + 2048, &a.tmap, 64, row_k, bar);
        tma_load_2d(st + kTileBytes, &a.tmap, 0, row_v, bar);
        tma_load_2d(st + kTileBytes + 2048, &a.tmap, 64, row_v, bar);
      }
      return;
    }
    if (i < my_count) {
      const int p = my_first + i * W;
      if (s_pages[p - p_begin] >= a.pool_pages) __trap();  // corrupt block table: fail loudly
      const uint8_t* page = a.pool + static_cast<uint64_t>(s_pages[p - p_begin]) * a.page_bytes;
      const uint8_t* k_src = page + static_cast<uint64_t>(h) * kTileBytes;
      const uint8_t* v_src = page + static_cast<uint64_t>(a.heads + h) * kTileBytes;
      uint8_t* st = ring + (i % kStages) * kStageBytes;
#pragma unroll
      for (int j = 0; j < 8; ++j) {
        const int c = lane + 32 * j, row = c >> 4, col = c & 15;
        cp_async16(st + swz(row, col), k_src + c * 16);
        cp_async16(st + kTileBytes + swz(row, col), v_src + c * 16);
      }
    }
    cp_async_commit();
  };
  // Early prefetch of this warp's first pages unless one of them is the
  // request's last page (the one this step's token goes into).
  const int last_i = (n_pages - 1 - my_first) / W;
  const bool holds_last = my_count > 0 && n_pages - 1 >= my_first && (n_pages - 1 - my_first) % W == 0 &&
                          last_i < kStages - 1;
  const bool prefetched = early && !holds_last;
  if (prefetched) {
#pragma unroll
    for (int i = 0; i < kStages - 1; ++i) issue(i);
  }
  if (early) {
    asm volatile("griddepcontrol.wait;" ::: "memory");
    load_q();
  }

  if (a.new_k != nullptr && p_begin < p_end && p_end == n_pages) {
    // Fused append (the decode step's append_blocks(1), kvstore.cpp:202-271 /
    // engine.cpp:132-166): this CTA streams the request's last page, so it
    // writes this step's K and V row of kv head h into their slot first;
    // no other CTA reads that page, and the barrier below makes the rows
    // visible to this CTA's page loads.
    if (threadIdx.x < 32) {
      const int t = ctx - 1, slot = t - (n_pages - 1) * kT;
      const uint32_t last_page = s_pages[n_pages - 1 - p_begin];
      if (last_page >= a.pool_pages) __trap();  // corrupt block table: fail loudly
      uint8_t* page = const_cast<uint8_t*>(a.pool) + static_cast<uint64_t>(last_page) * a.page_bytes;
      const int kv = threadIdx.x >> 4, c = threadIdx.x & 15;  // lanes 0-15: K row, 16-31: V row (16 x 16 B)
      const uint16_t* src = (kv ? a.new_v : a.new_k) + (static_cast<uint64_t>(b) * a.heads + h) * kD;
      uint8_t* dst = page + static_cast<uint64_t>((kv * a.heads + h) * kT + slot) * (kD * 2);
      reinterpret_cast<uint4*>(dst)[c] = reinterpret_cast<const uint4*>(src)[c];
      // The page is read next by the TMA unit (async proxy).
      if (kTma) asm volatile("fence.proxy.async.global;" ::: "memory");
    }
    __syncthreads();
  }
  KVX_TRACE(2);
  if (!prefetched) {
#pragma unroll
    for (int i = 0; i < kStages - 1; ++i) issue(i);
  }

  float o[kD / 8][4];
#pragma unroll
  for (int i = 0; i < kD / 8; ++i) o[i][0] = o[i][1] = o[i][2] = o[i][3] = 0.f;
  float m_r = -INFINITY, m_r8 = -INFINITY, l_r = 0.f, l_r8 = 0.f;

  for (int i = 0; i < my_count; ++i) {
    issue(i + kStages - 1);
    if (kTma) {
      mbar_wait(&s_full[warp * kStages + (i % kStages)], static_cast<uint32_t>((i / kStages) & 1));
    } else {
      cp_async_wait<kStages - 1>();
    }
    __syncwarp();
    if (i == 0) KVX_TRACE(3);
    const uint32_t ks = ring_s + (i % kStages) * kStageBytes;
    const uint32_t vs = ks + kTileBytes;
    const int tok0 = (my_first + i * W) * kT;

    // S^T[head][tok] = Q . K^T, two n-tiles of 8 tokens.
    // Even and odd k-steps accumulate separately: four independent mma
    // chains of depth 4 instead of two of depth 8 (shorter per-page latency).
    float s[2][4], s_odd[2][4];
#pragma unroll
    for (int j = 0; j < 2; ++j) {
      s[j][0] = s[j][1] = s[j][2] = s[j][3] = 0.f;
      s_odd[j][0] = s_odd[j][1] = s_odd[j][2] = s_odd[j][3] = 0.f;
      const int row = j * 8 + (lane & 7);
#pragma unroll
      for (int kk = 0; kk < kD / 16; kk += 2) {
        uint32_t b0, b1, b2, b3;
        ldsm_x4(ks + (kTma ? swz_tma(row, 2 * kk + (lane >> 3)) : swz(row, 2 * kk + (lane >> 3))), b0, b1, b2, b3);
        mma_bf16(s[j], qa[kk], b0, b1);
        mma_bf16(s_odd[j], qa[kk + 1], b2, b3);
      }
#pragma unroll
      for (int e = 0; e < 4; ++e) s[j][e] += s_odd[j][e];
    }
    // Online softmax (base 2), rows lane/4 and lane/4 + 8.
    float mx = -INFINITY, mx8 = -INFINITY;
#pragma unroll
    for (int j = 0; j < 2; ++j)
#pragma unroll
      for (int e = 0; e < 2; ++e) {
        const bool valid = tok0 + j * 8 + (lane & 3) * 2 + e < ctx;
        s[j][e] = valid ? s[j][e] * a.scale_log2 : -INFINITY;
        s[j][e + 2] = valid ? s[j][e + 2] * a.scale_log2 : -INFINITY;
        mx = fmaxf(mx, s[j][e]);
        mx8 = fmaxf(mx8, s[j][e + 2]);
      }
    mx = fmaxf(mx, __shfl_xor_sync(0xffffffffu, mx, 1));
    mx = fmaxf(mx, __shfl_xor_sync(0xffffffffu, mx, 2));
    mx8 = fmaxf(mx8, __shfl_xor_sync(0xffffffffu, mx8, 1));
    mx8 = fmaxf(mx8, __shfl_xor_sync(0xffffffffu, mx8, 2));
    const float mn = fmaxf(m_r, mx), mn8 = fmaxf(m_r8, mx8);
    const float base = mn == -INFINITY ? 0.f : mn, base8 = mn8 == -INFINITY ? 0.f : mn8;
    const float corr = exp2f(m_r - base), corr8 = exp2f(m_r8 - base8);
    m_r = mn;
    m_r8 = mn8;
    float p[2][4];
#pragma unroll
    for (int j = 0; j < 2; ++j) {
      p[j][0] = exp2f(s[j][0] - base);
      p[j][1] = exp2f(s[j][1] - base);
      p[j][2] = exp2f(s[j][2] - base8);
      p[j][3] = exp2f(s[j][3] - base8);
    }
    l_r = l_r * corr + (p[0][0] + p[0][1] + p[1][0] + p[1][1]);
    l_r8 = l_r8 * corr8 + (p[0][2] + p[0][3] + p[1][2] + p[1][3]);
    // Rescale O only when some row's running max moved (corr == 1 exactly
    // otherwise): after the first pages the max rarely changes.
    if (__any_sync(0xffffffffu, corr != 1.f || corr8 != 1.f)) {
#pragma unroll
      for (int n = 0; n < kD / 8; ++n) {
        o[n][0] *= corr;
        o[n][1] *= corr;
        o[n][2] *= corr8;
        o[n][3] *= corr8;
      }
    }
    // O[head][d] += P[head][tok] . V[tok][d]; P straight from the S fragments.
    uint32_t pa[4];
    pa[0] = pack_bf16(p[0][0], p[0][1]);
    pa[1] = pack_bf16(p[0][2], p[0][3]);
    pa[2] = pack_bf16(p[1][0], p[1][1]);
    pa[3] = pack_bf16(p[1][2], p[1][3]);
    const int vrow = ((lane >> 3) & 1) * 8 + (lane & 7);
#pragma unroll
    for (int n = 0; n < kD / 8; n += 2) {
      uint32_t b0, b1, b2, b3;
      ldsm_x4_t(vs + (kTma ? swz_tma(vrow, n + (lane >> 4)) : swz(vrow, n + (lane >> 4))), b0, b1, b2, b3);
      mma_bf16(o[n], pa, b0, b1);
      mma_bf16(o[n + 1], pa, b2, b3);
    }
    // The stage is refilled next by the TMA unit (async proxy): every lane
    // orders its ldmatrix reads of it before that write (WAR across proxies).
    if (kTma) asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
    __syncwarp();
  }
  if (!kTma) cp_async_wait<0>();
  KVX_TRACE(4);
  KVX_TRACE_IF(lane == 0, 16 + warp);  // per-warp loop end (slots 16..16+W-1)
  // All our global reads of the pool are done: let the next kernel's CTAs
  // start launching into SMs as ours drain. Cluster launches with many CTAs
  // each streaming a long slice signal only at the very end (below): there,
  // dependents resident this early cost more than their early start gains
  // (host-side choice, signal_at; profiles/attn_trace/r01_cluster_signal.log).
  if (a.signal_at == 1 || (!a.cluster_merge && a.signal_at == 0))
    asm volatile("griddepcontrol.launch_dependents;" ::: "memory");

  // Full row sums across the 4 lanes sharing a row.
  l_r += __shfl_xor_sync(0xffffffffu, l_r, 1);
  l_r += __shfl_xor_sync(0xffffffffu, l_r, 2);
  l_r8 += __shfl_xor_sync(0xffffffffu, l_r8, 1);
  l_r8 += __shfl_xor_sync(0xffffffffu, l_r8, 2);

  // Combine the W warps of the CTA through shared memory (reusing the rings).
  // Only the group's rows are real (the rest is mma padding); rows are padded
  // to kOs floats so the 8-byte fragment stores of a warp hit distinct banks
  // (a 128-float stride put all 8 row-lanes of a column on one bank).
  __syncthreads();
  KVX_TRACE(8);
  constexpr int kOs = kD + 8;
  float* so = reinterpret_cast<float*>(smem);                   // [warp][16][kOs]
  float* sml = so + W * 16 * kOs;                               // [warp][16][2]
  {
    const int r = lane >> 2, c = (lane & 3) * 2;
    float* ow = so + warp * 16 * kOs;
    if (r < a.group) {
#pragma unroll
      for (int n = 0; n < kD / 8; ++n)
        *reinterpret_cast<float2*>(ow + r * kOs + n * 8 + c) = make_float2(o[n][0], o[n][1]);
    }
    if (r + 8 < a.group) {
#pragma unroll
      for (int n = 0; n < kD / 8; ++n)
        *reinterpret_cast<float2*>(ow + (r + 8) * kOs + n * 8 + c) = make_float2(o[n][2], o[n][3]);
    }
    if ((lane & 3) == 0) {
      sml[(warp * 16 + r) * 2] = m_r;
      sml[(warp * 16 + r) * 2 + 1] = l_r;
      sml[(warp * 16 + r + 8) * 2] = m_r8;
      sml[(warp * 16 + r + 8) * 2 + 1] = l_r8;
    }
  }
  __syncthreads();
  const int rows = a.group;
  if (a.cluster_merge) {
    // Per-row weights of each warp's partial, then pushes: every CTA sends
    // its (m, l) per row to every owner (one 8-byte st.async per (row, owner))
    // and each float4 of its partial O to the owner of that slice. The
    // owner's mbarrier completes when all bytes have landed.
    // Every thread derives the weights of the row it pushes itself (redundant
    // but parallel: measured faster than a few threads + a barrier here).
    auto row_weights = [&](int r, float (&f)[W], float& M, float& L) {
      M = -INFINITY;
#pragma unroll
      for (int w = 0; w < W; ++w) M = fmaxf(M, sml[(w * 16 + r) * 2]);
      const float Mb = M == -INFINITY ? 0.f : M;
      L = 0.f;
#pragma unroll
      for (int w = 0; w < W; ++w) {
        f[w] = exp2f(sml[(w * 16 + r) * 2] - Mb);
        L += f[w] * sml[(w * 16 + r) * 2 + 1];
      }
    };
    asm volatile("barrier.cluster.wait.acquire.aligned;" ::: "memory");  // every owner's barrier is armed
    const uint32_t bar_local = smem_u32(&s_merge_bar);
    if (threadIdx.x < rows * csize) {
      const int r = threadIdx.x / csize, owner = threadIdx.x - r * csize;
      float f[W], M, L;
      row_weights(r, f, M, L);
      st_async_v2(map_rank(smem_u32(s_recv_ml + (crank * 16 + r) * 2), owner), M, L, map_rank(bar_local, owner));
    }
    for (int q = threadIdx.x; q < rows * kD / 4; q += blockDim.x) {
      const int e = 4 * q, r = e / kD, d = e - r * kD;
      float f[W], M, L;
      row_weights(r, f, M, L);
      float4 O = make_float4(0.f, 0.f, 0.f, 0.f);
#pragma unroll
      for (int w = 0; w < W; ++w) {
        const float4 v = *reinterpret_cast<const float4*>(so + (w * 16 + r) * kOs + d);
        O.x += f[w] * v.x;
        O.y += f[w] * v.y;
        O.z += f[w] * v.z;
        O.w += f[w] * v.w;
      }
      const int owner = e / chunk;
      st_async_v4(map_rank(smem_u32(s_recv_o + crank * chunk + (e - owner * chunk)), owner), O,
                  map_rank(bar_local, owner));
    }
    KVX_TRACE(5);
    // Our slice: wait for every split's bytes, merge from local shared memory.
    // No CTA exits before every push into it has landed and none reads
    // another CTA's memory, so no closing cluster barrier is needed.
    mbar_wait_cluster(&s_merge_bar, 0);
    KVX_TRACE(10);
    const int ns = csize;
    const int e_begin = crank * chunk, e_end = min(rows * kD, (crank + 1) * chunk);
    const int G = a.cgroups, cg = split / csize;
    const uint64_t row0 = static_cast<uint64_t>(b) * a.heads * a.group + hq0;
    for (int e = e_begin + threadIdx.x; e < e_end; e += blockDim.x) {
      const int r = e / kD, d = e - r * kD, off = e - e_begin;
      float M = -INFINITY;
      for (int s2 = 0; s2 < ns; ++s2) M = fmaxf(M, s_recv_ml[(s2 * 16 + r) * 2]);
      const float Mb = M == -INFINITY ? 0.f : M;
      float L = 0.f, O = 0.f;
      for (int s2 = 0; s2 < ns; ++s2) {
        const float f = exp2f(s_recv_ml[(s2 * 16 + r) * 2] - Mb);
        L += f * s_recv_ml[(s2 * 16 + r) * 2 + 1];
        O += f * s_recv_o[s2 * chunk + off];
      }
      if (G == 1) {
        a.out[(row0 + r) * kD + d] = L > 0.f ? O / L : 0.f;
      } else {  // this cluster's partial of the slice, for the merge across clusters
        a.part_o[((row0 + r) * G + cg) * kD + d] = O;
        if (d == 0 || e == e_begin) {  // (M, L) of the row: identical in every owner of this cluster
          a.part_ml[((row0 + r) * G + cg) * 2] = M;
          a.part_ml[((row0 + r) * G + cg) * 2 + 1] = L;
        }
      }
    }
    if (G > 1) {
      // Merge across the G clusters of this (request, kv head), slice by
      // slice: the owners of slice crank arrive on one counter; the last one
      // combines the G partials in cluster order (deterministic) and resets it.
      __threadfence();
      __syncthreads();
      uint32_t* arrive = a.arrivals + (static_cast<uint64_t>(b) * a.heads + h) * kMaxClusterSplits + crank;
      if (threadIdx.x == 0) s_last = atomicAdd(arrive, 1u) == static_cast<uint32_t>(G - 1);
      __syncthreads();
      if (s_last) {
        __threadfence();
        for (int e = e_begin + threadIdx.x; e < e_end; e += blockDim.x) {
          const int r = e / kD, d = e - r * kD;
          const float* ml = a.part_ml + (row0 + r) * G * 2;
          float M = -INFINITY;
          for (int g2 = 0; g2 < G; ++g2) M = fmaxf(M, __ldcg(ml + 2 * g2));
          const float Mb = M == -INFINITY ? 0.f : M;
          float L = 0.f, O = 0.f;
          for (int g2 = 0; g2 < G; ++g2) {
            const float f = exp2f(__ldcg(ml + 2 * g2) - Mb);
            L += f * __ldcg(ml + 2 * g2 + 1);
            O += f * __ldcg(a.part_o + ((row0 + r) * G + g2) * kD + d);
          }
          a.out[(row0 + r) * kD + d] = L > 0.f ? O / L : 0.f;
        }
        if (threadIdx.x == 0) *arrive = 0;  // ready for the next launch
      }
    }
    KVX_TRACE(6);
    if (a.signal_at == 0) asm volatile("griddepcontrol.launch_dependents;" ::: "memory");
    return;
  }
  for (int e = threadIdx.x; e < rows * kD; e += blockDim.x) {
    const int r = e / kD, d = e - r * kD;
    float M = -INFINITY;
#pragma unroll
    for (int w = 0; w < W; ++w) M = fmaxf(M, sml[(w * 16 + r) * 2]);
    const float Mb = M == -INFINITY ? 0.f : M;
    float L = 0.f, O = 0.f;
#pragma unroll
    for (int w = 0; w < W; ++w) {
      const float f = exp2f(sml[(w * 16 + r) * 2] - Mb);
      L += f * sml[(w * 16 + r) * 2 + 1];
      O += f * so[(w * 16 + r) * kOs + d];
    }
    const uint64_t row = static_cast<uint64_t>(b) * a.heads * a.group + hq0 + r;
    if (a.splits == 1) {
      a.out[row * kD + d] = L > 0.f ? O / L : 0.f;
    } else {
      a.part_o[(row * a.splits + split) * kD + d] = O;
      if (d == 0) {
        a.part_ml[(row * a.splits + split) * 2] = M;
        a.part_ml[(row * a.splits + split) * 2 + 1] = L;
      }
    }
  }
  KVX_TRACE(5);
  if (a.splits == 1) return;

  // Split-K merge fused in: the last CTA of this (request, kv head) to finish
  // merges every split's partial (L2-resident) — no second launch.
  __threadfence();
  __syncthreads();
  if (threadIdx.x == 0) {
    const uint32_t prev = atomicAdd(a.arrivals + static_cast<uint64_t>(b) * a.heads + h, 1u);
    s_last = prev == static_cast<uint32_t>(a.splits - 1);
  }
  __syncthreads();
  if (!s_last) return;
  __threadfence();
  // Stage every split's (m, l) in shared memory with one load per thread,
  // turn them into per-row weights, then stream the partial O rows with
  // 8 independent L2 loads in flight per thread.
  float* sm_m = reinterpret_cast<float*>(smem);  // [splits][16]
  float* sm_l = sm_m + a.splits * 16;            // [splits][16] -> weights
  float* sm_inv = sm_l + a.splits * 16;          // [16] 1 / L
  const uint64_t row0 = static_cast<uint64_t>(b) * a.heads * a.group + hq0;
  for (int i = threadIdx.x; i < rows * a.splits; i += blockDim.x) {
    const int r = i / a.splits, s = i - r * a.splits;
    const float* ml = a.part_ml + ((row0 + r) * a.splits + s) * 2;
    sm_m[s * 16 + r] = __ldcg(ml);
    sm_l[s * 16 + r] = __ldcg(ml + 1);
  }
  __syncthreads();
  if (threadIdx.x < rows) {
    const int r = threadIdx.x;
    float M = -INFINITY;
    for (int s = 0; s < a.splits; ++s) M = fmaxf(M, sm_m[s * 16 + r]);
    const float Mb = M == -INFINITY ? 0.f : M;
    float L = 0.f;
    for (int s = 0; s < a.splits; ++s) {
      const float f = exp2f(sm_m[s * 16 + r] - Mb);
      L += f * sm_l[s * 16 + r];
      sm_l[s * 16 + r] = f;
    }
    sm_inv[r] = L > 0.f ? 1.f / L : 0.f;
  }
  __syncthreads();
  for (int e = threadIdx.x; e < rows * kD; e += blockDim.x) {
    const int r = e / kD, d = e - r * kD;
    const float* po = a.part_o + (row0 + r) * a.splits * kD + d;
    float acc0 = 0.f, acc1 = 0.f;
    int s = 0;
    for (; s + 8 <= a.splits; s += 8) {
      float v[8];
#pragma unroll
      for (int j = 0; j < 8; ++j) v[j] = __ldcg(po + (s + j) * kD);
#pragma unroll
      for (int j = 0; j < 8; j += 2) {
        acc0 += sm_l[(s + j) * 16 + r] * v[j];
        acc1 += sm_l[(s + j + 1) * 16 + r] * v[j + 1];
      }
    }
    for (; s < a.splits; ++s) acc0 += sm_l[s * 16 + r] * __ldcg(po + s * kD);
    a.out[(row0 + r) * kD + d] = (acc0 + acc1) * sm_inv[r];
  }
  if (threadIdx.x == 0) a.arrivals[static_cast<uint64_t>(b) * a.heads + h] = 0;  // ready for the next launch
  KVX_TRACE(6);
}

// Generic path (any head_dim <= 256 that is a multiple of 32, fp32 or bf16,
// any block_tokens): one warp per (request, query head), fp32 online softmax.
// Serves the tiny fp32 configuration; not a performance path.
template <typename T>
__device__ __forceinline__ float ld_elt(const T* p);
template <>
__device__ __forceinline__ float ld_elt<float>(const float* p) { return *p; }
template <>
__device__ __forceinline__ float ld_elt<uint16_t>(const uint16_t* p) {
  return __uint_as_float(static_cast<uint32_t>(*p) << 16);
}

template <typename T>
__global__ void attn_generic(const uint8_t* pool, uint64_t page_bytes, uint64_t pool_pages, const uint32_t* tables,
                             const int32_t* ctx_lens, const T* q, float* out, int heads, int group, int head_dim,
                             int block_tokens, int max_blocks, float scale) {
  const int b = blockIdx.y, hq = blockIdx.x, h = hq / group, lane = threadIdx.x;
  if (ctx_lens[b] < 0 || ctx_lens[b] > max_blocks * block_tokens) __trap();  // past the table row
  const int per_lane = head_dim / 32;
  float qv[8], acc[8];
  const T* qrow = q + (static_cast<uint64_t>(b) * heads * group + hq) * head_dim;
  for (int i = 0; i < per_lane; ++i) {
    qv[i] = ld_elt<T>(qrow + lane + 32 * i);
    acc[i] = 0.f;
  }
  const int ctx = ctx_lens[b];
  float m = -INFINITY, l = 0.f;
  for (int t = 0; t < ctx; ++t) {
    const uint32_t page = tables[static_cast<uint64_t>(b) * max_blocks + t / block_tokens];
    if (page >= pool_pages) __trap();  // corrupt block table: fail loudly
    const int slot = t % block_tokens;
    const T* base = reinterpret_cast<const T*>(pool + static_cast<uint64_t>(page) * page_bytes);
    const T* k = base + (static_cast<uint64_t>(h) * block_tokens + slot) * head_dim;
    const T* v = base + (static_cast<uint64_t>(heads + h) * block_tokens + slot) * head_dim;
    float dot = 0.f;
    for (int i = 0; i < per_lane; ++i) dot += qv[i] * ld_elt<T>(k + lane + 32 * i);
#pragma unroll
    for (int off = 16; off > 0; off >>= 1) dot += __shfl_xor_sync(0xffffffffu, dot, off);
    const float x = dot * scale;
    const float mn = fmaxf(m, x);
    const float corr = __expf(m - mn), p = __expf(x - mn);
    l = l * corr + p;
    for (int i = 0; i < per_lane; ++i) acc[i] = acc[i] * corr + p * ld_elt<T>(v + lane + 32 * i);
    m = mn;
  }
  float* orow = out + (static_cast<uint64_t>(b) * heads * group + hq) * head_dim;
  for (int i = 0; i < per_lane; ++i) orow[lane + 32 * i] = l > 0.f ? acc[i] / l : 0.f;
}

// The decode step's append for the generic path: request b's token at
// position ctx_lens[b] - 1 goes to its slot in the page its block table
// names (one CTA per request, every kv head's K and V row).
__global__ void __launch_bounds__(128) append_from_table(uint8_t* pool, uint64_t page_bytes, uint64_t pool_pages,
                                                         const uint32_t* tables, const int32_t* ctx_lens,
                                                         const uint8_t* new_k, const uint8_t* new_v, int heads,
                                                         int block_tokens, int row_bytes, int max_blocks) {
  const int b = blockIdx.x;
  const int t = ctx_lens[b] - 1;
  if (t < 0) return;
  if (t / block_tokens >= max_blocks) __trap();  // past the table row
  const uint32_t page = tables[static_cast<uint64_t>(b) * max_blocks + t / block_tokens];
  if (page >= pool_pages) __trap();
  const int slot = t % block_tokens;
  uint8_t* base = pool + static_cast<uint64_t>(page) * page_bytes;
  const int vecs = row_bytes / 16;
  for (int e = threadIdx.x; e < 2 * heads * vecs; e += blockDim.x) {
    const int kv = e / (heads * vecs), rem = e - kv * heads * vecs, h = rem / vecs, c = rem - h * vecs;
    const uint8_t* src = (kv ? new_v : new_k) + (static_cast<uint64_t>(b) * heads + h) * row_bytes;
    uint8_t* dst = base + (static_cast<uint64_t>(kv * heads + h) * block_tokens + slot) * row_bytes;
    reinterpret_cast<uint4*>(dst)[c] = reinterpret_cast<const uint4*>(src)[c];
  }
}

bool fast_path(const kvx_page_layout* l) {
  return l->dtype == KVX_DTYPE_BF16 && l->head_dim == kD && l->block_tokens == kT;
}

// Split-K factor, from the B200 split sweeps (profiles/r01_attn_split_sweep_long.jsonl:
// batch 1-16 x ctx 8K/32K x 32/64 q heads, every split count, both merges).
// One-wave grids (8 warps per CTA, one CTA per SM) are best with ~2/3 of the
// SMs streaming: splits = round(0.65 * SMs / (requests x kv heads)) (batch 2
// -> 6, 4 -> 3, 8 -> 2, 16 -> 1; batch 1 -> 12, which plan_attention steps
// down to the largest co-resident cluster). A sub-wave grid of 2-CTA/SM
// blocks over a very long context (>= 1024 pages per CTA) is split 4x more
// so the CTAs balance over the SMs (batch 16 x 32K: 2 -> 8 splits, -5%).
// Bounded by the block-table staging limit and by >= 16 pages per CTA.
int choose_splits(int batch, int heads, int max_ctx, int requested, int sms) {
  const int pages = std::max(1, (max_ctx + kT - 1) / kT);
  const int min_splits = (pages + kMaxPagesPerCta - 1) / kMaxPagesPerCta;
  if (requested > 0) return std::max(requested, min_splits);  // <= kMaxSplits, checked by the caller
  const int max_splits = std::max(min_splits, pages / (kWarps * 4));
  const long base = std::max(1L, static_cast<long>(batch) * heads);
  int s = std::max(min_splits, static_cast<int>(std::lround(0.65 * sms / static_cast<double>(base))));
  s = std::max(1, std::min(s, kMaxSplits));
  if (s * base > sms && s * base < 2L * sms && pages / s >= 1024) s *= 4;
  return std::max(min_splits, std::min(max_splits, s));
}

// Split partials ([B][Hq][S][kD + 2] floats) + arrival counters
// ([B][H][kMaxClusterSplits]: one per (request, kv head), or per output slice
// when the splits form several clusters). Sized for at least
// kMaxClusterSplits splits, so any plan of this launch shape fits.
uint64_t workspace_for(uint64_t batch, uint64_t hq, uint64_t heads, int splits) {
  if (splits <= 1) return 0;
  const uint64_t s = static_cast<uint64_t>(std::max(splits, kMaxClusterSplits));
  return batch * hq * s * (kD + 2) * sizeof(float) + batch * heads * kMaxClusterSplits * sizeof(uint32_t);
}

// One-time per-device kernel attributes (dynamic smem, cluster sizes > 8).
// Idempotent, so concurrent first calls from several host threads are fine;
// the flags are atomics so the check itself is race-free.
template <bool kTma>
int configure_variant() {
  constexpr int slack = kTma ? 1024 : 0;  // 1024-B alignment of the TMA ring
  KVX_CUDA_TRY(cudaFuncSetAttribute(attn_bf16_d128<kStagesWide, 4, kTma>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                    smem_bytes(kStagesWide, 4) + slack),
               "kvx_decode_attention: smem attribute");
  KVX_CUDA_TRY(cudaFuncSetAttribute(attn_bf16_d128<kNarrowStages, kNarrowW, kTma>,
                                    cudaFuncAttributeMaxDynamicSharedMemorySize,
                                    smem_bytes(kNarrowStages, kNarrowW) + slack),
               "kvx_decode_attention: smem attribute");
  KVX_CUDA_TRY(cudaFuncSetAttribute(attn_bf16_d128<kNarrowStages, kNarrowW, kTma>,
                                    cudaFuncAttributeNonPortableClusterSizeAllowed, 1),
               "kvx_decode_attention: cluster attribute");
  return KVX_OK;
}

int configure(int device) {
  static std::atomic<bool> configured[64] = {};
  const int slot = device < 0 ? 0 : device % 64;
  if (configured[slot].load(std::memory_order_acquire)) return KVX_OK;
  if (int rc = configure_variant<false>()) return rc;
  if (int rc = configure_variant<true>()) return rc;
  configured[slot].store(true, std::memory_order_release);
  return KVX_OK;
}

// The pool as a 2-D tensor for K4's TMA feed: 256-B rows (one token of one
// kv head's K or V), boxes of 64 columns x 16 rows with SWIZZLE_128B. Built
// once per pool through the driver's cuTensorMapEncodeTiled (resolved via
// the runtime, so libkvx needs no libcuda link). nullptr when the pool
// cannot be described (too many rows, misaligned base).
using EncodeTiled = CUresult (*)(CUtensorMap*, CUtensorMapDataType, cuuint32_t, void*, const cuuint64_t*,
                                 const cuuint64_t*, const cuuint32_t*, const cuuint32_t*, CUtensorMapInterleave,
                                 CUtensorMapSwizzle, CUtensorMapL2promotion, CUtensorMapFloatOOBfill);

const CUtensorMap* attn_tensor_map(kvx_pool* pool, int heads) {
  std::lock_guard<std::mutex> lock(pool->tmap_mu);
  if (pool->tmap_heads == heads) return &pool->tmap;
  if (pool->tmap_heads == -2) return nullptr;
  static EncodeTiled encode = nullptr;
  if (!encode) {
    void* fn = nullptr;
    cudaDriverEntryPointQueryResult q{};
    if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &fn, cudaEnableDefault, &q) != cudaSuccess ||
        q != cudaDriverEntryPointSuccess || !fn) {
      cudaGetLastError();
      pool->tmap_heads = -2;
      return nullptr;
    }
    encode = reinterpret_cast<EncodeTiled>(fn);
  }
  const uint64_t rows = pool->num_pages * pool->page_bytes / 256;
  if (pool->page_bytes % 256 || rows >= (1ull << 31) || reinterpret_cast<uintptr_t>(pool->base) % 16) {
    pool->tmap_heads = -2;
    return nullptr;
  }
  const cuuint64_t dims[2] = {kD, rows};
  const cuuint64_t strides[1] = {256};
  const cuuint32_t box[2] = {64, kT};
  const cuuint32_t elem[2] = {1, 1};
  const CUresult r = encode(&pool->tmap, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 2, pool->base, dims, strides, box, elem,
                            CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B,
                            CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  pool->tmap_heads = r == CUDA_SUCCESS ? heads : -2;
  return r == CUDA_SUCCESS ? &pool->tmap : nullptr;
}

// How many clusters of `splits` one-SM CTAs (8 warps, 192 KiB smem) the
// device runs at once (cudaOccupancyMaxActiveClusters; GPC-shape dependent).
int cluster_capacity(int device, int splits, bool tma) {
  static std::atomic<int> cache[64][2][kMaxClusterSplits + 1] = {};
  const int slot = device < 0 ? 0 : device % 64;
  std::atomic<int>& cached = cache[slot][tma ? 1 : 0][splits];
  int c = cached.load(std::memory_order_relaxed);
  if (c == 0) {
    cudaLaunchConfig_t cfg{};
    cfg.gridDim = dim3(splits, 1, 1);
    cfg.blockDim = dim3(kNarrowW * 32);
    cfg.dynamicSmemBytes = smem_bytes(kNarrowStages, kNarrowW) + (tma ? 1024 : 0);
    cudaLaunchAttribute attr[1];
    attr[0].id = cudaLaunchAttributeClusterDimension;
    attr[0].val.clusterDim.x = splits;
    attr[0].val.clusterDim.y = 1;
    attr[0].val.clusterDim.z = 1;
    cfg.attrs = attr;
    cfg.numAttrs = 1;
    int n = 0;
    const cudaError_t e = tma ? cudaOccupancyMaxActiveClusters(&n, attn_bf16_d128<kNarrowStages, kNarrowW, true>, &cfg)
                              : cudaOccupancyMaxActiveClusters(&n, attn_bf16_d128<kNarrowStages, kNarrowW, false>, &cfg);
    c = e == cudaSuccess ? std::max(n, 0) : 0;
    if (c == 0) {
      cudaGetLastError();
      c = -1;  // cached "does not fit"
    }
    cached.store(c, std::memory_order_relaxed);
  }
  return c;
}

struct Plan {
  int splits;
  bool cluster;    // merge over DSMEM (cluster size = splits / groups)
  bool narrow;     // 8 warps per CTA
  int groups = 1;  // clusters per (request, kv head); > 1: their results merge in the workspace
};

// Launch plan: the split count from choose_splits; the splits of each
// (request, kv head) merge over DSMEM when they fit one cluster and all
// B x H clusters are co-resident (one CTA per SM), else through the
// workspace. Traced on B200 (tools/attn_trace.cu, profiles/r01_summary.md):
// the DSMEM merge saves ~1 us per launch at batch 1-4 (12 and 16-CTA
// clusters do not co-reside 8 at a time on B200's GPCs and run in two
// waves, which the occupancy check catches). Explicit split counts and
// merge modes are honoured (tests, sweeps).
Plan plan_attention(int batch, int heads, int max_ctx, int requested, int merge, int device, bool tma,
                    int req_groups = 1) {
  const int sms = sm_count(device);
  const long groups = std::max(1L, static_cast<long>(batch) * heads);
  const int pages = std::max(1, (max_ctx + kT - 1) / kT);
  const int min_splits = (pages + kMaxPagesPerCta - 1) / kMaxPagesPerCta;
  Plan p{choose_splits(batch, heads, max_ctx, requested, sms), false, false};
  if (merge != KVX_MERGE_GLOBAL) {
    // The largest cluster size in [~3/4 of the target, target] whose clusters
    // are all co-resident (one wave); explicit split counts are taken as is.
    const int target = p.splits;
    const int lowest = requested > 0 ? target : std::max(2, (3 * target + 3) / 4);
    for (int s = std::min(target, kMaxClusterSplits); s >= lowest; --s) {
      const bool ok = s >= 2 && s >= min_splits && groups * s <= sms &&
                      cluster_capacity(device, s, tma) >= (requested > 0 ? 1 : groups);
      if (ok) {
        p = Plan{s, true, true};
        break;
      }
    }
  }
  // Two-level merge on request (KVX_ATTN_CLUSTERS(G) in the flags with an
  // explicit split count S): S/G-CTA clusters, G per (request, kv head).
  if (req_groups > 1 && requested > 0 && merge != KVX_MERGE_GLOBAL)
    return Plan{requested, true, true, req_groups};
  if (!p.cluster) p.narrow = static_cast<long>(p.splits) * groups <= sms;
  // KVX_ATTN_NARROW=0|1 forces the 4-warp (2 CTAs/SM) / 8-warp variant of a
  // workspace-merged launch (measurement knob).
  static const char* narrow_env = std::getenv("KVX_ATTN_NARROW");
  if (!p.cluster && narrow_env && (narrow_env[0] == '0' || narrow_env[0] == '1')) p.narrow = narrow_env[0] == '1';
  return p;
}

}  // namespace
}  // namespace kvx

extern "C" {

uint64_t kvx_decode_attention_workspace(const kvx_page_layout* layout, const kvx_attn_params* params, int32_t batch,
                                        int32_t max_ctx) {
  if (!layout || !params || batch <= 0 || !kvx::fast_path(layout)) return 0;
  const int splits = kvx::choose_splits(batch, layout->num_kv_heads, max_ctx, params->num_splits, kvx::sm_count(0));
  return kvx::workspace_for(batch, params->num_q_heads, layout->num_kv_heads, splits);
}

}  // extern "C"

namespace kvx {
namespace {

int decode_attention(const kvx_pool* pool, const kvx_page_layout* layout, const kvx_attn_params* params,
                     const uint32_t* d_block_tables, const int32_t* d_ctx_lens, const void* d_q, const void* d_new_k,
                     const void* d_new_v, float* d_out, int32_t batch, int32_t max_ctx, void* d_workspace,
                     uint64_t workspace_bytes, void* stream) {
  if (!pool || !layout || !params || !d_block_tables || !d_ctx_lens || !d_q || !d_out)
    return kvx::fail_arg("kvx_decode_attention: null argument");
  if (pool->fd >= 0) return kvx::fail_arg("kvx_decode_attention: not on a file pool");
  if (batch <= 0) return KVX_OK;
  const int H = layout->num_kv_heads, Hq = params->num_q_heads;
  if (H <= 0 || Hq <= 0 || Hq % H != 0) return kvx::fail_arg("kvx_decode_attention: num_q_heads must be a multiple of num_kv_heads");
  if (kvx_page_bytes(layout) != pool->page_bytes) return kvx::fail_arg("kvx_decode_attention: layout/page size mismatch");
  if (max_ctx < 0 || static_cast<int64_t>(max_ctx) > static_cast<int64_t>(params->max_blocks) * layout->block_tokens)
    return kvx::fail_arg("kvx_decode_attention: max_ctx exceeds the block-table row (max_blocks * block_tokens)");
  const int group = Hq / H;
  const float scale = params->scale > 0.f ? params->scale : 1.0f / std::sqrt(static_cast<float>(layout->head_dim));
  const cudaStream_t st = kvx::as_stream(stream);
  kvx::DeviceGuard guard(pool->device);

  if (params->num_splits < 0 || params->num_splits > kvx::kMaxSplits)
    return kvx::fail_arg("kvx_decode_attention: num_splits must be in [0, 256]");
  if (kvx::fast_path(layout) && group <= 16) {
    const int dev = pool->device < 0 ? 0 : pool->device;
    if (int rc = kvx::configure(dev)) return rc;
    if (params->split_merge < KVX_MERGE_AUTO || params->split_merge > KVX_MERGE_CLUSTER)
      return kvx::fail_arg("kvx_decode_attention: unknown split_merge");
    // TMA feed (default) unless disabled by KVX_ATTN_TMA=0 (measurement knob)
    // or the pool cannot be described as a tensor.
    static const char* tma_env = std::getenv("KVX_ATTN_TMA");
    const CUtensorMap* tmap = (tma_env && tma_env[0] == '0')
                                  ? nullptr
                                  : kvx::attn_tensor_map(const_cast<kvx_pool*>(pool), H);
    const bool tma = tmap != nullptr;
    const int req_groups = (params->flags >> 8) & 0xF;
    if (req_groups > 1 && (params->num_splits <= 0 || params->num_splits % req_groups ||
                           params->num_splits / req_groups < 2 ||
                           params->num_splits / req_groups > kvx::kMaxClusterSplits ||
                           params->split_merge == KVX_MERGE_GLOBAL))
      return kvx::fail_arg("kvx_decode_attention: KVX_ATTN_CLUSTERS(G) needs num_splits = G x C, 2 <= C <= 16, "
                           "and a cluster merge");
    const kvx::Plan plan =
        kvx::plan_attention(batch, H, max_ctx, params->num_splits, params->split_merge, dev, tma, req_groups);
    if (params->split_merge == KVX_MERGE_CLUSTER && !plan.cluster && plan.splits > 1)
      return kvx::fail_arg("kvx_decode_attention: split_merge=CLUSTER but the splits do not fit one cluster");
    const int splits = plan.splits;
    kvx::AttnArgs a{};
    if (tma) a.tmap = *tmap;
    a.pool = pool->base;
    a.page_bytes = pool->page_bytes;
    a.pool_pages = pool->num_pages;
    a.tables = d_block_tables;
    a.ctx_lens = d_ctx_lens;
    a.q = static_cast<const uint16_t*>(d_q);
    a.new_k = static_cast<const uint16_t*>(d_new_k);
    a.new_v = static_cast<const uint16_t*>(d_new_v);
    a.out = d_out;
    a.heads = H;
    a.group = group;
    a.max_blocks = params->max_blocks;
    a.spec_pages = std::min(params->max_blocks, (max_ctx + kvx::kT - 1) / kvx::kT);
    a.splits = splits;
    a.scale_log2 = scale * kvx::kLog2e;
    a.cluster_merge = plan.cluster ? 1 : 0;
    a.cgroups = plan.cluster ? plan.groups : 1;
    a.csize = plan.cluster ? splits / plan.groups : splits;
    a.early_prefetch = (params->flags & KVX_ATTN_EARLY_PREFETCH) ? 1 : 0;
    {
      // Measured with early prefetch on (32 / 64 q heads, batch 1-8,
      // 8K-131K): signalling dependents right after the page loop wins 5-11%
      // when the grid is small (<= 80 CTAs) or each CTA's slice is short
      // (<= 256 pages); with ~100+ CTAs each streaming 340+ pages the late
      // signal is 2-3% better. Without early prefetch the early-resident
      // dependents only spin and the late signal wins everywhere.
      const int pages = std::max(1, (max_ctx + kvx::kT - 1) / kvx::kT);
      const int per_cta = (pages + splits - 1) / splits;
      const long ctas = static_cast<long>(splits) * H * batch;
      a.signal_at = (a.early_prefetch && (ctas <= 80 || per_cta <= 256)) ? 1 : 0;
      // KVX_ATTN_SIGNAL=0|1|2 (after merge / after loop / at start): measurement knob.
      static const char* sig_env = std::getenv("KVX_ATTN_SIGNAL");
      if (sig_env && sig_env[0] >= '0' && sig_env[0] <= '2') a.signal_at = sig_env[0] - '0';
    }
    if (splits > 1 && (!plan.cluster || plan.groups > 1)) {
      const uint64_t rows = static_cast<uint64_t>(batch) * Hq;
      if (!d_workspace || workspace_bytes < kvx::workspace_for(batch, Hq, H, splits))
        return kvx::fail_arg("kvx_decode_attention: workspace too small");
      a.part_o = static_cast<float*>(d_workspace);
      a.part_ml = a.part_o + rows * splits * kvx::kD;
      a.arrivals = reinterpret_cast<uint32_t*>(a.part_ml + rows * splits * 2);
    }
    dim3 grid(splits, H, batch);
    // One wave or less: 8 warps per CTA (two per scheduler) halve each warp's
    // serial page chain; otherwise 4 warps and 2 CTAs per SM.
    const bool narrow = plan.narrow;
    cudaLaunchConfig_t cfg{};
    cfg.gridDim = grid;
    cfg.blockDim = dim3(narrow ? kvx::kNarrowW * 32 : 4 * 32);
    cfg.dynamicSmemBytes = (narrow ? kvx::smem_bytes(kvx::kNarrowStages, kvx::kNarrowW) : kvx::smem_bytes(kvx::kStagesWide, 4)) +
                           (tma ? 1024 : 0);
    cfg.stream = st;
    cudaLaunchAttribute attr[2];
    attr[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;  // PDL
    attr[0].val.programmaticStreamSerializationAllowed = 1;
    attr[1].id = cudaLaunchAttributeClusterDimension;
    attr[1].val.clusterDim.x = plan.cluster ? splits / plan.groups : 1;
    attr[1].val.clusterDim.y = 1;
    attr[1].val.clusterDim.z = 1;
    // Cluster launches use PDL too, with launch_dependents at the very end of
    // the kernel (after the split merge): signalled after the page loop, the
    // early-resident dependent clusters fragmented the GPCs and cost 4-11 us
    // per launch at batch 1 >= 32K; signalled at the end they save 0.3-0.6 us
    // per launch at every clustered shape (profiles/attn_trace/
    // r01_cluster_pdl_late.log). KVX_ATTN_CLUSTER_PDL=0 turns it off
    // (measurement knob).
    static const char* cluster_pdl_env = std::getenv("KVX_ATTN_CLUSTER_PDL");
    const bool cluster_pdl = !(cluster_pdl_env && cluster_pdl_env[0] == '0');
    if (plan.cluster && !cluster_pdl) attr[0].val.programmaticStreamSerializationAllowed = 0;
    cfg.attrs = attr;
    cfg.numAttrs = plan.cluster ? 2 : 1;
    if (narrow && tma)
      KVX_CUDA_TRY(cudaLaunchKernelEx(&cfg, kvx::attn_bf16_d128<kvx::kNarrowStages, kvx::kNarrowW, true>, a),
                   "kvx_decode_attention");
    else if (narrow)
      KVX_CUDA_TRY(cudaLaunchKernelEx(&cfg, kvx::attn_bf16_d128<kvx::kNarrowStages, kvx::kNarrowW, false>, a),
                   "kvx_decode_attention");
    else if (tma)
      KVX_CUDA_TRY(cudaLaunchKernelEx(&cfg, kvx::attn_bf16_d128<kvx::kStagesWide, 4, true>, a), "kvx_decode_attention");
    else
      KVX_CUDA_TRY(cudaLaunchKernelEx(&cfg, kvx::attn_bf16_d128<kvx::kStagesWide, 4, false>, a), "kvx_decode_attention");
    KVX_CUDA_TRY(cudaGetLastError(), "kvx_decode_attention");
    kvx::note_launch();
    return KVX_OK;
  }

  if (layout->head_dim % 32 != 0 || layout->head_dim > 256) {
    kvx::set_error("kvx_decode_attention: head_dim must be a multiple of 32 and <= 256");
    return KVX_ERR_UNSUPPORTED;
  }
  if (d_new_k) {
    const int row_bytes = layout->head_dim * (layout->dtype == KVX_DTYPE_BF16 ? 2 : 4);
    kvx::append_from_table<<<batch, 128, 0, st>>>(pool->base, pool->page_bytes, pool->num_pages, d_block_tables,
                                                  d_ctx_lens, static_cast<const uint8_t*>(d_new_k),
                                                  static_cast<const uint8_t*>(d_new_v), H, layout->block_tokens,
                                                  row_bytes, params->max_blocks);
    KVX_CUDA_TRY(cudaGetLastError(), "kvx_decode_attention_append(append)");
    kvx::note_launch();
  }
  dim3 grid(Hq, batch);
  if (layout->dtype == KVX_DTYPE_F32)
    kvx::attn_generic<float><<<grid, 32, 0, st>>>(pool->base, pool->page_bytes, pool->num_pages, d_block_tables, d_ctx_lens,
                                                  static_cast<const float*>(d_q), d_out, H, group, layout->head_dim,
                                                  layout->block_tokens, params->max_blocks, scale);
  else
    kvx::attn_generic<uint16_t><<<grid, 32, 0, st>>>(pool->base, pool->page_bytes, pool->num_pages, d_block_tables, d_ctx_lens,
                                                     static_cast<const uint16_t*>(d_q), d_out, H, group,
                                                     layout->head_dim, layout->block_tokens, params->max_blocks,
                                                     scale);
  KVX_CUDA_TRY(cudaGetLastError(), "kvx_decode_attention(generic)");
  kvx::note_launch();
  return KVX_OK;
}

}  // namespace
}  // namespace kvx

extern "C" {

int kvx_decode_attention(const kvx_pool* pool, const kvx_page_layout* layout, const kvx_attn_params* params,
                         const uint32_t* d_block_tables, const int32_t* d_ctx_lens, const void* d_q, float* d_out,
                         int32_t batch, int32_t max_ctx, void* d_workspace, uint64_t workspace_bytes, void* stream) {
  return kvx::decode_attention(pool, layout, params, d_block_tables, d_ctx_lens, d_q, nullptr, nullptr, d_out, batch,
                               max_ctx, d_workspace, workspace_bytes, stream);
}

int kvx_decode_attention_append(kvx_pool* pool, const kvx_page_layout* layout, const kvx_attn_params* params,
                                const uint32_t* d_block_tables, const int32_t* d_ctx_lens, const void* d_q,
                                const void* d_new_k, const void* d_new_v, float* d_out, int32_t batch,
                                int32_t max_ctx, void* d_workspace, uint64_t workspace_bytes, void* stream) {
  if (!d_new_k || !d_new_v) return kvx::fail_arg("kvx_decode_attention_append: null new K/V");
  if (pool && layout) {
    const int row_bytes = layout->head_dim * (layout->dtype == KVX_DTYPE_BF16 ? 2 : 4);
    if (row_bytes % 16) return kvx::fail_arg("kvx_decode_attention_append: head_dim * sizeof(dtype) must be a multiple of 16");
  }
  return kvx::decode_attention(pool, layout, params, d_block_tables, d_ctx_lens, d_q, d_new_k, d_new_v, d_out, batch,
                               max_ctx, d_workspace, workspace_bytes, stream);
}

}  // extern "C"
