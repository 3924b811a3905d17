// K4 timeline tracer: builds the decode-attention kernel with per-CTA
// %globaltimer stamps (KVX_ATTN_TRACE) and prints where one launch's time
// goes — launch/PDL wait, block-table staging, first page, page loop,
// CTA combine, split-K merge. Diagnostic only; not part of the product.
//
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 -Iinclude \
//     tools/attn_trace.cu paper_2412_16434_b200/csrc/kernels/kvx_pool.cu \
//     paper_2412_16434_b200/csrc/kernels/kvx_copy.cu -lcuda -o build/attn_trace
//   build/attn_trace BATCH CTX [SPLITS [MERGE [Q_HEADS [FLAGS]]]]   (Q_HEADS 32: Llama-3.1-8B, 64: 70B; FLAGS 1 = early prefetch)
#include <cstdint>
__device__ unsigned long long kvx_attn_trace[32 * 65536];
#define KVX_ATTN_TRACE 1
#include "../paper_2412_16434_b200/csrc/kernels/kvx_attn.cu"

#include <algorithm>
#include <cstdio>
#include <cstdlib>
#include <numeric>
#include <random>
#include <vector>

#define CK(x)                                                                  \
  do {                                                                         \
    int rc_ = (x);                                                             \
    if (rc_) {                                                                 \
      fprintf(stderr, "%s:%d %s -> %d %s\n", __FILE__, __LINE__, #x, rc_, kvx_last_error()); \
      exit(1);                                                                 \
    }                                                                          \
  } while (0)

static double pct(std::vector<double> v, double p) {
  if (v.empty()) return 0;
  std::sort(v.begin(), v.end());
  return v[std::min(v.size() - 1, static_cast<size_t>(p * (v.size() - 1) + 0.5))];
}

int main(int argc, char** argv) {
  const int batch = argc > 1 ? atoi(argv[1]) : 1;
  const int ctx = argc > 2 ? atoi(argv[2]) : 8192;
  const int splits_req = argc > 3 ? atoi(argv[3]) : 0;
  const int merge = argc > 4 ? atoi(argv[4]) : KVX_MERGE_AUTO;
  const int H = 8, Hq = argc > 5 ? atoi(argv[5]) : 32, D = 128, T = 16;
  kvx_page_layout lay{H, D, T, KVX_DTYPE_BF16};
  const uint64_t pb = kvx_page_bytes(&lay);
  const int blocks = (ctx + T - 1) / T;
  const uint64_t per_set = static_cast<uint64_t>(batch) * blocks;
  // rotate over enough request sets that each launch reads cold HBM (> L2)
  int sets = static_cast<int>(std::max<uint64_t>(2, (512ull << 20) / (per_set * pb) + 1));
  const uint64_t pages = per_set * sets;
  kvx_pool* pool;
  CK(kvx_pool_create(0, pages, pb, &pool));
  cudaMemset(kvx_pool_base(pool), 0x3c, pages * pb);
  std::mt19937 rng(7);
  std::vector<uint32_t> ids(pages);
  std::iota(ids.begin(), ids.end(), 0u);
  if (!getenv("KVX_TRACE_SEQUENTIAL")) std::shuffle(ids.begin(), ids.end(), rng);  // sequential: pages in table order
  uint32_t* d_tables;
  cudaMalloc(&d_tables, pages * 4);
  cudaMemcpy(d_tables, ids.data(), pages * 4, cudaMemcpyHostToDevice);
  std::vector<int32_t> lens(batch, ctx);
  int32_t* d_lens;
  cudaMalloc(&d_lens, batch * 4);
  cudaMemcpy(d_lens, lens.data(), batch * 4, cudaMemcpyHostToDevice);
  std::vector<uint16_t> q(static_cast<size_t>(batch) * Hq * D);
  for (auto& x : q) x = 0x3C00 | (rng() & 0x7F);
  uint16_t* d_q;
  cudaMalloc(&d_q, q.size() * 2);
  cudaMemcpy(d_q, q.data(), q.size() * 2, cudaMemcpyHostToDevice);
  float* d_out;
  cudaMalloc(&d_out, q.size() * 4);
  const int flags = argc > 6 ? atoi(argv[6]) : 0;  // KVX_ATTN_* (1 = early prefetch)
  kvx_attn_params prm{Hq, blocks, splits_req, 0.f, merge, flags};
  const uint64_t ws_bytes = std::max<uint64_t>(16, kvx_decode_attention_workspace(&lay, &prm, batch, ctx));
  void* d_ws;
  cudaMalloc(&d_ws, ws_bytes);
  cudaMemset(d_ws, 0, ws_bytes);
  cudaStream_t st;
  cudaStreamCreateWithFlags(&st, cudaStreamNonBlocking);
  auto launch = [&](int i) {
    CK(kvx_decode_attention(pool, &lay, &prm, d_tables + (i % sets) * per_set, d_lens, d_q, d_out, batch, ctx, d_ws,
                            ws_bytes, st));
  };
  for (int i = 0; i < 20; ++i) launch(i);
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0);
  cudaEventCreate(&e1);
  const int iters = 200;
  cudaEventRecord(e0, st);
  for (int i = 0; i < iters; ++i) launch(i);
  cudaEventRecord(e1, st);
  cudaEventSynchronize(e1);
  float ms;
  cudaEventElapsedTime(&ms, e0, e1);
  const double us_launch = ms * 1e3 / iters;
  // the same launches replayed from a CUDA graph (one node per launch)
  cudaGraph_t graph;
  cudaGraphExec_t exec;
  const int graph_n = 2 * sets > 32 ? 2 * sets : 32;
  cudaStreamBeginCapture(st, cudaStreamCaptureModeThreadLocal);
  for (int i = 0; i < graph_n; ++i) launch(i);
  cudaStreamEndCapture(st, &graph);
  cudaGraphInstantiate(&exec, graph, 0);
  cudaGraphLaunch(exec, st);
  cudaEventRecord(e0, st);
  for (int r = 0; r < 5; ++r) cudaGraphLaunch(exec, st);
  cudaEventRecord(e1, st);
  cudaEventSynchronize(e1);
  cudaEventElapsedTime(&ms, e0, e1);
  const double us_graph = ms * 1e3 / (5 * graph_n);
  // one isolated, traced launch (idle GPU before it)
  cudaStreamSynchronize(st);
  launch(iters + 1);
  cudaStreamSynchronize(st);
  const char* tma_env = getenv("KVX_ATTN_TMA");
  const kvx::Plan plan = kvx::plan_attention(batch, H, ctx, splits_req, merge, 0, !(tma_env && tma_env[0] == '0'), (flags >> 8) & 0xF);
  const int splits = plan.splits;
  const int ctas = splits * H * batch;
  std::vector<unsigned long long> tr(static_cast<size_t>(ctas) * 32);
  cudaMemcpyFromSymbol(tr.data(), kvx_attn_trace, tr.size() * 8);
  if (cudaGetLastError() != cudaSuccess) { fprintf(stderr, "cuda error\n"); return 1; }
  unsigned long long t0 = ~0ull, tend = 0;
  for (int c = 0; c < ctas; ++c) {
    t0 = std::min(t0, tr[c * 32 + 0]);
    tend = std::max(tend, std::max(tr[c * 32 + 5], tr[c * 32 + 6]));
  }
  std::vector<double> start, wait, table, first, loop, combine, mergev;
  std::vector<double> warp_skew, last_warp, push, fence, mwait, mlocal;
  std::vector<int> sm_use(256, 0);
  const int W = plan.narrow ? kvx::kNarrowW : 4;
  for (int c = 0; c < ctas; ++c) {
    const unsigned long long* r = &tr[c * 32];
    start.push_back((r[0] - t0) * 1e-3);
    wait.push_back((r[1] - r[0]) * 1e-3);
    table.push_back((r[2] - r[1]) * 1e-3);
    first.push_back((r[3] - r[2]) * 1e-3);
    loop.push_back((r[4] - r[3]) * 1e-3);
    combine.push_back((r[5] - r[4]) * 1e-3);
    if (r[6] > r[5]) mergev.push_back((r[6] - r[5]) * 1e-3);
    sm_use[r[31] & 255]++;
    unsigned long long wmin = ~0ull, wmax = 0;
    for (int w = 0; w < W; ++w) {
      wmin = std::min(wmin, r[16 + w]);
      wmax = std::max(wmax, r[16 + w]);
    }
    warp_skew.push_back((wmax - wmin) * 1e-3);           // first to last warp out of the page loop
    last_warp.push_back((r[8] - wmax) * 1e-3 + 0.0);      // last warp out -> CTA barrier passed
    push.push_back((r[5] - r[8]) * 1e-3);                 // smem combine + row weights + st.async pushes
    if (r[10] > r[5]) {
      mwait.push_back((r[10] - r[5]) * 1e-3);             // wait for every split's partial bytes
      mlocal.push_back((r[6] - r[10]) * 1e-3);            // local merge + output stores
    }
  }
  int sms_used = 0, max_per_sm = 0;
  for (int v : sm_use) { sms_used += v > 0; max_per_sm = std::max(max_per_sm, v); }
  const double bytes = static_cast<double>(batch) * ctx * H * D * 2 * 2;
  printf("{\"hq\": %d, \"batch\": %d, \"ctx\": %d, \"splits\": %d, \"cluster\": %d, \"ctas\": %d, \"sms_used\": %d, \"max_ctas_per_sm\": %d, "
         "\"us_per_launch\": %.2f, \"us_graph\": %.2f, \"gbs\": %.0f, \"traced_span_us\": %.2f}\n",
         Hq, batch, ctx, splits, plan.cluster ? 1 : 0, ctas, sms_used, max_per_sm, us_launch, us_graph, bytes / us_launch * 1e-3, (tend - t0) * 1e-3);
  auto row = [](const char* n, const std::vector<double>& v) {
    printf("  %-10s p0 %7.2f  p50 %7.2f  p90 %7.2f  max %7.2f us\n", n, pct(v, 0), pct(v, .5), pct(v, .9), pct(v, 1));
  };
  row("start", start);
  row("pdl_wait", wait);
  row("table", table);
  row("1st_page", first);
  row("loop", loop);
  row("combine", combine);
  row("merge", mergev);
  row("warp_skew", warp_skew);
  row("last->bar", last_warp);
  row("push", push);
  row("mbar_wait", mwait);
  row("merge_loc", mlocal);
  return 0;
}
