// Host-side cost of the store's migration / load bookkeeping at the bench
// shapes, product vs reference (both through the kvs ABI). Measurement tool.
// usage: store_ops_bench <product.so> <oracle.so>
#include <chrono>
#include <cstdio>
#include <vector>

#include "kvs_dyn.hpp"

namespace {
double us_since(std::chrono::steady_clock::time_point t0) {
  return std::chrono::duration<double, std::micro>(std::chrono::steady_clock::now() - t0).count();
}

void run(KvsApi& A, const char* name, int layers, int tokens) {
  kvs_gpu_profile gpu{8192.0, 12.0, 16.0, 180'000'000'000, static_cast<int64_t>(layers) * 4096, layers, 0, nullptr, nullptr};
  kvs_link_profile links{55e9, 3e9, 770e9, 10'000};
  kvs_options opts{0, 16, 0, 1'000'000'000'000LL, -1, 1};
  const int reps = 20;
  double t_append = 0, t_import = 0, t_apply = 0, t_plan = 0, t_purge = 0, t_release = 0;
  for (int r = 0; r < reps; ++r) {
    kvs_store* s = nullptr;
    A.kvs_create(&gpu, &links, &opts, &s);
    A.kvs_register_session(s, 0, "a", 0);
    A.kvs_register_session(s, 1, "b", 0);
    A.kvs_finalize_sessions(s);
    auto t0 = std::chrono::steady_clock::now();
    A.kvs_append_blocks(s, 0, tokens, 0);
    t_append += us_since(t0);
    const kvs_scheduled* x;
    size_t n = A.kvs_out_scheduled(s, &x);
    std::vector<kvs_scheduled> pend(x, x + n);
    for (auto& p : pend) {
      kvs_apply_result ar;
      A.kvs_apply_transfer(s, p.id, p.complete_at, &ar);
    }
    t0 = std::chrono::steady_clock::now();
    A.kvs_import_migration(s, 1, tokens, 1'000'000'000);
    t_import += us_since(t0);
    n = A.kvs_out_scheduled(s, &x);
    pend.assign(x, x + n);
    t0 = std::chrono::steady_clock::now();
    for (auto& p : pend) {
      kvs_apply_result ar;
      A.kvs_apply_transfer(s, p.id, p.complete_at, &ar);
    }
    t_apply += us_since(t0);
    int64_t freed = 0;
    t0 = std::chrono::steady_clock::now();
    A.kvs_purge_from_device(s, 1LL << 50, 2'000'000'000, 0, &freed);
    t_purge += us_since(t0);
    kvs_load_plan plan;
    t0 = std::chrono::steady_clock::now();
    A.kvs_plan_layerwise_load(s, 1, 3'000'000'000, 100'000, 1, &plan);
    t_plan += us_since(t0);
    t0 = std::chrono::steady_clock::now();
    A.kvs_release_session(s, 0, 4'000'000'000);
    t_release += us_since(t0);
    A.kvs_destroy(s);
  }
  std::printf("%-9s L=%d tokens=%d  append %.1f  import %.1f  apply_arrivals %.1f  purge_all %.1f  plan_load %.1f  release %.1f us\n",
              name, layers, tokens, t_append / reps, t_import / reps, t_apply / reps, t_purge / reps, t_plan / reps,
              t_release / reps);
}
}  // namespace

int main(int argc, char** argv) {
  if (argc < 3) return 2;
  KvsApi P(argv[1]), R(argv[2]);
  for (auto [L, T] : {std::pair<int, int>{32, 8192}, {80, 32768}}) {
    run(P, "b200", L, T);
    run(R, "reference", L, T);
  }
  return 0;
}
