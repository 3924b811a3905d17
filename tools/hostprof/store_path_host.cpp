// Host bookkeeping of the store-path migration of one Llama-3.1-70B @32K
// session (80 layers x 2,048 blocks), as tools/store_path_70b.py runs it on
// the GPU — mark_migrating_out, import_migration, 80 x apply (NetArrive),
// release_session, plan_layerwise_load, 80 x apply (LoadH2D) — but linked
// against tools/hostprof/kvx_stub.cpp instead of libkvx, so the host cost of
// KvStore + NodePayload alone can be timed and profiled (gprof) without a
// GPU. DIAGNOSTIC ONLY. Build + run: tools/hostprof/run.sh
#include <algorithm>
#include <chrono>
#include <cstdio>
#include <cstdlib>
#include <map>
#include <string>
#include <vector>

#include "symsim/payload.hpp"

using namespace symsim;

namespace {
constexpr int kLayers = 80, kBlocks = 2048, kTokens = 32768, kHeads = 8, kDim = 128;
using Clock = std::chrono::steady_clock;
std::map<std::string, double> acc;

template <typename F>
auto timed(const char* name, F&& f) {
  const auto t0 = Clock::now();
  auto r = f();
  acc[name] += std::chrono::duration<double, std::micro>(Clock::now() - t0).count();
  return r;
}

void apply_all(KvStore& st, std::vector<ScheduledTransfer> s, const char* name) {
  std::sort(s.begin(), s.end(), [](const auto& a, const auto& b) {
    return a.complete_at != b.complete_at ? a.complete_at < b.complete_at : a.id < b.id;
  });
  for (const auto& t : s) timed(name, [&] { return st.apply_transfer(t.id, t.complete_at); });
}
}  // namespace

int main(int argc, char** argv) {
  const int reps = argc > 1 ? std::atoi(argv[1]) : 5;
  GpuProfile gpu;
  gpu.kv_bytes_per_token = static_cast<std::int64_t>(kLayers) * 2 * kHeads * kDim * 2;
  gpu.num_layers = kLayers;
  gpu.hbm_capacity = 1'000'000'000'000;
  LinkProfile links;
  links.network_bandwidth = 770e9;
  links.pcie_bandwidth = 55e9;
  PayloadCluster cluster;
  const std::uint64_t pages = static_cast<std::uint64_t>(kLayers) * kBlocks;
  std::vector<std::unique_ptr<KvStore>> stores;
  std::vector<std::unique_ptr<NodePayload>> nodes;
  for (int n = 0; n < 2; ++n) {
    KvStore::Options o;
    o.node_id = n;
    o.write_behind = false;
    o.host_capacity = 1ll << 45;
    stores.push_back(std::make_unique<KvStore>(gpu, links, o));
    PayloadOptions po;
    po.device = 0;
    po.layout = kvx_page_layout{kHeads, kDim, 16, KVX_DTYPE_BF16};
    po.device_pages = pages;
    po.host_pages = 1;
    po.landing_pages = n == 0 ? 1 : pages;
    po.disk_pages = 1;
    po.seed = 0x70B;
    po.free_running = true;
    nodes.push_back(std::make_unique<NodePayload>(&cluster, n, po));
    if (!std::getenv("NOBACKEND")) stores[n]->attach_backend(nodes[n].get());
    for (int r = 0; r < reps; ++r) stores[n]->register_session(r, "s" + std::to_string(r), PriorityClass::Normal);
    stores[n]->finalize_sessions();
  }
  KvStore& src = *stores[0];
  KvStore& dst = *stores[1];
  Ns now = 0;
  for (int r = 0; r < reps; ++r) {
    std::vector<ScheduledTransfer> s;
    src.append_blocks(r, kTokens, now, s);
    apply_all(src, s, "apply(created)");
    timed("mark_migrating_out", [&] { src.mark_migrating_out(r); return 0; });
    auto imp = timed("import_migration", [&] { return dst.import_migration(r, kTokens, now + 1'000'000); });
    apply_all(dst, imp, "apply(net_arrive)");
    timed("release_session", [&] { src.release_session(r, now + 100'000'000); return 0; });
    std::vector<ScheduledTransfer> l;
    timed("plan_layerwise_load",
          [&] { return dst.plan_layerwise_load(r, now + 200'000'000, 100'000, TransferReason::Demand, l); });
    apply_all(dst, l, "apply(load_h2d)");
    dst.release_session(r, now + 300'000'000);
    now += 1'000'000'000;
  }
  double total = 0;
  for (const char* k : {"import_migration", "apply(net_arrive)", "plan_layerwise_load", "apply(load_h2d)"}) {
    const double us = acc[k] / reps / kLayers;
    total += us;
    std::printf("%-22s %8.2f us/layer\n", k, us);
  }
  std::printf("%-22s %8.2f us/layer (host, no GPU)\n", "migration total", total);
  static const char* kPhase[] = {"posted", "retired", "issue", "reclaim", "upload", "launch", "close", "alloc"};
  for (int n = 0; n < 2; ++n) {
    std::printf("node%d:", n);
    for (int k = 0; k < NodePayload::kHostPhases; ++k)
      std::printf(" %s %.1f", kPhase[k], nodes[n]->host_ns()[k] / 1e3 / reps / kLayers);
    std::printf(" us/layer\n");
  }
  return 0;
}
