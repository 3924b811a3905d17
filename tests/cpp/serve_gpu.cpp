// Configs 4 and 5 served on the B200: the reference's UNCHANGED cluster
// simulator (Simulation, NodeManager, ClusterScheduler, workload / report,
// compiled from /root/reference) driving this repo's KvStore + NodePayload +
// Engine, with every engine quantum EXECUTED on the GPU (GpuStepExecutor:
// a Llama-3.1-8B-shaped decode step with K4 over the pages each node's
// payload holds; prefill's dense work) and lasting its measured duration.
// MEASUREMENT INFRASTRUCTURE, built by tests/cpp/build_serve_gpu.sh into
// oracle/_ref/serve_gpu (it links reference sources, so it is built here and
// shipped prebuilt).
//
// All nodes share the one GPU of the box (each node = one Symphony GPU, its
// own pools and streams): a node's decode step runs alone on the device and
// is timed alone (the engine loop is sequential), migration / load / persist
// moves of every node run concurrently on their lanes. So a node's quanta
// are what one B200 takes for its batch, except that other nodes' data
// movement shares the device (contention the real 8-GPU box would not have
// for moves between other GPUs).
//
// Per run it prints one JSON line: policy, load, requests, steady req/s
// (reference steady_rps), p50 / p90 TTFT, TPOT and normalized latency
// (product traffic::latency_stats), migrations, the executed quanta (steps,
// mean / p50 step ms, batch, gated layers), and — with --verify-every K —
// every page the K-th decode steps attended, scrubbed against its oracle
// content (kvx_verify_block_tables), plus all pages of every node at the end.
//
// usage: serve_gpu --config 4|5 --policies a,b --users u1,u2 [--sessions S] [--nodes N]
//                  [--think-s T] [--wpm W] [--device-gb G] [--host-gb H] [--disk-dir D]
//                  [--verify-every K] [--seed X] [--calibrate-only]

#include <algorithm>
#include <chrono>
#include <cinttypes>
#include <cmath>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <memory>
#include <string>
#include <vector>

#include "symsim/payload.hpp"
#include "symsim/simcore.hpp"
#include "symsim/step_executor.hpp"
#include "symsim/traffic.hpp"

using namespace symsim;

namespace {

struct Args {
  int config = 5;
  std::vector<std::string> policies{"symphony"};
  std::vector<int> users{64};
  int sessions = 0;
  int nodes = 4;
  double think_s = 1.0;
  double wpm = 4000.0;
  double device_gb = 16.0, host_gb = 8.0;
  std::string disk_dir;
  int verify_every = 0;
  std::uint64_t seed = 0;
  bool calibrate_only = false;
  int profile_batch = 0;   // --profile-batch B: only time decode steps at batch B (ncu / nsys target)
  int profile_steps = 20;
  int profile_ctx = 1024;
  int max_batch = 64;
};

std::vector<std::string> split(const std::string& s) {
  std::vector<std::string> out;
  std::size_t pos = 0;
  while (pos <= s.size()) {
    const std::size_t c = s.find(',', pos);
    out.push_back(s.substr(pos, c == std::string::npos ? std::string::npos : c - pos));
    if (c == std::string::npos) break;
    pos = c + 1;
  }
  return out;
}

Ns typing(std::int64_t words, double wpm) { return ns_from_sec(static_cast<double>(words) * 60.0 / wpm); }

void poisson_think(Trace& t, double mean_s, std::uint64_t seed) {
  std::size_t n = 0;
  for (const auto& e : t.events) n += e.kind == EventKind::Inference && e.turn_index != 0;
  const std::vector<Ns> gaps = traffic::poisson_gaps(n, mean_s, seed);
  std::size_t k = 0;
  for (auto& e : t.events) {
    if (e.kind != EventKind::Inference || e.turn_index == 0) continue;
    const auto& s = t.sessions[e.session_index];
    e.delta = gaps[k++] + typing(s.turns[e.turn_index].prompt_words, s.user.typing_wpm);
  }
}

// Config 4: ShareGPT-like corpus (reference synthesize_corpus defaults),
// Poisson turns. Config 5: all multi-turn, Zipf(1.2) popularity -> turns.
Trace make_trace(const Args& a, int users) {
  SyntheticSpec spec;
  const std::uint64_t seed = a.config == 5 ? 505 + a.seed : 404 + a.seed;
  if (a.config == 5) {
    spec.sessions = a.sessions > 0 ? a.sessions : 600;
    spec.multi_turn_fraction = 1.0;
  } else if (a.sessions > 0) {
    spec.sessions = a.sessions;
  }
  auto scripts = synthesize_corpus(spec, seed);
  if (a.config == 5) {
    const std::vector<int> want = traffic::zipf_turns(scripts.size(), 1.2, 64.0, 2, seed + 7);
    for (std::size_t i = 0; i < scripts.size(); ++i) {
      std::vector<Turn> turns;
      for (int k = 0; k < want[i]; ++k) turns.push_back(scripts[i].turns[static_cast<std::size_t>(k) % scripts[i].turns.size()]);
      scripts[i].turns = std::move(turns);
    }
  }
  SpeedModel speeds;
  speeds.typing_wpm_mean = a.wpm;
  Trace t = synthesize_arrivals(std::move(scripts), users, seed + 1, speeds);
  poisson_think(t, a.think_s, seed + 2);
  return inject_advisories(std::move(t), 0.0, seed + 3);
}

constexpr int kLayers = 32, kHeads = 8, kDim = 128;
constexpr std::int64_t kPageBytes = 2LL * kHeads * 16 * kDim * 2;  // 64 KiB
constexpr std::int64_t kBytesPerToken = static_cast<std::int64_t>(kLayers) * 2 * kHeads * kDim * 2;

PayloadOptions node_options(const Args& a, int node_id, std::uint64_t device_pages, std::uint64_t host_pages) {
  PayloadOptions o;
  o.device = 0;
  o.layout = kvx_page_layout{kHeads, kDim, 16, KVX_DTYPE_BF16};
  o.device_pages = device_pages;
  o.host_pages = host_pages;
  o.landing_pages = host_pages;
  o.disk_pages = a.disk_dir.empty() ? host_pages * 4 : (std::uint64_t{1} << 29) / 64;  // files: 32 GiB sparse
  if (!a.disk_dir.empty()) o.disk_path = a.disk_dir + "/node" + std::to_string(node_id) + ".pages";
  o.seed = 0x5EEDBA5Eull;  // one content function for every node: migrated pages stay checkable
  o.fill_mode = KVX_FILL_VALUES;
  o.free_running = true;
  return o;
}

// Measured decode curve (batch -> ms) and prefill throughput of the model on
// this GPU, for the engine's planning estimates (step_estimate, pause
// budget, layer-wise load plans); the quanta themselves are measured.
struct Calibration {
  std::vector<std::pair<int, double>> curve;
  double prefill_tps = 0;
};

Calibration calibrate(ModelRuntime& rt, int ctx, int only_batch = 0, int reps = 5) {
  Calibration cal;
  std::vector<int> batches = {1, 2, 4, 8, 16, 32, 64};
  if (only_batch > 0) batches = {only_batch};
  const int sessions = std::max(64, only_batch);
  GpuProfile gpu;
  gpu.kv_bytes_per_token = kBytesPerToken;
  gpu.num_layers = kLayers;
  gpu.hbm_capacity = static_cast<std::int64_t>(sessions) * (ctx + 64) * kBytesPerToken * 2;
  KvStore::Options ko;
  ko.write_behind = false;
  KvStore store(gpu, LinkProfile{}, ko);
  PayloadCluster cluster;
  Args a;
  const std::uint64_t pages = static_cast<std::uint64_t>(sessions) * kLayers * ((ctx + 64) / 16 + 2);
  NodePayload node(&cluster, 0, node_options(a, 0, pages, 16));
  store.attach_backend(&node);
  for (int s = 0; s < sessions; ++s) store.register_session(s, "cal" + std::to_string(s), PriorityClass::Normal);
  store.finalize_sessions();
  for (int s = 0; s < sessions; ++s) {
    std::vector<ScheduledTransfer> x;
    store.append_blocks(s, ctx, 0, x);
  }
  node.synchronize();
  GpuStepExecutor exec(rt, node);
  for (int b : batches) {
    std::vector<StepExecutor::Row> rows;
    for (int i = 0; i < b; ++i) rows.push_back({static_cast<std::uint32_t>(i), ctx});
    std::vector<double> ms;
    for (int rep = 0; rep < reps; ++rep) ms.push_back(to_ms(exec.decode_step(rows)));
    cal.curve.emplace_back(b, traffic::percentile(ms, 0.5));
  }
  if (only_batch > 0) return cal;
  double tps = 0;
  for (int tokens : {512, 2048}) {
    std::vector<double> ns;
    for (int rep = 0; rep < 3; ++rep) ns.push_back(static_cast<double>(exec.prefill(0, tokens)));
    tps += tokens / (traffic::percentile(ns, 0.5) * 1e-9) / 2;
  }
  cal.prefill_tps = tps;
  return cal;
}

std::string json_stats(const traffic::LatencyStats& s) {
  char buf[160];
  std::snprintf(buf, sizeof buf, "{\"p50\": %.6g, \"p90\": %.6g, \"p99\": %.6g, \"mean\": %.6g}", s.p50, s.p90, s.p99,
                s.mean);
  return buf;
}

}  // namespace

int main(int argc, char** argv) {
  Args a;
  for (int i = 1; i < argc; ++i) {
    const std::string k = argv[i];
    auto next = [&]() -> std::string { return i + 1 < argc ? argv[++i] : ""; };
    if (k == "--config") a.config = std::atoi(next().c_str());
    else if (k == "--policies") a.policies = split(next());
    else if (k == "--users") {
      a.users.clear();
      for (const auto& u : split(next())) a.users.push_back(std::atoi(u.c_str()));
    } else if (k == "--sessions") a.sessions = std::atoi(next().c_str());
    else if (k == "--nodes") a.nodes = std::atoi(next().c_str());
    else if (k == "--think-s") a.think_s = std::atof(next().c_str());
    else if (k == "--wpm") a.wpm = std::atof(next().c_str());
    else if (k == "--device-gb") a.device_gb = std::atof(next().c_str());
    else if (k == "--host-gb") a.host_gb = std::atof(next().c_str());
    else if (k == "--disk-dir") a.disk_dir = next();
    else if (k == "--verify-every") a.verify_every = std::atoi(next().c_str());
    else if (k == "--seed") a.seed = std::strtoull(next().c_str(), nullptr, 10);
    else if (k == "--max-batch") a.max_batch = std::atoi(next().c_str());
    else if (k == "--calibrate-only") a.calibrate_only = true;
    else if (k == "--profile-batch") a.profile_batch = std::atoi(next().c_str());
    else if (k == "--profile-steps") a.profile_steps = std::atoi(next().c_str());
    else if (k == "--profile-ctx") a.profile_ctx = std::atoi(next().c_str());
  }
  const auto t_start = std::chrono::steady_clock::now();
  ModelRuntime rt(0, llama31_8b_config(), 0x8B8B8Bull);
  if (a.profile_batch > 0) {  // profiling target: decode steps only
    const Calibration p = calibrate(rt, a.profile_ctx, a.profile_batch, a.profile_steps);
    std::printf("{\"profile\": {\"batch\": %d, \"ctx\": %d, \"steps\": %d, \"decode_ms_p50\": %.4f}}\n",
                a.profile_batch, a.profile_ctx, a.profile_steps, p.curve[0].second);
    return 0;
  }
  const Calibration cal = calibrate(rt, 1024);
  std::printf("{\"calibration\": {\"model\": \"llama-3.1-8b shape, random bf16 weights\", \"ctx\": 1024, "
              "\"decode_curve_ms\": [");
  for (std::size_t i = 0; i < cal.curve.size(); ++i)
    std::printf("%s[%d, %.4f]", i ? ", " : "", cal.curve[i].first, cal.curve[i].second);
  std::printf("], \"prefill_tokens_per_s\": %.1f}}\n", cal.prefill_tps);
  std::fflush(stdout);
  if (a.calibrate_only) return 0;

  const std::uint64_t device_pages = static_cast<std::uint64_t>(a.device_gb * 1e9 / kPageBytes) + 4096;
  const std::uint64_t host_pages = static_cast<std::uint64_t>(a.host_gb * 1e9 / kPageBytes) + 1024;
  for (const std::string& pol : a.policies)
    for (int users : a.users) {
      const Trace trace = make_trace(a, users);
      RunConfig cfg;
      cfg.policy = policy_from(pol);
      cfg.num_nodes = a.nodes;
      cfg.gpu.kv_bytes_per_token = kBytesPerToken;
      cfg.gpu.num_layers = kLayers;
      cfg.gpu.hbm_capacity = static_cast<std::int64_t>(a.device_gb * 1e9);
      cfg.gpu.prefill_throughput = cal.prefill_tps;
      cfg.gpu.decode_curve_ms = cal.curve;
      cfg.host_capacity = static_cast<std::int64_t>(a.host_gb * 1e9);
      cfg.links.pcie_bandwidth = 55e9;        // measured (profiles/calibration_r01.json)
      cfg.links.network_bandwidth = 770e9;    // measured peer copy (B200_PROFILING.md)
      cfg.engine.max_batch = a.max_batch;
      cfg.sample_period = ns_from_sec(5);
      cfg.invariant_stride = 4096;

      PayloadCluster cluster;
      std::vector<std::unique_ptr<NodePayload>> payloads;
      std::vector<std::unique_ptr<GpuStepExecutor>> execs;
      set_default_tier_backend_factory([&](int node_id) -> TierBackend* {
        payloads.push_back(std::make_unique<NodePayload>(&cluster, node_id, node_options(a, node_id, device_pages,
                                                                                           host_pages)));
        return payloads.back().get();
      });
      set_default_step_executor_factory([&](KvStore& st) -> StepExecutor* {
        auto* np = dynamic_cast<NodePayload*>(st.backend());
        if (!np) throw std::runtime_error("serve_gpu: engine without a payload node");
        execs.push_back(std::make_unique<GpuStepExecutor>(rt, *np));
        execs.back()->verify_every(a.verify_every);
        return execs.back().get();
      });
      const auto t0 = std::chrono::steady_clock::now();
      RunReport rep;
      std::string error;
      try {
        rep = run_simulation(trace, cfg);
      } catch (const std::exception& e) {
        error = e.what();
      }
      const double wall_s = std::chrono::duration<double>(std::chrono::steady_clock::now() - t0).count();
      set_default_tier_backend_factory(nullptr);
      set_default_step_executor_factory(nullptr);
      for (auto& p : payloads) p->synchronize();
      if (!error.empty()) {
        std::printf("{\"config\": %d, \"policy\": \"%s\", \"users\": %d, \"error\": \"%s\"}\n", a.config, pol.c_str(),
                    users, error.substr(0, 300).c_str());
        std::fflush(stdout);
        execs.clear();
        payloads.clear();
        continue;
      }
      std::vector<double> ttft, tpot, norm;
      for (const auto& r : rep.records) {
        ttft.push_back(r.ttft_s() * 1e3);
        tpot.push_back(r.tpot_ms());
        norm.push_back(r.normalized_latency_ms_per_token());
      }
      std::int64_t mig_bytes = 0, mig_rows = 0;
      for (const auto& t : rep.transfers)
        if (t.reason == TransferReason::Migrate) {
          mig_bytes += t.bytes;
          ++mig_rows;
        }
      std::int64_t steps = 0, step_ns = 0, prefills = 0, prefill_ns = 0, gated = 0, attended = 0, max_b = 0,
                   table_ns = 0, rows = 0;
      std::vector<double> all_steps;
      std::uint64_t verified = 0, mismatched = 0;
      for (auto& e : execs) {
        const auto& s = e->stats();
        steps += s.steps;
        step_ns += s.step_ns;
        prefills += s.prefills;
        prefill_ns += s.prefill_ns;
        gated += s.gated_layers;
        attended += s.attended_tokens;
        rows += s.rows;
        max_b = std::max(max_b, s.max_batch);
        table_ns += s.host_table_ns;
        verified += e->verified_pages();
        mismatched += e->mismatched_pages();
      }
      std::uint64_t apply_wait = 0, moved_net = 0;
      for (auto& p : payloads) {
        apply_wait += p->apply_wait_ns();
        moved_net += p->bytes_moved()[static_cast<int>(BlockEvent::NetArrive)];
      }
      std::printf(
          "{\"config\": %d, \"policy\": \"%s\", \"users\": %d, \"sessions\": %zu, \"nodes\": %d, \"requests\": %zu, "
          "\"steady_rps\": %.4f, \"ttft_ms\": %s, \"tpot_ms\": %s, \"norm_latency_ms_per_token\": %s, "
          "\"makespan_s\": %.3f, \"migrations\": {\"ledger_rows\": %" PRId64 ", \"bytes\": %" PRId64
          ", \"net_arrive_bytes_moved\": %" PRIu64 "}, "
          "\"executed\": {\"decode_steps\": %" PRId64 ", \"decode_ms_mean\": %.4f, \"tokens_per_step\": %.2f, "
          "\"max_batch\": %" PRId64 ", \"attended_ctx_mean\": %.1f, \"gated_layer_launches\": %" PRId64
          ", \"prefills\": %" PRId64 ", \"prefill_ms_mean\": %.4f, \"host_table_us_per_step\": %.2f}, "
          "\"verify\": {\"every\": %d, \"pages\": %" PRIu64 ", \"mismatched\": %" PRIu64 "}, "
          "\"payload_apply_wait_ms\": %.3f, \"wall_s\": %.1f}\n",
          a.config, pol.c_str(), users, trace.sessions.size(), a.nodes, rep.records.size(), steady_rps(rep),
          json_stats(traffic::latency_stats(ttft)).c_str(), json_stats(traffic::latency_stats(tpot)).c_str(),
          json_stats(traffic::latency_stats(norm)).c_str(), to_sec(rep.makespan), mig_rows, mig_bytes, moved_net, steps,
          steps ? step_ns / 1e6 / steps : 0.0, steps ? static_cast<double>(rows) / steps : 0.0, max_b,
          rows ? static_cast<double>(attended) / rows : 0.0, gated, prefills,
          prefills ? prefill_ns / 1e6 / prefills : 0.0, steps ? table_ns / 1e3 / steps : 0.0, a.verify_every, verified,
          mismatched, apply_wait / 1e6, wall_s);
      std::fflush(stdout);
      execs.clear();
      payloads.clear();
    }
  std::fprintf(stderr, "serve_gpu: total %.1f s\n",
               std::chrono::duration<double>(std::chrono::steady_clock::now() - t_start).count());
  return 0;
}
