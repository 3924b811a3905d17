// Configs 4 and 5 through the reference's UNCHANGED cluster simulator.
// TEST / MEASUREMENT INFRASTRUCTURE, built by tests/cpp/build_serve_sim.sh
// into oracle/_ref/ (it links the reference's Simulation, Engine,
// NodeManager, ClusterScheduler and workload generators compiled from
// /root/reference). Two builds of this file:
//   serve_sim      this repo's KvStore + cost model + Engine
//   serve_sim_ref  the reference KvStore + cost model
//
// Modes:
//   digest   run one (config, policy, users) cell and print a digest of the
//            whole run (every ledger row and request record, hashed, plus
//            totals). The two builds must print identical digests: state
//            parity at serving scale (1,000 sessions, 8 nodes).
//   sweep    the calibrated serving metric of BASELINE.json ("requests/s at
//            equal p50 latency"): for each policy, sweep concurrent users,
//            report steady requests/s (reference steady_rps, middle 80%) and
//            p50 TPOT; then requests/s at the highest load meeting a common
//            p50-TPOT SLO. The GPU profile is calibrated from B200
//            measurements passed on the command line (--decode-curve,
//            --network-gbs, --pcie-gbs); see DESIGN.md §6.
//
// Trace generators (new; the reference has neither), built on
// the product module include/symsim/traffic.hpp (Poisson gaps, Zipf turns,
// percentiles):
//   config 4  ShareGPT-like corpus (reference synthesize_corpus defaults:
//             1,000 sessions, 73.4% multi-turn, lognormal lengths), Poisson
//             turns: think time ~ Exp(mean) + the reference's typing time, so
//             inject_advisories (reference) can place each advisory exactly
//             at the end of the think pause; advisory miss 0 or 0.1.
//   config 5  load-imbalance stress: session popularity ~ Zipf(1.2) mapped
//             to turns per session; the hottest sessions dominate arrivals.
//
// usage: serve_sim digest <4|5> <policy> <users> [miss] [calibration flags]
//        serve_sim sweep  <4|5> [calibration flags]

#include <algorithm>
#include <cinttypes>
#include <cmath>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <random>
#include <string>
#include <vector>

#include "symsim/simcore.hpp"
#include "symsim/traffic.hpp"

using namespace symsim;

namespace {

std::uint64_t fnv(std::uint64_t h, std::uint64_t v) {
  for (int i = 0; i < 8; ++i) {
    h ^= (v >> (8 * i)) & 0xFF;
    h *= 1099511628211ULL;
  }
  return h;
}

Ns think_ns_like_reference(std::int64_t words, double wpm) {
  // same rounding as the reference's think_ns (workload.cpp): words / wpm min
  return ns_from_sec(static_cast<double>(words) * 60.0 / wpm);
}

int g_sessions = 0;           // --sessions override (0: config default)
double g_typing_wpm = 40.0;   // --typing-wpm (reference SpeedModel default 40)

// Poisson turns: each follow-up prompt arrives an Exp(mean) think time plus
// the reference's typing time after the previous turn completed.
void add_poisson_think(Trace& t, double mean_think_s, std::uint64_t seed) {
  std::size_t n = 0;
  for (const auto& e : t.events) n += e.kind == EventKind::Inference && e.turn_index != 0;
  const std::vector<Ns> gaps = traffic::poisson_gaps(n, mean_think_s, seed);
  std::size_t k = 0;
  for (auto& e : t.events) {
    if (e.kind != EventKind::Inference || e.turn_index == 0) continue;
    const auto& s = t.sessions[e.session_index];
    e.delta = gaps[k++] + think_ns_like_reference(s.turns[e.turn_index].prompt_words, s.user.typing_wpm);
  }
}

Trace config4(int users, double miss, double mean_think_s, std::uint64_t seed) {
  SyntheticSpec spec;  // reference defaults: 1000 sessions, 73.4% multi-turn
  if (g_sessions > 0) spec.sessions = g_sessions;
  auto scripts = synthesize_corpus(spec, seed);
  SpeedModel speeds;
  speeds.typing_wpm_mean = g_typing_wpm;
  Trace t = synthesize_arrivals(std::move(scripts), users, seed + 1, speeds);
  add_poisson_think(t, mean_think_s, seed + 2);
  return inject_advisories(std::move(t), miss, seed + 3);
}

Trace config5(int users, double miss, double mean_think_s, std::uint64_t seed) {
  SyntheticSpec spec;
  spec.sessions = g_sessions > 0 ? g_sessions : 600;
  spec.multi_turn_fraction = 1.0;
  auto scripts = synthesize_corpus(spec, seed);
  // Zipf(1.2) popularity over a seeded ranking of sessions: rank r gets
  // turns ~ 64 / r^1.2 (at least 2), drawn from the session's own turn list
  // (cycled when it is shorter).
  const std::vector<int> want = traffic::zipf_turns(scripts.size(), 1.2, 64.0, 2, seed + 7);
  for (std::size_t i = 0; i < scripts.size(); ++i) {
    auto& sc = scripts[i];
    std::vector<Turn> turns;
    for (int k = 0; k < want[i]; ++k) turns.push_back(sc.turns[static_cast<std::size_t>(k) % sc.turns.size()]);
    sc.turns = std::move(turns);
  }
  SpeedModel speeds;
  speeds.typing_wpm_mean = g_typing_wpm;
  Trace t = synthesize_arrivals(std::move(scripts), users, seed + 1, speeds);
  add_poisson_think(t, mean_think_s, seed + 8);
  return inject_advisories(std::move(t), miss, seed + 3);
}

struct Calibration {
  std::vector<std::pair<int, double>> decode_curve;  // (batch, ms)
  double network_gbs = 12.5;
  double pcie_gbs = 25.0;
  double disk_gbs = 3.0;          // reference LinkProfile default (costmodel.hpp:31)
  double prefill_tps = 8192.0;
  double think_s = 0.0;           // 0: config default
  std::vector<int> users;         // sweep loads; empty: default list
  std::vector<std::string> policies;  // sweep policies; empty: all four
  std::int64_t kv_bytes_per_token = 131'072;  // Llama-3.1-8B, bf16
  std::int64_t hbm_capacity = 160'000'000'000;
};

RunConfig make_cfg(const Calibration& c, Policy p) {
  RunConfig cfg;
  cfg.policy = p;
  cfg.num_nodes = 8;
  cfg.gpu.kv_bytes_per_token = c.kv_bytes_per_token;
  cfg.gpu.num_layers = 32;
  cfg.gpu.hbm_capacity = c.hbm_capacity;
  cfg.gpu.prefill_throughput = c.prefill_tps;
  cfg.gpu.decode_curve_ms = c.decode_curve;
  cfg.links.network_bandwidth = c.network_gbs * 1e9;
  cfg.links.pcie_bandwidth = c.pcie_gbs * 1e9;
  cfg.links.disk_bandwidth = c.disk_gbs * 1e9;
  cfg.sample_period = ns_from_sec(5);
  cfg.invariant_stride = 1024;
  return cfg;
}

double percentile(const std::vector<double>& v, double q) { return traffic::percentile(v, q); }

struct Cell {
  double rps = 0, p50_tpot_ms = 0, p50_ttft_s = 0, p50_norm_ms = 0;
  std::size_t requests = 0;
  std::int64_t migrate_bytes = 0;
};

Cell summarize(const RunReport& rep) {
  Cell c;
  c.rps = steady_rps(rep);
  std::vector<double> tpot, ttft, norm;
  for (const auto& r : rep.records) {
    tpot.push_back(r.tpot_ms());
    ttft.push_back(r.ttft_s());
    norm.push_back(r.normalized_latency_ms_per_token());
  }
  c.p50_tpot_ms = percentile(tpot, 0.5);
  c.p50_ttft_s = percentile(ttft, 0.5);
  c.p50_norm_ms = percentile(norm, 0.5);
  c.requests = rep.records.size();
  for (const auto& t : rep.transfers)
    if (t.reason == TransferReason::Migrate) c.migrate_bytes += t.bytes;
  return c;
}

Calibration parse_calibration(int argc, char** argv, int from) {
  Calibration c;
  for (int i = from; i < argc; ++i) {
    if (!std::strcmp(argv[i], "--decode-curve") && i + 1 < argc) {
      // "b:ms,b:ms,..."
      std::string s = argv[++i];
      std::size_t pos = 0;
      while (pos < s.size()) {
        const std::size_t comma = s.find(',', pos);
        const std::string item = s.substr(pos, comma == std::string::npos ? std::string::npos : comma - pos);
        const std::size_t colon = item.find(':');
        c.decode_curve.emplace_back(std::atoi(item.substr(0, colon).c_str()), std::atof(item.substr(colon + 1).c_str()));
        if (comma == std::string::npos) break;
        pos = comma + 1;
      }
    } else if (!std::strcmp(argv[i], "--network-gbs") && i + 1 < argc) {
      c.network_gbs = std::atof(argv[++i]);
    } else if (!std::strcmp(argv[i], "--pcie-gbs") && i + 1 < argc) {
      c.pcie_gbs = std::atof(argv[++i]);
    } else if (!std::strcmp(argv[i], "--disk-gbs") && i + 1 < argc) {
      c.disk_gbs = std::atof(argv[++i]);
    } else if (!std::strcmp(argv[i], "--prefill-tps") && i + 1 < argc) {
      c.prefill_tps = std::atof(argv[++i]);
    } else if (!std::strcmp(argv[i], "--typing-wpm") && i + 1 < argc) {
      g_typing_wpm = std::atof(argv[++i]);
    } else if (!std::strcmp(argv[i], "--sessions") && i + 1 < argc) {
      g_sessions = std::atoi(argv[++i]);
    } else if (!std::strcmp(argv[i], "--think-s") && i + 1 < argc) {
      c.think_s = std::atof(argv[++i]);
    } else if (!std::strcmp(argv[i], "--policies") && i + 1 < argc) {
      std::string u = argv[++i];
      for (std::size_t pos = 0; pos < u.size();) {
        const std::size_t comma = u.find(',', pos);
        c.policies.push_back(u.substr(pos, comma - pos));
        if (comma == std::string::npos) break;
        pos = comma + 1;
      }
    } else if (!std::strcmp(argv[i], "--users") && i + 1 < argc) {
      std::string u = argv[++i];
      for (std::size_t pos = 0; pos < u.size();) {
        const std::size_t comma = u.find(',', pos);
        c.users.push_back(std::atoi(u.substr(pos, comma - pos).c_str()));
        if (comma == std::string::npos) break;
        pos = comma + 1;
      }
    }
  }
  return c;
}

}  // namespace

int main(int argc, char** argv) {
  if (argc < 3) {
    std::fprintf(stderr, "usage: %s digest <4|5> <policy> <users> [miss] [flags] | sweep <4|5> [flags]\n", argv[0]);
    return 2;
  }
  const std::string mode = argv[1];
  const int config = std::atoi(argv[2]);
  double think_override = 0.0;
  auto make_trace = [&](int users, double miss) {
    return config == 5 ? config5(users, miss, think_override > 0 ? think_override : 6.0, 505)
                       : config4(users, miss, think_override > 0 ? think_override : 10.0, 404);
  };

  if (mode == "digest") {
    const Policy p = policy_from(argv[3]);
    const int users = std::atoi(argv[4]);
    const double miss = argc > 5 && argv[5][0] != '-' ? std::atof(argv[5]) : 0.0;
    const Calibration cal = parse_calibration(argc, argv, 5);
    think_override = cal.think_s;
    const Trace tr = make_trace(users, miss);
    const RunReport rep = run_simulation(tr, make_cfg(cal, p));
    std::uint64_t h = 1469598103934665603ULL;
    for (const auto& t : rep.transfers) {
      h = fnv(h, static_cast<std::uint64_t>(t.time));
      h = fnv(h, (static_cast<std::uint64_t>(t.node) << 40) ^ (static_cast<std::uint64_t>(t.session) << 8) ^
                     static_cast<std::uint64_t>(t.reason));
      h = fnv(h, (static_cast<std::uint64_t>(t.layer_lo) << 32) | (static_cast<std::uint64_t>(t.layer_hi) << 16) |
                     (static_cast<std::uint64_t>(t.from) << 4) | static_cast<std::uint64_t>(t.to));
      h = fnv(h, static_cast<std::uint64_t>(t.bytes));
    }
    std::uint64_t hr = 1469598103934665603ULL;
    for (const auto& r : rep.records) {
      hr = fnv(hr, (static_cast<std::uint64_t>(r.session) << 32) | r.turn);
      hr = fnv(hr, static_cast<std::uint64_t>(r.node));
      hr = fnv(hr, static_cast<std::uint64_t>(r.arrival));
      hr = fnv(hr, static_cast<std::uint64_t>(r.admit));
      hr = fnv(hr, static_cast<std::uint64_t>(r.first_token));
      hr = fnv(hr, static_cast<std::uint64_t>(r.finish));
      hr = fnv(hr, static_cast<std::uint64_t>(r.load_stall));
    }
    const Cell c = summarize(rep);
    std::printf("config %d policy %s users %d miss %.2f sessions %zu requests %zu transfers %zu ledger_hash %016" PRIx64
                " records_hash %016" PRIx64 " makespan_ns %" PRId64 " migrate_bytes %" PRId64 "\n",
                config, rep.policy.c_str(), users, miss, tr.sessions.size(), c.requests, rep.transfers.size(), h, hr,
                rep.makespan, c.migrate_bytes);
    return 0;
  }

  if (mode == "sweep") {
    const Calibration cal = parse_calibration(argc, argv, 3);
    think_override = cal.think_s;
    const std::vector<int> loads = cal.users.empty() ? std::vector<int>{32, 64, 128, 256, 384, 512} : cal.users;
    std::vector<Policy> policies = {Policy::Symphony, Policy::Retain, Policy::Swap, Policy::Recompute};
    if (!cal.policies.empty()) {
      policies.clear();
      for (const auto& p : cal.policies) policies.push_back(policy_from(p));
    }
    std::printf("{\"config\": %d, \"cells\": [", config);
    bool first = true;
    for (Policy p : policies)
      for (int users : loads) {
        if (users > (g_sessions > 0 ? g_sessions : (config == 5 ? 600 : 1000))) continue;
        Cell c;
        try {
          c = summarize(run_simulation(make_trace(users, 0.0), make_cfg(cal, p)));
        } catch (const std::exception& e) {
          std::fprintf(stderr, "cell %s %d failed: %s\n", policy_name(p), users, e.what());
          continue;
        }
        std::printf("%s{\"policy\": \"%s\", \"users\": %d, \"rps\": %.4f, \"p50_tpot_ms\": %.4f, "
                    "\"p50_ttft_s\": %.4f, \"p50_norm_ms\": %.4f, \"requests\": %zu, \"migrate_gb\": %.3f}",
                    first ? "" : ", ", policy_name(p), users, c.rps, c.p50_tpot_ms, c.p50_ttft_s, c.p50_norm_ms,
                    c.requests, c.migrate_bytes / 1e9);
        first = false;
        std::fflush(stdout);
      }
    std::printf("]}\n");
    return 0;
  }
  return 2;
}
