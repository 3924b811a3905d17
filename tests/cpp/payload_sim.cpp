// Config-1 parity run through the reference's UNCHANGED cluster simulator.
// TEST INFRASTRUCTURE (built by tests/cpp/build_payload_sim.sh into
// oracle/_ref/, because it links the reference's Simulation/Engine/
// NodeManager/ClusterScheduler sources compiled from /root/reference).
//
// Two builds of this one file:
//   payload_sim      this repo's KvStore + NodePayload: every store the
//                    reference Simulation constructs gets real pages on the
//                    GPU (via set_default_tier_backend_factory), so the trace's
//                    appends, write-behind persists, advisory promotions and
//                    node-to-node migrations move real bytes with the kvx
//                    kernels. At the end every copy of every block on every
//                    node is read back and checked bit-exact against the CPU
//                    restatement's content for its (session, layer, block).
//   payload_sim_ref  the reference KvStore, no payload: the state oracle.
// Both print the full transfer ledger and per-request records; the test
// requires the two outputs to be identical.
//
// Trace: tiny Llama-style KV (2 layers, 4 KV heads, head_dim 64, fp32: 32 KiB
// pages), 8 sessions x 4 turns on 2 nodes, closed-loop chat with advisories
// leading each turn by more than a migration takes; first turns are staggered
// so least-loaded routing piles them onto node 0 and advisory re-planning
// then migrates sessions to node 1 (the trick of
// /root/reference/proj/tests/acceptance.cpp:172-188).
//
// usage: payload_sim [--device-pages N] [--policy symphony|swap|retain|recompute] [--free-running]
//                    [--disk-dir DIR] [--zipf S | --sharegpt S] [--users U] [--nodes N] [--pages P] [--digest]

#include <algorithm>
#include <cinttypes>
#include <cmath>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <memory>
#include <random>
#include <string>
#include <vector>

#include "symsim/simcore.hpp"

#ifdef WITH_PAYLOAD
#include "../../oracle/kvx_oracle.h"
#include "symsim/payload.hpp"
#endif

using namespace symsim;

namespace {

// KV shape: config 1's tiny fp32 shape by default; --shape 8b switches to
// Llama-3.1-8B's (32 layers, 8 kv heads, head_dim 128, bf16: 64 KiB pages).
int kLayers = 2, kHeads = 4, kDim = 64, kElt = 4, kDtype = 0;
constexpr int kBlockTokens = 16;
constexpr std::uint64_t kSeed = 0x5EEDC0DE;

Trace chat_trace(std::uint64_t seed) {
  std::mt19937_64 rng(seed);
  auto draw = [&rng](Ns lo, Ns hi) { return std::uniform_int_distribution<Ns>(lo, hi)(rng); };
  Trace t;
  t.seed = seed;
  t.concurrency_target = 8;
  for (int s = 0; s < 8; ++s) {
    SessionScript sc;
    sc.session_id = "chat" + std::to_string(s);
    for (int k = 0; k < 4; ++k) {
      const std::int64_t prompt = 24 + 8 * ((s + k) % 5), resp = 6 + (s * 3 + k) % 9;
      sc.turns.push_back({prompt, resp, prompt, resp});
    }
    t.sessions.push_back(sc);
    for (std::uint32_t k = 0; k < 4; ++k) {
      TraceEvent e;
      e.session_index = static_cast<std::uint32_t>(s);
      e.turn_index = k;
      if (k == 0) {
        e.anchor = AnchorPoint::SlotOpen;
        e.delta = s < 5 ? ns_from_ms(1) * s : ns_from_ms(400) + ns_from_ms(3) * s;  // pile onto node 0 first
      } else {
        e.anchor = AnchorPoint::PrevCompletion;
        e.anchor_turn = k - 1;
        e.delta = draw(ns_from_ms(200), ns_from_ms(900));
        TraceEvent adv = e;
        adv.kind = EventKind::Advisory;
        adv.delta = std::max<Ns>(0, e.delta - ns_from_ms(150));  // lead >> per-layer transfer time
        t.events.push_back(adv);
      }
      e.kind = EventKind::Inference;
      t.events.push_back(e);
    }
  }
  return t;
}

// Config 5's traffic at test scale (--zipf S): S multi-turn sessions from the
// reference corpus generator, session popularity Zipf(1.2) mapped to turns
// per session (rank r gets max(2, 64 / r^1.2) turns, cycling its own turn
// list), fast closed-loop users (4,000 wpm, Exp(0.5 s) think), advisories
// injected by the reference generator. Same construction as
// tests/cpp/serve_sim.cpp config5(); here on the tiny KV shape so every page
// of every node fits one GPU.
Trace zipf_trace(int sessions, int users, std::uint64_t seed) {
  SyntheticSpec spec;
  spec.sessions = sessions;
  spec.multi_turn_fraction = 1.0;
  auto scripts = synthesize_corpus(spec, seed);
  std::mt19937_64 rng(seed + 7);
  std::vector<std::size_t> order(scripts.size());
  for (std::size_t i = 0; i < order.size(); ++i) order[i] = i;
  std::shuffle(order.begin(), order.end(), rng);
  for (std::size_t r = 0; r < order.size(); ++r) {
    auto& sc = scripts[order[r]];
    const int want = std::max(2, static_cast<int>(std::lround(64.0 / std::pow(static_cast<double>(r + 1), 1.2))));
    std::vector<Turn> turns;
    for (int k = 0; k < want; ++k) turns.push_back(sc.turns[static_cast<std::size_t>(k) % sc.turns.size()]);
    sc.turns = std::move(turns);
  }
  SpeedModel speeds;
  speeds.typing_wpm_mean = 4000.0;
  Trace t = synthesize_arrivals(std::move(scripts), users, seed + 1, speeds);
  std::exponential_distribution<double> think(2.0);
  for (auto& e : t.events) {
    if (e.kind != EventKind::Inference || e.turn_index == 0) continue;
    const auto& sc = t.sessions[e.session_index];
    e.delta = ns_from_sec(think(rng)) +
              ns_from_sec(static_cast<double>(sc.turns[e.turn_index].prompt_words) * 60.0 / sc.user.typing_wpm);
  }
  return inject_advisories(std::move(t), 0.0, seed + 3);
}

// Config 4's traffic at test scale (--sharegpt S): the reference corpus
// generator's ShareGPT-like defaults (73.4% multi-turn, lognormal lengths)
// for S sessions, fast closed-loop users, Poisson think times (Exp, mean
// 0.5 s), advisories from the reference generator (serve_sim.cpp config4()).
Trace sharegpt_trace(int sessions, int users, std::uint64_t seed) {
  SyntheticSpec spec;
  spec.sessions = sessions;
  auto scripts = synthesize_corpus(spec, seed);
  SpeedModel speeds;
  speeds.typing_wpm_mean = 4000.0;
  Trace t = synthesize_arrivals(std::move(scripts), users, seed + 1, speeds);
  std::mt19937_64 rng(seed + 2);
  std::exponential_distribution<double> think(2.0);
  for (auto& e : t.events) {
    if (e.kind != EventKind::Inference || e.turn_index == 0) continue;
    const auto& sc = t.sessions[e.session_index];
    e.delta = ns_from_sec(think(rng)) +
              ns_from_sec(static_cast<double>(sc.turns[e.turn_index].prompt_words) * 60.0 / sc.user.typing_wpm);
  }
  return inject_advisories(std::move(t), 0.0, seed + 3);
}

std::uint64_t fnv(std::uint64_t h, std::uint64_t v) {
  for (int i = 0; i < 8; ++i) {
    h ^= (v >> (8 * i)) & 0xFF;
    h *= 1099511628211ULL;
  }
  return h;
}

const char* tier_s(Tier t) { return tier_name(t); }

}  // namespace

int main(int argc, char** argv) {
  std::int64_t device_pages = 0;
  std::string policy = "symphony";
  bool free_running = false;
  std::string disk_dir;  // --disk-dir: DISK tier in files (one per node) instead of pinned host memory
  int zipf_sessions = 0, sharegpt_sessions = 0, users = 64, num_nodes = 2;
  std::int64_t pool_pages = 0;  // --pages: per-node DEVICE / HOST / landing pages (and the store's capacities)
  bool digest = false;          // --digest: hashes of the ledger and records instead of every row
  std::uint64_t trace_seed = 0; // --seed: base seed of the --zipf / --sharegpt generators (0 = fixed default)
  for (int i = 1; i < argc; ++i) {
    if (!std::strcmp(argv[i], "--zipf") && i + 1 < argc) zipf_sessions = std::atoi(argv[++i]);
    if (!std::strcmp(argv[i], "--sharegpt") && i + 1 < argc) sharegpt_sessions = std::atoi(argv[++i]);
    if (!std::strcmp(argv[i], "--users") && i + 1 < argc) users = std::atoi(argv[++i]);
    if (!std::strcmp(argv[i], "--nodes") && i + 1 < argc) num_nodes = std::atoi(argv[++i]);
    if (!std::strcmp(argv[i], "--pages") && i + 1 < argc) pool_pages = std::atoll(argv[++i]);
    if (!std::strcmp(argv[i], "--digest")) digest = true;
    if (!std::strcmp(argv[i], "--seed") && i + 1 < argc) trace_seed = std::strtoull(argv[++i], nullptr, 10);
    if (!std::strcmp(argv[i], "--shape") && i + 1 < argc && !std::strcmp(argv[++i], "8b")) {
      kLayers = 32;
      kHeads = 8;
      kDim = 128;
      kElt = 2;
      kDtype = 1;
    }
    if (!std::strcmp(argv[i], "--disk-dir") && i + 1 < argc) disk_dir = argv[++i];
    if (!std::strcmp(argv[i], "--device-pages") && i + 1 < argc) device_pages = std::atoll(argv[++i]);
    if (!std::strcmp(argv[i], "--policy") && i + 1 < argc) policy = argv[++i];
    if (!std::strcmp(argv[i], "--free-running")) free_running = true;
  }
  (void)free_running;
  (void)disk_dir;
  RunConfig cfg;
  cfg.policy = policy_from(policy);
  cfg.num_nodes = num_nodes;
  cfg.gpu.num_layers = kLayers;
  cfg.gpu.kv_bytes_per_token = static_cast<std::int64_t>(kLayers) * 2 * kHeads * kDim * kElt;
  cfg.gpu.hbm_capacity = 80'000'000'000;
  const std::int64_t page = cfg.gpu.kv_bytes_per_token / kLayers * kBlockTokens;
  if (device_pages > 0) cfg.device_capacity = device_pages * page;  // force cooperative purges
  cfg.host_capacity = 4096 * page;
  if (pool_pages > 0) {  // the store's tiers are exactly the pools behind them
    cfg.device_capacity = pool_pages * page;
    cfg.host_capacity = pool_pages * page;
  }
  cfg.sample_period = ns_from_sec(5);
  const Trace trace = zipf_sessions > 0      ? zipf_trace(zipf_sessions, users, trace_seed ? trace_seed : 505)
                      : sharegpt_sessions > 0 ? sharegpt_trace(sharegpt_sessions, users, trace_seed ? trace_seed : 404)
                                              : chat_trace(20260417);

#ifdef WITH_PAYLOAD
  PayloadCluster cluster;
  std::vector<std::unique_ptr<NodePayload>> nodes;
  PayloadOptions po;
  po.device = 0;  // both nodes on the one visible GPU (peer path = local HBM)
  po.layout = kvx_page_layout{kHeads, kDim, kBlockTokens, kDtype ? KVX_DTYPE_BF16 : KVX_DTYPE_F32};
  po.device_pages = static_cast<std::uint64_t>(device_pages > 0 ? device_pages + 64 : 2048);
  po.host_pages = 4096;
  po.landing_pages = 4096;
  po.disk_pages = 8192;
  if (pool_pages > 0) {
    po.device_pages = static_cast<std::uint64_t>(pool_pages) + 64;
    po.host_pages = static_cast<std::uint64_t>(pool_pages);
    po.landing_pages = static_cast<std::uint64_t>(pool_pages);
    po.disk_pages = 4 * static_cast<std::uint64_t>(pool_pages);
  }
  po.seed = kSeed;
  po.free_running = free_running;
  set_default_tier_backend_factory([&](int node_id) -> TierBackend* {
    PayloadOptions o = po;
    if (!disk_dir.empty()) o.disk_path = disk_dir + "/node" + std::to_string(node_id) + ".pages";
    nodes.push_back(std::make_unique<NodePayload>(&cluster, node_id, o));
    return nodes.back().get();
  });
#endif

  Simulation sim(trace, cfg);
  const RunReport rep = sim.run();

  std::printf("policy %s nodes %d transfers %zu records %zu\n", rep.policy.c_str(), rep.num_nodes,
              rep.transfers.size(), rep.records.size());
  std::size_t migrate_rows = 0;
  std::uint64_t hl = 1469598103934665603ULL, hr = 1469598103934665603ULL;
  for (const auto& r : rep.transfers) {
    if (r.reason == TransferReason::Migrate) ++migrate_rows;
    if (digest) {
      hl = fnv(hl, static_cast<std::uint64_t>(r.time));
      hl = fnv(hl, (static_cast<std::uint64_t>(r.node) << 40) ^ (static_cast<std::uint64_t>(r.session) << 8) ^
                       static_cast<std::uint64_t>(r.reason));
      hl = fnv(hl, (static_cast<std::uint64_t>(r.layer_lo) << 32) | (static_cast<std::uint64_t>(r.layer_hi) << 16) |
                       (static_cast<std::uint64_t>(r.from) << 4) | static_cast<std::uint64_t>(r.to));
      hl = fnv(hl, static_cast<std::uint64_t>(r.bytes));
      continue;
    }
    std::printf("T %" PRId64 " n%d s%u l%u-%u %s>%s %" PRId64 " %s\n", r.time, r.node, r.session, r.layer_lo,
                r.layer_hi, tier_s(r.from), tier_s(r.to), r.bytes, reason_name(r.reason));
  }
  for (const auto& r : rep.records) {
    if (digest) {
      hr = fnv(hr, (static_cast<std::uint64_t>(r.session) << 32) | r.turn);
      hr = fnv(hr, static_cast<std::uint64_t>(r.node));
      hr = fnv(hr, static_cast<std::uint64_t>(r.arrival));
      hr = fnv(hr, static_cast<std::uint64_t>(r.first_token));
      hr = fnv(hr, static_cast<std::uint64_t>(r.finish));
      hr = fnv(hr, static_cast<std::uint64_t>(r.load_stall));
      continue;
    }
    std::printf("R s%u t%u n%d arr %" PRId64 " adm %" PRId64 " ft %" PRId64 " fin %" PRId64 " stall %" PRId64 "\n",
                r.session, r.turn, r.node, r.arrival, r.admit, r.first_token, r.finish, r.load_stall);
  }
  if (digest)
    std::printf("digest ledger %016" PRIx64 " records %016" PRIx64 " rows %zu records %zu\n", hl, hr,
                rep.transfers.size(), rep.records.size());
  std::printf("migrate_rows %zu\n", migrate_rows);

#ifdef WITH_PAYLOAD
  // Every copy on every node, bit-exact against the CPU restatement.
  std::vector<std::uint8_t> got(static_cast<std::size_t>(page)), want(static_cast<std::size_t>(page));
  const kvxo_layout ol{kHeads, kDim, kBlockTokens, kDtype};
  std::size_t copies = 0, bad = 0, pages_held[4] = {0, 0, 0, 0};
  for (int n = 0; n < cfg.num_nodes; ++n) {
    const KvStore& st = sim.node(n).store();
    NodePayload* node = cluster.node(n);
    for (std::uint32_t s = 0; s < trace.sessions.size(); ++s)
      for (int l = 0; l < kLayers; ++l)
        for (std::uint32_t b = 0; b < st.blocks_in_layer(s, static_cast<std::uint16_t>(l)); ++b) {
          const std::uint8_t res = st.residency(s, static_cast<std::uint16_t>(l), b);
          for (int t = 0; t < 3; ++t) {
            const int pool = node->pool_of(s, static_cast<std::uint16_t>(l), b, static_cast<Tier>(t));
            if (!(res & (1u << t))) {
              if (pool >= 0) ++bad;
              continue;
            }
            ++copies;
            if (pool < 0 || !node->read_block(s, static_cast<std::uint16_t>(l), b, static_cast<Tier>(t), got.data())) {
              ++bad;
              continue;
            }
            ++pages_held[pool];
            const std::uint32_t id0 = 0;
            const kvxo_tag tag{s, static_cast<std::uint32_t>(l), b};
            kvxo_fill_pages(want.data(), static_cast<std::uint64_t>(page), &id0, &tag, 1, kSeed, &ol, 1);
            if (std::memcmp(got.data(), want.data(), got.size()) != 0) ++bad;
          }
        }
    for (int p = 0; p < 4; ++p)
      if (node->pages_in_use(static_cast<NodePayload::Pool>(p)) != pages_held[p]) ++bad;  // leak or loss
    const std::uint64_t* mv = node->bytes_moved();
    std::printf("payload node %d posted %" PRIu64 " apply_wait_us %.1f\n", n, node->transfers_posted(),
                node->apply_wait_ns() / 1e3);
    std::printf("payload node %d pages dev %zu host %zu landing %zu disk %zu moved created %" PRIu64
                " h2d %" PRIu64 " host_copy %" PRIu64 " disk_write %" PRIu64 " net_arrive %" PRIu64 "\n",
                n, pages_held[0], pages_held[1], pages_held[2], pages_held[3], mv[0], mv[1], mv[3], mv[4], mv[6]);
    for (auto& h : pages_held) h = 0;
  }
  std::printf("payload verified_copies %zu mismatches %zu\n", copies, bad);
  set_default_tier_backend_factory({});
  return bad == 0 ? 0 : 1;
#else
  return 0;
#endif
}
