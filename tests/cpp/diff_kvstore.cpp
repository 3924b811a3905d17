// Differential state-parity fuzzer: drives the product KvStore and the
// reference KvStore (oracle/_ref) through identical randomized call sequences
// via the shared kvs_* C ABI and compares every observable after every call:
// status codes and exception messages, scheduled transfers (ids and
// completion times), created keys, load plans, promote results, purge
// results, all tier counters, every session's state, the full ledger, the
// evictable-block order and the device usage diagnostic.
//
// The op mix follows the reference's own randomized suites
// (/root/reference/proj/tests/property_suites.hpp:47-141, TransferPool-style
// completion in (time, id) order) but also exercises error paths, voiding,
// tight HOST/DISK capacities and write-behind off. Test infrastructure.
//
// usage: diff_kvstore <product.so> <oracle.so> [cases] [ops] [seed]

#include <algorithm>
#include <cinttypes>
#include <cstdio>
#include <cstring>
#include <random>
#include <sstream>
#include <string>
#include <vector>

#include "kvs_dyn.hpp"

namespace {

struct Pair {
  KvsApi& a;  // product
  KvsApi& b;  // oracle
  kvs_store* sa = nullptr;
  kvs_store* sb = nullptr;
};

int g_failures = 0;
std::string g_context;

void fail(const std::string& what) {
  if (g_failures < 20) std::fprintf(stderr, "MISMATCH [%s]: %s\n", g_context.c_str(), what.c_str());
  ++g_failures;
}

template <typename T>
std::string str(const T& v) {
  std::ostringstream os;
  os << v;
  return os.str();
}

bool same_status(Pair& p, const char* op, int ra, int rb) {
  if (ra != rb) {
    fail(std::string(op) + ": status " + str(ra) + " vs " + str(rb) + " (" + p.a.kvs_last_error() + " | " +
         p.b.kvs_last_error() + ")");
    return false;
  }
  if (ra != 0 && std::strcmp(p.a.kvs_last_error(), p.b.kvs_last_error()) != 0)
    fail(std::string(op) + ": message '" + p.a.kvs_last_error() + "' vs '" + p.b.kvs_last_error() + "'");
  return true;
}

void cmp_out(Pair& p, const char* op) {
  const kvs_scheduled *xa, *xb;
  const size_t na = p.a.kvs_out_scheduled(p.sa, &xa), nb = p.b.kvs_out_scheduled(p.sb, &xb);
  if (na != nb) {
    fail(std::string(op) + ": scheduled count " + str(na) + " vs " + str(nb));
  } else {
    for (size_t i = 0; i < na; ++i)
      if (xa[i].id != xb[i].id || xa[i].complete_at != xb[i].complete_at)
        fail(std::string(op) + ": scheduled[" + str(i) + "] " + str(xa[i].id) + "@" + str(xa[i].complete_at) +
             " vs " + str(xb[i].id) + "@" + str(xb[i].complete_at));
  }
  const kvs_block_key *ka, *kb;
  const size_t nka = p.a.kvs_out_keys(p.sa, &ka), nkb = p.b.kvs_out_keys(p.sb, &kb);
  if (nka != nkb) fail(std::string(op) + ": keys count");
  else
    for (size_t i = 0; i < nka; ++i)
      if (ka[i].session != kb[i].session || ka[i].layer != kb[i].layer || ka[i].block_index != kb[i].block_index)
        fail(std::string(op) + ": key " + str(i));
  const int64_t *ta, *tb;
  const size_t nta = p.a.kvs_out_times(p.sa, &ta), ntb = p.b.kvs_out_times(p.sb, &tb);
  if (nta != ntb || !std::equal(ta, ta + nta, tb)) fail(std::string(op) + ": layer_ready");
}

void cmp_state(Pair& p, int num_sessions, bool deep) {
  kvs_counters ca{}, cb{};
  p.a.kvs_get_counters(p.sa, &ca);
  p.b.kvs_get_counters(p.sb, &cb);
  if (std::memcmp(&ca, &cb, sizeof ca) != 0)
    fail("counters dev " + str(ca.device_used) + "/" + str(cb.device_used) + " host " + str(ca.host_used) + "/" +
         str(cb.host_used) + " disk " + str(ca.disk_used) + "/" + str(cb.disk_used));
  for (int s = 0; s < num_sessions + 1; ++s) {  // +1: an unregistered id
    kvs_session_info ia{}, ib{};
    const int ra = p.a.kvs_get_session(p.sa, s, &ia), rb = p.b.kvs_get_session(p.sb, s, &ib);
    if (!same_status(p, "get_session", ra, rb)) continue;
    if (ra == 0 && std::memcmp(&ia, &ib, sizeof ia) != 0) fail("session " + str(s) + " info");
    int64_t la = 0, lb = 0;
    const int r1 = p.a.kvs_bytes_for_load(p.sa, s, &la), r2 = p.b.kvs_bytes_for_load(p.sb, s, &lb);
    if (same_status(p, "bytes_for_load", r1, r2) && la != lb) fail("bytes_for_load " + str(s));
  }
  const size_t la = p.a.kvs_ledger_size(p.sa), lb = p.b.kvs_ledger_size(p.sb);
  if (la != lb) {
    fail("ledger size " + str(la) + " vs " + str(lb));
  } else if (la > 0) {
    std::vector<kvs_record> ra(la), rb(lb);
    p.a.kvs_ledger_copy(p.sa, 0, la, ra.data());
    p.b.kvs_ledger_copy(p.sb, 0, lb, rb.data());
    for (size_t i = 0; i < la; ++i)
      if (std::memcmp(&ra[i], &rb[i], sizeof(kvs_record)) != 0) {
        fail("ledger row " + str(i) + " t=" + str(ra[i].time) + "/" + str(rb[i].time) + " s=" +
             str(ra[i].session) + "/" + str(rb[i].session) + " bytes=" + str(ra[i].bytes) + "/" + str(rb[i].bytes));
        break;
      }
  }
  if (!deep) return;
  for (int spare = 0; spare < 2; ++spare) {
    const int r1 = p.a.kvs_evictable_blocks(p.sa, spare), r2 = p.b.kvs_evictable_blocks(p.sb, spare);
    if (!same_status(p, "evictable_blocks", r1, r2)) continue;
    const kvs_block_meta *ma, *mb;
    const size_t na = p.a.kvs_out_metas(p.sa, &ma), nb = p.b.kvs_out_metas(p.sb, &mb);
    if (na != nb) {
      fail("evictable count " + str(na) + " vs " + str(nb));
      continue;
    }
    for (size_t i = 0; i < na; ++i)
      if (ma[i].key.session != mb[i].key.session || ma[i].key.layer != mb[i].key.layer ||
          ma[i].key.block_index != mb[i].key.block_index || ma[i].session_bytes != mb[i].session_bytes ||
          std::strcmp(ma[i].session_id, mb[i].session_id) != 0) {
        fail("evictable order at " + str(i));
        break;
      }
  }
  char da[256], db[256];
  p.a.kvs_device_usage_debug(p.sa, da, sizeof da);
  p.b.kvs_device_usage_debug(p.sb, db, sizeof db);
  if (std::strcmp(da, db) != 0) fail(std::string("usage debug '") + da + "' vs '" + db + "'");
  const int r1 = p.a.kvs_check_budgets(p.sa), r2 = p.b.kvs_check_budgets(p.sb);
  same_status(p, "check_budgets", r1, r2);
}

struct Pending {
  int64_t at;
  uint64_t id;
  bool operator<(const Pending& o) const { return at != o.at ? at < o.at : id < o.id; }
};

void take_sched(Pair& p, std::vector<Pending>& pending) {
  const kvs_scheduled* x;
  const size_t n = p.a.kvs_out_scheduled(p.sa, &x);
  for (size_t i = 0; i < n; ++i) pending.push_back({x[i].complete_at, x[i].id});
}

int pick(std::mt19937_64& rng, int lo, int hi) { return std::uniform_int_distribution<int>(lo, hi)(rng); }

void run_case(KvsApi& A, KvsApi& B, std::uint64_t seed, int ops) {
  std::mt19937_64 rng(seed);
  kvs_gpu_profile gpu{};
  gpu.prefill_throughput = 8192.0;
  gpu.decode_base_ms = 12.0;
  gpu.decode_half_batch = 16.0;
  gpu.hbm_capacity = 80'000'000'000;
  gpu.num_layers = pick(rng, 1, 5);
  static const int64_t kPerToken[] = {1'100'000, 4096, 131'072, 327'680, 1000, 7};
  gpu.kv_bytes_per_token = kPerToken[pick(rng, 0, 5)];
  kvs_link_profile links{25e9, 3e9, 12.5e9, 10'000};
  if (pick(rng, 0, 3) == 0) links.per_transfer_latency = pick(rng, 0, 3) * 7;
  if (pick(rng, 0, 3) == 0) links.network_bandwidth = 900e9;
  kvs_options opts{};
  opts.node_id = pick(rng, 0, 3);
  static const int kBlockTokens[] = {1, 2, 4, 16};
  opts.block_tokens = kBlockTokens[pick(rng, 0, 3)];
  int64_t lbb = 0;
  A.kvs_kv_bytes_per_layer(opts.block_tokens, &gpu, &lbb);
  opts.device_capacity = lbb * gpu.num_layers * pick(rng, 1, 12) + (pick(rng, 0, 2) == 0 ? pick(rng, 0, 5) : 0);
  const int host_mode = pick(rng, 0, 3);
  opts.host_capacity = host_mode == 0   ? 0
                       : host_mode == 1 ? lbb * pick(rng, 1, 40)
                                        : 256'000'000'000LL;
  opts.disk_capacity = pick(rng, 0, 4) == 0 ? lbb * pick(rng, 0, 60) : -1;
  opts.write_behind = pick(rng, 0, 3) != 0;

  Pair p{A, B};
  const int ra = A.kvs_create(&gpu, &links, &opts, &p.sa), rb = B.kvs_create(&gpu, &links, &opts, &p.sb);
  if (!same_status(p, "create", ra, rb) || ra != 0) return;

  const int nsess = pick(rng, 1, 5);
  static const char* kIds[] = {"s0", "alpha", "b", "s0b", "zz", "a", "m"};
  for (int s = 0; s < nsess; ++s) {
    const char* id = kIds[pick(rng, 0, 6)];
    const int prio = pick(rng, 0, 3) == 0;
    same_status(p, "register", A.kvs_register_session(p.sa, s, id, prio), B.kvs_register_session(p.sb, s, id, prio));
  }
  if (pick(rng, 0, 4) != 0) same_status(p, "finalize", A.kvs_finalize_sessions(p.sa), B.kvs_finalize_sessions(p.sb));

  std::vector<Pending> pending;
  int64_t now = 0;
  for (int op = 0; op < ops; ++op) {
    g_context = "seed " + str(seed) + " op " + str(op);
    now += pick(rng, 0, 3) == 0 ? 0 : pick(rng, 0, 200'000);
    const uint32_t s = static_cast<uint32_t>(pick(rng, 0, nsess));  // nsess == unknown session
    const int which = pick(rng, 0, 21);
    switch (which) {
      case 0:
      case 1:
      case 2: {
        const int64_t toks = pick(rng, 0, 12) == 0 ? pick(rng, -2, 0) : pick(rng, 1, 3 * opts.block_tokens + 3);
        int64_t need_a = 0, need_b = 0;
        const int q1 = A.kvs_bytes_for_new_blocks(p.sa, s, toks, &need_a), q2 = B.kvs_bytes_for_new_blocks(p.sb, s, toks, &need_b);
        if (same_status(p, "bytes_for_new_blocks", q1, q2) && need_a != need_b) fail("bytes_for_new_blocks");
        const int r1 = A.kvs_append_blocks(p.sa, s, toks, now), r2 = B.kvs_append_blocks(p.sb, s, toks, now);
        same_status(p, "append", r1, r2);
        cmp_out(p, "append");
        take_sched(p, pending);
        break;
      }
      case 3:
      case 4: {
        int64_t fa = -1, fb = -1;
        const int64_t need = pick(rng, 0, 5) == 0 ? pick(rng, -1, 0) : lbb * pick(rng, 1, 3 * gpu.num_layers) + pick(rng, 0, 1);
        const int spare = pick(rng, 0, 1);
        const int r1 = A.kvs_purge_from_device(p.sa, need, now, spare, &fa);
        const int r2 = B.kvs_purge_from_device(p.sb, need, now, spare, &fb);
        if (same_status(p, "purge", r1, r2) && fa != fb) fail("purge freed " + str(fa) + " vs " + str(fb));
        cmp_out(p, "purge");
        take_sched(p, pending);
        break;
      }
      case 5:
      case 6: {
        kvs_load_plan la{}, lb2{};
        const int64_t cpl = pick(rng, 0, 500'000);
        const int reason = pick(rng, 0, 4);
        const int r1 = A.kvs_plan_layerwise_load(p.sa, s, now, cpl, reason, &la);
        const int r2 = B.kvs_plan_layerwise_load(p.sb, s, now, cpl, reason, &lb2);
        if (same_status(p, "plan", r1, r2) && r1 == 0 && std::memcmp(&la, &lb2, sizeof la) != 0) fail("plan result");
        cmp_out(p, "plan");
        take_sched(p, pending);
        break;
      }
      case 7: {
        kvs_promote_result xa{}, xb{};
        const int r1 = A.kvs_promote(p.sa, s, now, &xa), r2 = B.kvs_promote(p.sb, s, now, &xb);
        if (same_status(p, "promote", r1, r2) && r1 == 0 && std::memcmp(&xa, &xb, sizeof xa) != 0) fail("promote result");
        cmp_out(p, "promote");
        take_sched(p, pending);
        break;
      }
      case 8: {
        const int r1 = A.kvs_offload_session(p.sa, s, now), r2 = B.kvs_offload_session(p.sb, s, now);
        same_status(p, "offload", r1, r2);
        cmp_out(p, "offload");
        take_sched(p, pending);
        break;
      }
      case 9:
        if (pick(rng, 0, 2) == 0)
          same_status(p, "release", A.kvs_release_session(p.sa, s, now), B.kvs_release_session(p.sb, s, now));
        break;
      case 10:
        same_status(p, "mark_out", A.kvs_mark_migrating_out(p.sa, s), B.kvs_mark_migrating_out(p.sb, s));
        break;
      case 11: {
        const int64_t toks = pick(rng, 0, 8) == 0 ? 0 : pick(rng, 1, 4 * opts.block_tokens);
        const int r1 = A.kvs_import_migration(p.sa, s, toks, now), r2 = B.kvs_import_migration(p.sb, s, toks, now);
        same_status(p, "import", r1, r2);
        cmp_out(p, "import");
        take_sched(p, pending);
        break;
      }
      case 12:
      case 13: {
        const int act = pick(rng, 0, 1);
        same_status(p, "set_active", A.kvs_set_active(p.sa, s, act, now), B.kvs_set_active(p.sb, s, act, now));
        break;
      }
      case 14: {
        const int64_t bytes = pick(rng, 0, 6) == 0 ? -1 : lbb * pick(rng, 0, 4);
        if (pick(rng, 0, 1))
          same_status(p, "reserve", A.kvs_reserve_device(p.sa, bytes), B.kvs_reserve_device(p.sb, bytes));
        else
          same_status(p, "unreserve", A.kvs_unreserve_device(p.sa, bytes), B.kvs_unreserve_device(p.sb, bytes));
        break;
      }
      case 15:
        if (pick(rng, 0, 1))
          same_status(p, "void_loads", A.kvs_void_session_loads(p.sa, s), B.kvs_void_session_loads(p.sb, s));
        else
          same_status(p, "void_offload", A.kvs_void_session_offload(p.sa, s), B.kvs_void_session_offload(p.sb, s));
        break;
      default: {  // complete the next few transfers in (time, id) order
        std::sort(pending.begin(), pending.end());
        const int k = std::min<int>(pick(rng, 1, 6), static_cast<int>(pending.size()));
        for (int i = 0; i < k; ++i) {
          const Pending t = pending[static_cast<size_t>(i)];
          now = std::max(now, t.at);
          kvs_apply_result xa{}, xb{};
          const int r1 = A.kvs_apply_transfer(p.sa, t.id, t.at, &xa), r2 = B.kvs_apply_transfer(p.sb, t.id, t.at, &xb);
          if (same_status(p, "apply", r1, r2) && r1 == 0 && std::memcmp(&xa, &xb, sizeof xa) != 0)
            fail("apply result id " + str(t.id));
        }
        pending.erase(pending.begin(), pending.begin() + k);
        if (pick(rng, 0, 9) == 0) {  // an id nobody scheduled
          kvs_apply_result xa{}, xb{};
          same_status(p, "apply_unknown", A.kvs_apply_transfer(p.sa, 999'999, now, &xa),
                      B.kvs_apply_transfer(p.sb, 999'999, now, &xb));
        }
      }
    }
    cmp_state(p, nsess, op % 4 == 0 || op == ops - 1);
  }
  // Drain, as every reference driver does at the end.
  std::sort(pending.begin(), pending.end());
  for (const auto& t : pending) {
    kvs_apply_result xa{}, xb{};
    const int r1 = A.kvs_apply_transfer(p.sa, t.id, t.at, &xa), r2 = B.kvs_apply_transfer(p.sb, t.id, t.at, &xb);
    if (same_status(p, "drain", r1, r2) && r1 == 0 && std::memcmp(&xa, &xb, sizeof xa) != 0) fail("drain result");
  }
  cmp_state(p, nsess, true);
  A.kvs_destroy(p.sa);
  B.kvs_destroy(p.sb);
}

void free_functions(KvsApi& A, KvsApi& B, std::uint64_t seed) {
  std::mt19937_64 rng(seed);
  Pair p{A, B};
  for (int c = 0; c < 2000; ++c) {
    g_context = "free seed " + str(seed) + " case " + str(c);
    // evict_order on random candidates (ties included)
    const int n = pick(rng, 0, 12);
    std::vector<kvs_block_meta> cands(n);
    static const char* kIds[] = {"a", "b", "aa", "ab", ""};
    for (auto& m : cands) {
      m.key.layer = static_cast<uint16_t>(pick(rng, 0, 3));
      m.key.block_index = static_cast<uint32_t>(pick(rng, 0, 4));
      m.session_bytes = pick(rng, 0, 3) * 50;
      m.session_id = kIds[pick(rng, 0, 4)];
      m.pinned = pick(rng, 0, 30) == 0;
    }
    std::vector<uint32_t> oa(n), ob(n);
    const int r1 = A.kvs_evict_order(cands.data(), n, oa.data()), r2 = B.kvs_evict_order(cands.data(), n, ob.data());
    if (same_status(p, "evict_order", r1, r2) && r1 == 0 && oa != ob) fail("evict_order permutation");
    // pipeline gate
    const int L = pick(rng, 0, 9);
    std::vector<int64_t> ready(L);
    for (auto& r : ready) r = pick(rng, 0, 3'000'000);
    const int64_t cr = pick(rng, 0, 2'000'000), step = pick(rng, 0, 40'000'003);
    kvs_gate_result ga{}, gb{};
    const int g1 = A.kvs_pipeline_gate(ready.data(), L, cr, step, &ga), g2 = B.kvs_pipeline_gate(ready.data(), L, cr, step, &gb);
    if (same_status(p, "gate", g1, g2) && g1 == 0 && std::memcmp(&ga, &gb, sizeof ga) != 0) fail("gate");
    // cost model
    kvs_link_profile links{pick(rng, 1, 100) * 1e9, pick(rng, 1, 10) * 1e9, pick(rng, 1, 900) * 1e9, pick(rng, -1, 20'000)};
    const int64_t bytes = pick(rng, 0, 10) == 0 ? -1 : static_cast<int64_t>(rng() % 20'000'000'000ULL);
    const int link = pick(rng, 0, 4);
    int64_t ta = 0, tb = 0;
    const int t1 = A.kvs_transfer_time(bytes, link, &links, &ta), t2 = B.kvs_transfer_time(bytes, link, &links, &tb);
    if (same_status(p, "transfer_time", t1, t2) && ta != tb) fail("transfer_time");
    kvs_gpu_profile gpu{8192.0, 12.0, 16.0, 80'000'000'000, 1'100'000, 32, 0, nullptr, nullptr};
    gpu.decode_base_ms = pick(rng, 1, 40) * 0.37;
    gpu.decode_half_batch = pick(rng, 1, 64) * 0.5;
    gpu.prefill_throughput = pick(rng, 100, 20000) * 1.3;
    std::vector<int32_t> cb;
    std::vector<double> cm;
    if (pick(rng, 0, 1)) {
      int b = 0;
      for (int i = 0, k = pick(rng, 1, 6); i < k; ++i) {
        b += pick(rng, 1, 20);
        cb.push_back(b);
        cm.push_back(pick(rng, 1, 900) * 0.11);
      }
      gpu.curve_points = static_cast<int32_t>(cb.size());
      gpu.curve_batch = cb.data();
      gpu.curve_ms = cm.data();
    }
    const int batch = pick(rng, -1, 130);
    int64_t da = 0, db = 0;
    const int d1 = A.kvs_decode_step_time(batch, &gpu, &da), d2 = B.kvs_decode_step_time(batch, &gpu, &db);
    if (same_status(p, "decode_step_time", d1, d2) && da != db) fail("decode_step_time");
    const int64_t toks = pick(rng, -2, 100'000);
    const int p1 = A.kvs_prefill_time(toks, &gpu, &da), p2 = B.kvs_prefill_time(toks, &gpu, &db);
    if (same_status(p, "prefill_time", p1, p2) && da != db) fail("prefill_time");
    gpu.kv_bytes_per_token = pick(rng, 1, 2'000'000);
    gpu.num_layers = pick(rng, 1, 100);
    const int k1 = A.kvs_kv_bytes_per_layer(toks, &gpu, &da), k2 = B.kvs_kv_bytes_per_layer(toks, &gpu, &db);
    if (same_status(p, "kv_bytes_per_layer", k1, k2) && da != db) fail("kv_bytes_per_layer");
  }
}

}  // namespace

int main(int argc, char** argv) {
  if (argc < 3) {
    std::fprintf(stderr, "usage: %s <product.so> <oracle.so> [cases] [ops] [seed]\n", argv[0]);
    return 2;
  }
  KvsApi A(argv[1]), B(argv[2]);
  if (A.kvs_is_product() != 1 || B.kvs_is_product() != 0) {
    std::fprintf(stderr, "expected <product> then <oracle> library\n");
    return 2;
  }
  const int cases = argc > 3 ? std::atoi(argv[3]) : 2000;
  const int ops = argc > 4 ? std::atoi(argv[4]) : 80;
  const std::uint64_t seed0 = argc > 5 ? std::strtoull(argv[5], nullptr, 10) : 20260417;
  free_functions(A, B, seed0);
  for (int c = 0; c < cases; ++c) run_case(A, B, seed0 * 1000003ULL + static_cast<std::uint64_t>(c), ops);
  std::printf("diff_kvstore: %d cases x %d ops, %d mismatches\n", cases, ops, g_failures);
  return g_failures == 0 ? 0 : 1;
}
