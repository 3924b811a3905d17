// kvs_* C ABI over symsim::KvStore (include/kvs.h).
//
// Compiled twice from this one file: into the product library against this
// repo's headers (KVS_PRODUCT defined), and by oracle/Makefile into
// oracle/_ref against the reference headers with `symsim` renamed to
// `symsim_oracle` (the macro renames every `symsim::` below consistently).
// It must therefore use only the public API the two KvStores share
// (reference: /root/reference/proj/include/symsim/kvstore.hpp:107-229).
// Exceptions never cross the ABI: they become KVS_ERR_* plus a message.

#include "kvs.h"

#include <cstring>
#include <stdexcept>
#include <string>
#include <vector>

#include "symsim/kvstore.hpp"

namespace {

thread_local std::string g_last_error;

template <typename F>
int guarded(F&& fn) {
  try {
    fn();
    return KVS_OK;
  } catch (const std::logic_error& e) {
    g_last_error = e.what();
    return KVS_ERR_LOGIC;
  } catch (const std::runtime_error& e) {
    g_last_error = e.what();
    return KVS_ERR_RUNTIME;
  } catch (const std::exception& e) {
    g_last_error = e.what();
    return KVS_ERR_OTHER;
  } catch (...) {
    g_last_error = "unknown exception";
    return KVS_ERR_OTHER;
  }
}

symsim::GpuProfile to_gpu(const kvs_gpu_profile* g) {
  symsim::GpuProfile p;
  if (!g) return p;
  p.prefill_throughput = g->prefill_throughput;
  p.decode_base_ms = g->decode_base_ms;
  p.decode_half_batch = g->decode_half_batch;
  p.hbm_capacity = g->hbm_capacity;
  p.kv_bytes_per_token = g->kv_bytes_per_token;
  p.num_layers = g->num_layers;
  for (int i = 0; i < g->curve_points; ++i) p.decode_curve_ms.emplace_back(g->curve_batch[i], g->curve_ms[i]);
  return p;
}

symsim::LinkProfile to_links(const kvs_link_profile* l) {
  symsim::LinkProfile p;
  if (!l) return p;
  p.pcie_bandwidth = l->pcie_bandwidth;
  p.disk_bandwidth = l->disk_bandwidth;
  p.network_bandwidth = l->network_bandwidth;
  p.per_transfer_latency = l->per_transfer_latency;
  return p;
}

symsim::KvStore::Options to_opts(const kvs_options* o) {
  symsim::KvStore::Options p;
  if (!o) return p;
  p.node_id = o->node_id;
  p.block_tokens = o->block_tokens;
  p.device_capacity = o->device_capacity;
  p.host_capacity = o->host_capacity;
  p.disk_capacity = o->disk_capacity;
  p.write_behind = o->write_behind != 0;
  return p;
}

}  // namespace

struct kvs_store {
  symsim::KvStore store;
  std::vector<kvs_scheduled> sched;
  std::vector<kvs_block_key> keys;
  std::vector<std::int64_t> times;
  std::vector<kvs_block_meta> metas;
  std::vector<std::string> meta_ids;

  kvs_store(const symsim::GpuProfile& g, const symsim::LinkProfile& l, const symsim::KvStore::Options& o)
      : store(g, l, o) {}

  void clear_out() {
    sched.clear();
    keys.clear();
    times.clear();
  }
  void take(const std::vector<symsim::ScheduledTransfer>& v) {
    for (const auto& t : v) sched.push_back(kvs_scheduled{t.id, t.complete_at});
  }
};

extern "C" {

const char* kvs_last_error(void) { return g_last_error.c_str(); }

int kvs_is_product(void) {
#ifdef KVS_PRODUCT
  return 1;
#else
  return 0;
#endif
}

int kvs_create(const kvs_gpu_profile* gpu, const kvs_link_profile* links, const kvs_options* opts,
               kvs_store** out) {
  return guarded([&] { *out = new kvs_store(to_gpu(gpu), to_links(links), to_opts(opts)); });
}

void kvs_destroy(kvs_store* s) { delete s; }

int kvs_register_session(kvs_store* s, uint32_t session, const char* id, int32_t priority) {
  return guarded([&] {
    s->store.register_session(session, id ? id : "",
                              priority ? symsim::PriorityClass::High : symsim::PriorityClass::Normal);
  });
}

int kvs_finalize_sessions(kvs_store* s) {
  return guarded([&] { s->store.finalize_sessions(); });
}

int kvs_get_counters(kvs_store* s, kvs_counters* out) {
  return guarded([&] {
    out->device_capacity = s->store.device_capacity();
    out->device_used = s->store.device_used();
    out->device_free = s->store.device_free();
    out->host_used = s->store.host_used();
    out->disk_used = s->store.disk_used();
    out->layer_block_bytes = s->store.layer_block_bytes();
  });
}

int kvs_get_session(kvs_store* s, uint32_t session, kvs_session_info* out) {
  return guarded([&] {
    std::memset(out, 0, sizeof(*out));
    out->cached_tokens = s->store.cached_tokens(session);
    out->session_bytes = s->store.session_bytes(session);
    out->fully_device_resident = s->store.fully_device_resident(session);
    out->has_any_copy = s->store.has_any_copy(session);
    out->pending_persists = s->store.pending_persists(session);
    out->migrating_out = s->store.migrating_out(session);
    out->is_active = s->store.is_active(session);
  });
}

int kvs_bytes_for_new_blocks(kvs_store* s, uint32_t session, int64_t new_tokens, int64_t* out) {
  return guarded([&] { *out = s->store.bytes_for_new_blocks(session, new_tokens); });
}
int kvs_bytes_for_load(kvs_store* s, uint32_t session, int64_t* out) {
  return guarded([&] { *out = s->store.bytes_for_load(session); });
}
int kvs_bytes_for_promote(kvs_store* s, uint32_t session, int64_t* out) {
  return guarded([&] { *out = s->store.bytes_for_promote(session); });
}
int kvs_reserve_device(kvs_store* s, int64_t bytes) {
  return guarded([&] { s->store.reserve_device(bytes); });
}
int kvs_unreserve_device(kvs_store* s, int64_t bytes) {
  return guarded([&] { s->store.unreserve_device(bytes); });
}
int kvs_set_active(kvs_store* s, uint32_t session, int32_t active, int64_t now) {
  return guarded([&] { s->store.set_active(session, active != 0, now); });
}

int kvs_append_blocks(kvs_store* s, uint32_t session, int64_t new_tokens, int64_t now) {
  s->clear_out();
  std::vector<symsim::ScheduledTransfer> sched;
  const int rc = guarded([&] {
    for (const auto& k : s->store.append_blocks(session, new_tokens, now, sched))
      s->keys.push_back(kvs_block_key{k.session, k.layer, 0, k.block_index});
  });
  s->take(sched);  // transfers posted before an exception are still in flight
  return rc;
}

int kvs_purge_from_device(kvs_store* s, int64_t bytes_needed, int64_t now, int32_t spare_high_priority,
                          int64_t* freed) {
  s->clear_out();
  std::vector<symsim::ScheduledTransfer> sched;
  const int rc = guarded([&] { *freed = s->store.purge_from_device(bytes_needed, now, spare_high_priority != 0, sched); });
  s->take(sched);
  return rc;
}

int kvs_plan_layerwise_load(kvs_store* s, uint32_t session, int64_t now, int64_t compute_per_layer,
                            int32_t reason, kvs_load_plan* out) {
  s->clear_out();
  std::vector<symsim::ScheduledTransfer> sched;
  const int rc = guarded([&] {
    std::memset(out, 0, sizeof(*out));
    auto plan = s->store.plan_layerwise_load(session, now, compute_per_layer,
                                             static_cast<symsim::TransferReason>(reason), sched);
    if (!plan) return;
    out->has_plan = 1;
    out->any_load = plan->any_load;
    out->decode_start = plan->decode_start;
    out->finish = plan->finish;
    out->total_stall = plan->total_stall;
    s->times.assign(plan->layer_ready.begin(), plan->layer_ready.end());
  });
  s->take(sched);
  return rc;
}

int kvs_promote(kvs_store* s, uint32_t session, int64_t now, kvs_promote_result* out) {
  s->clear_out();
  std::vector<symsim::ScheduledTransfer> sched;
  const int rc = guarded([&] {
    const auto r = s->store.promote(session, now, sched);
    out->device_layers = r.device_layers;
    out->staged_layers = r.staged_layers;
    out->scheduled = r.scheduled;
  });
  s->take(sched);
  return rc;
}

int kvs_offload_session(kvs_store* s, uint32_t session, int64_t now) {
  s->clear_out();
  std::vector<symsim::ScheduledTransfer> sched;
  const int rc = guarded([&] { s->store.offload_session(session, now, sched); });
  s->take(sched);
  return rc;
}

int kvs_release_session(kvs_store* s, uint32_t session, int64_t now) {
  return guarded([&] { s->store.release_session(session, now); });
}
int kvs_mark_migrating_out(kvs_store* s, uint32_t session) {
  return guarded([&] { s->store.mark_migrating_out(session); });
}

int kvs_import_migration(kvs_store* s, uint32_t session, int64_t tokens, int64_t now) {
  s->clear_out();
  return guarded([&] { s->take(s->store.import_migration(session, tokens, now)); });
}

int kvs_apply_transfer(kvs_store* s, uint64_t id, int64_t now, kvs_apply_result* out) {
  return guarded([&] {
    const auto r = s->store.apply_transfer(id, now);
    std::memset(out, 0, sizeof(*out));
    out->session = r.session;
    out->layer = r.layer;
    out->device_layer_ready = r.device_layer_ready;
    out->persists_drained = r.persists_drained;
    out->migration_arrived = r.migration_arrived;
    out->migration_complete = r.migration_complete;
    out->voided = r.voided;
  });
}

int kvs_void_session_loads(kvs_store* s, uint32_t session) {
  return guarded([&] { s->store.void_session_loads(session); });
}
int kvs_void_session_offload(kvs_store* s, uint32_t session) {
  return guarded([&] { s->store.void_session_offload(session); });
}

int kvs_evictable_blocks(kvs_store* s, int32_t spare_high_priority) {
  s->metas.clear();
  s->meta_ids.clear();
  return guarded([&] {
    const auto v = s->store.evictable_blocks(spare_high_priority != 0);
    s->meta_ids.reserve(v.size());
    for (const auto& m : v) s->meta_ids.push_back(m.session_id);
    for (std::size_t i = 0; i < v.size(); ++i) {
      kvs_block_meta out{};
      out.key = kvs_block_key{v[i].key.session, v[i].key.layer, 0, v[i].key.block_index};
      out.session_bytes = v[i].session_bytes;
      out.session_id = s->meta_ids[i].c_str();
      out.pinned = v[i].pinned;
      s->metas.push_back(out);
    }
  });
}

int kvs_check_budgets(kvs_store* s) {
  return guarded([&] { s->store.check_budgets(); });
}

int kvs_device_usage_debug(kvs_store* s, char* buf, size_t cap) {
  return guarded([&] {
    const std::string d = s->store.device_usage_debug();
    if (cap == 0) return;
    const std::size_t n = d.size() < cap - 1 ? d.size() : cap - 1;
    std::memcpy(buf, d.data(), n);
    buf[n] = '\0';
  });
}

size_t kvs_ledger_size(kvs_store* s) { return s->store.ledger().size(); }

int kvs_ledger_copy(kvs_store* s, size_t start, size_t count, kvs_record* out) {
  return guarded([&] {
    const auto& led = s->store.ledger();
    if (start + count > led.size()) throw std::out_of_range("kvs_ledger_copy: range past end");
    for (std::size_t i = 0; i < count; ++i) {
      const auto& r = led[start + i];
      kvs_record o{};
      o.time = r.time;
      o.node = r.node;
      o.session = r.session;
      o.layer_lo = r.layer_lo;
      o.layer_hi = r.layer_hi;
      o.from = static_cast<int32_t>(r.from);
      o.to = static_cast<int32_t>(r.to);
      o.reason = static_cast<int32_t>(r.reason);
      o.bytes = r.bytes;
      out[i] = o;
    }
  });
}

size_t kvs_out_scheduled(kvs_store* s, const kvs_scheduled** out) {
  *out = s->sched.data();
  return s->sched.size();
}
size_t kvs_out_keys(kvs_store* s, const kvs_block_key** out) {
  *out = s->keys.data();
  return s->keys.size();
}
size_t kvs_out_times(kvs_store* s, const int64_t** out) {
  *out = s->times.data();
  return s->times.size();
}
size_t kvs_out_metas(kvs_store* s, const kvs_block_meta** out) {
  *out = s->metas.data();
  return s->metas.size();
}

int kvs_evict_order(const kvs_block_meta* candidates, size_t n, uint32_t* order) {
  return guarded([&] {
    std::vector<symsim::BlockMeta> v(n);
    for (std::size_t i = 0; i < n; ++i) {
      // key.session is not part of the order; it carries the input index so
      // the caller gets the permutation back.
      v[i].key.session = static_cast<std::uint32_t>(i);
      v[i].key.layer = candidates[i].key.layer;
      v[i].key.block_index = candidates[i].key.block_index;
      v[i].session_id = candidates[i].session_id ? candidates[i].session_id : "";
      v[i].session_bytes = candidates[i].session_bytes;
      v[i].pinned = candidates[i].pinned != 0;
    }
    const auto sorted = symsim::evict_order(std::move(v));
    for (std::size_t i = 0; i < n; ++i) order[i] = sorted[i].key.session;
  });
}

int kvs_pipeline_gate(const int64_t* layer_ready, size_t n, int64_t compute_ready, int64_t step_ns,
                      kvs_gate_result* out) {
  return guarded([&] {
    const std::vector<symsim::Ns> ready(layer_ready, layer_ready + n);
    const auto g = symsim::pipeline_gate(ready, compute_ready, step_ns);
    out->first_step_end = g.first_step_end;
    out->gate_start = g.gate_start;
    out->stall = g.stall;
  });
}

int kvs_transfer_time(int64_t bytes, int32_t link, const kvs_link_profile* links, int64_t* out) {
  return guarded([&] { *out = symsim::transfer_time(bytes, static_cast<symsim::Link>(link), to_links(links)); });
}
int kvs_decode_step_time(int32_t batch, const kvs_gpu_profile* gpu, int64_t* out) {
  return guarded([&] { *out = symsim::decode_step_time(batch, to_gpu(gpu)); });
}
int kvs_prefill_time(int64_t tokens, const kvs_gpu_profile* gpu, int64_t* out) {
  return guarded([&] { *out = symsim::prefill_time(tokens, to_gpu(gpu)); });
}
int kvs_kv_bytes_per_layer(int64_t tokens, const kvs_gpu_profile* gpu, int64_t* out) {
  return guarded([&] { *out = symsim::kv_bytes_per_layer(tokens, to_gpu(gpu)); });
}

int kvs_residency(kvs_store* s, uint32_t session, uint16_t layer, uint32_t block, uint8_t* out) {
#ifdef KVS_PRODUCT
  return guarded([&] { *out = s->store.residency(session, layer, block); });
#else
  (void)s, (void)session, (void)layer, (void)block, (void)out;
  g_last_error = "kvs_residency: not available in the oracle build";
  return KVS_ERR_UNSUPPORTED;
#endif
}

// ---- payload (product only) ----------------------------------------------

#ifdef KVS_PRODUCT
}  // extern "C"

#include <map>
#include <memory>
#include <mutex>

#include "symsim/payload.hpp"
#include "symsim/traffic.hpp"

struct kvs_cluster {
  symsim::PayloadCluster cluster;
  std::map<int, std::unique_ptr<symsim::NodePayload>> owned;
  std::mutex mu;
};
struct kvs_payload {
  symsim::NodePayload* node;
  bool owned;
};

namespace {
symsim::PayloadOptions to_payload_opts(const kvs_payload_options* o) {
  symsim::PayloadOptions p;
  p.device = o->device;
  p.layout = kvx_page_layout{o->num_kv_heads, o->head_dim, o->block_tokens, o->dtype};
  p.fill_mode = o->fill_mode;
  p.device_pages = o->device_pages;
  p.host_pages = o->host_pages;
  p.landing_pages = o->landing_pages;
  p.disk_pages = o->disk_pages;
  p.seed = o->seed;
  p.free_running = o->free_running != 0;
  if (o->disk_path) p.disk_path = o->disk_path;
  p.migrate_max_ctas = o->migrate_max_ctas;
  return p;
}
}  // namespace

extern "C" {

int kvs_cluster_create(kvs_cluster** out) {
  return guarded([&] { *out = new kvs_cluster; });
}
void kvs_cluster_destroy(kvs_cluster* c) { delete c; }

int kvs_payload_create(kvs_cluster* c, int32_t node_id, const kvs_payload_options* opts, kvs_payload** out) {
  return guarded([&] {
    auto* node = new symsim::NodePayload(c ? &c->cluster : nullptr, node_id, to_payload_opts(opts));
    *out = new kvs_payload{node, true};
  });
}

void kvs_payload_destroy(kvs_payload* p) {
  if (!p) return;
  if (p->owned) delete p->node;
  delete p;
}

int kvs_attach_payload(kvs_store* s, kvs_payload* p) {
  return guarded([&] { s->store.attach_backend(p ? p->node : nullptr); });
}

int kvs_payload_read_block(kvs_payload* p, uint32_t session, uint16_t layer, uint32_t block, int32_t tier,
                           void* out) {
  return guarded([&] {
    if (!p->node->read_block(session, layer, block, static_cast<symsim::Tier>(tier), out))
      throw std::logic_error("payload: no copy of that block in that tier");
  });
}

int kvs_payload_pages_in_use(kvs_payload* p, int32_t pool, uint64_t* out) {
  return guarded([&] {
    if (pool < 0 || pool > 3) throw std::logic_error("payload: pool index out of range");
    *out = p->node->pages_in_use(static_cast<symsim::NodePayload::Pool>(pool));
  });
}

int kvs_payload_pool_of(kvs_payload* p, uint32_t session, uint16_t layer, uint32_t block, int32_t tier,
                        int32_t* out) {
  return guarded([&] { *out = p->node->pool_of(session, layer, block, static_cast<symsim::Tier>(tier)); });
}

int kvs_payload_bytes_moved(kvs_payload* p, uint64_t* out7) {
  return guarded([&] {
    for (int i = 0; i < 7; ++i) out7[i] = p->node->bytes_moved()[i];
  });
}

int kvs_payload_stats(kvs_payload* p, uint64_t* out7) {
  return guarded([&] {
    out7[0] = p->node->apply_wait_ns();
    out7[1] = p->node->transfers_posted();
    for (int i = 0; i < 4; ++i) out7[2 + i] = p->node->pages_in_flight(static_cast<symsim::NodePayload::Pool>(i));
    out7[6] = p->node->cross_lane_waits();
  });
}

int kvs_payload_host_ns(kvs_payload* p, uint64_t* out8) {
  return guarded([&] {
    for (int i = 0; i < symsim::NodePayload::kHostPhases; ++i) out8[i] = p->node->host_ns()[i];
  });
}

int kvs_payload_block_table(kvs_payload* p, uint32_t session, uint16_t layer, uint32_t n, uint32_t* out) {
  return guarded([&] {
    if (!p->node->device_block_table(session, layer, n, out))
      throw std::logic_error("payload: block not DEVICE-resident");
  });
}

int kvs_payload_pool(kvs_payload* p, int32_t pool, void** out) {
  return guarded([&] {
    if (pool < 0 || pool > 3) throw std::logic_error("payload: pool index out of range");
    *out = p->node->pool(static_cast<symsim::NodePayload::Pool>(pool));
  });
}

int kvs_payload_synchronize(kvs_payload* p) {
  return guarded([&] { p->node->synchronize(); });
}

int kvs_payload_stream(kvs_payload* p, int32_t lane, void** out) {
  return guarded([&] {
    if (lane < 0 || lane >= symsim::NodePayload::kLanes) throw std::logic_error("payload: lane index out of range");
    *out = p->node->stream(static_cast<symsim::NodePayload::LaneId>(lane));
  });
}

int kvs_set_default_payload(kvs_cluster* c, const kvs_payload_options* tmpl, int32_t num_devices) {
  return guarded([&] {
    if (!c || !tmpl) {
      symsim::set_default_tier_backend_factory({});
      return;
    }
    const symsim::PayloadOptions base = to_payload_opts(tmpl);
    const int devices = num_devices > 0 ? num_devices : 1;
    symsim::set_default_tier_backend_factory([c, base, devices](int node_id) -> symsim::TierBackend* {
      std::lock_guard<std::mutex> lock(c->mu);
      auto& slot = c->owned[node_id];
      if (!slot) {
        symsim::PayloadOptions o = base;
        o.device = node_id % devices;
        if (!o.disk_path.empty()) o.disk_path += ".node" + std::to_string(node_id);  // one DISK file per node
        slot = std::make_unique<symsim::NodePayload>(&c->cluster, node_id, o);
      }
      return slot.get();
    });
  });
}

int kvs_cluster_node(kvs_cluster* c, int32_t node_id, kvs_payload** out) {
  return guarded([&] {
    symsim::NodePayload* n = c->cluster.node(node_id);
    if (!n) throw std::logic_error("payload: no such node");
    *out = new kvs_payload{n, false};
  });
}

int kvs_traffic_zipf_turns(uint64_t sessions, double s, double scale, int32_t min_turns, uint64_t seed,
                           int32_t* out) {
  return guarded([&] {
    const auto t = symsim::traffic::zipf_turns(sessions, s, scale, min_turns, seed);
    for (std::size_t i = 0; i < t.size(); ++i) out[i] = t[i];
  });
}

int kvs_traffic_poisson_gaps(uint64_t n, double mean_s, uint64_t seed, int64_t* out) {
  return guarded([&] {
    const auto g = symsim::traffic::poisson_gaps(n, mean_s, seed);
    for (std::size_t i = 0; i < g.size(); ++i) out[i] = g[i];
  });
}

int kvs_traffic_percentile(const double* values, uint64_t n, double q, double* out) {
  return guarded([&] { *out = symsim::traffic::percentile(std::vector<double>(values, values + n), q); });
}

int kvs_traffic_rps_within_slo(const int32_t* users, const double* rps, const double* p50, uint64_t n, double slo,
                               double* out) {
  return guarded([&] {
    std::vector<symsim::traffic::LoadPoint> sweep(n);
    for (uint64_t i = 0; i < n; ++i) sweep[i] = {users[i], rps[i], p50[i]};
    *out = symsim::traffic::rps_within_slo(sweep, slo);
  });
}

}  // extern "C"
#else
#define KVS_NO_PAYLOAD(name, ...)                                        \
  int name(__VA_ARGS__) {                                                \
    g_last_error = #name ": not available in the oracle build";         \
    return KVS_ERR_UNSUPPORTED;                                          \
  }
KVS_NO_PAYLOAD(kvs_cluster_create, kvs_cluster**)
void kvs_cluster_destroy(kvs_cluster*) {}
KVS_NO_PAYLOAD(kvs_payload_create, kvs_cluster*, int32_t, const kvs_payload_options*, kvs_payload**)
void kvs_payload_destroy(kvs_payload*) {}
KVS_NO_PAYLOAD(kvs_attach_payload, kvs_store*, kvs_payload*)
KVS_NO_PAYLOAD(kvs_payload_read_block, kvs_payload*, uint32_t, uint16_t, uint32_t, int32_t, void*)
KVS_NO_PAYLOAD(kvs_payload_pages_in_use, kvs_payload*, int32_t, uint64_t*)
KVS_NO_PAYLOAD(kvs_payload_pool_of, kvs_payload*, uint32_t, uint16_t, uint32_t, int32_t, int32_t*)
KVS_NO_PAYLOAD(kvs_payload_bytes_moved, kvs_payload*, uint64_t*)
KVS_NO_PAYLOAD(kvs_payload_stats, kvs_payload*, uint64_t*)
KVS_NO_PAYLOAD(kvs_payload_host_ns, kvs_payload*, uint64_t*)
KVS_NO_PAYLOAD(kvs_set_default_payload, kvs_cluster*, const kvs_payload_options*, int32_t)
KVS_NO_PAYLOAD(kvs_payload_block_table, kvs_payload*, uint32_t, uint16_t, uint32_t, uint32_t*)
KVS_NO_PAYLOAD(kvs_payload_pool, kvs_payload*, int32_t, void**)
KVS_NO_PAYLOAD(kvs_payload_synchronize, kvs_payload*)
KVS_NO_PAYLOAD(kvs_payload_stream, kvs_payload*, int32_t, void**)
KVS_NO_PAYLOAD(kvs_cluster_node, kvs_cluster*, int32_t, kvs_payload**)
KVS_NO_PAYLOAD(kvs_traffic_zipf_turns, uint64_t, double, double, int32_t, uint64_t, int32_t*)
KVS_NO_PAYLOAD(kvs_traffic_poisson_gaps, uint64_t, double, uint64_t, int64_t*)
KVS_NO_PAYLOAD(kvs_traffic_percentile, const double*, uint64_t, double, double*)
KVS_NO_PAYLOAD(kvs_traffic_rps_within_slo, const int32_t*, const double*, const double*, uint64_t, double, double*)
}  // extern "C"
#endif
