/* kvs.h — C ABI over the per-node tiered KV store (symsim::KvStore).
 *
 * The reference exposes its store only as a C++ class
 * (/root/reference/proj/include/symsim/kvstore.hpp:107-229); it has no FFI.
 * This flat C surface is what a non-C++ host (ctypes, cgo, JNI) binds, and it
 * is compiled twice from one source file (paper_2412_16434_b200/csrc/host/
 * kvs_capi.cpp): into the product library against this repo's KvStore, and
 * into the oracle library (oracle/_ref) against the reference KvStore. The two
 * libraries therefore export byte-identical entry points, which is what the
 * state-parity tests drive side by side.
 *
 * Conventions: every call returns 0 on success or a KVS_ERR_* code; the
 * message of the C++ exception that produced it is kvs_last_error() (thread
 * local). Variable-length results (scheduled transfers, created keys,
 * per-layer plan times, eviction candidates) are left in per-store output
 * buffers read through kvs_out_*(); they stay valid until the next call on the
 * same store. Times are int64 nanoseconds, sizes int64 bytes.
 */
#ifndef KVS_H_
#define KVS_H_

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define KVS_OK 0
#define KVS_ERR_LOGIC 1       /* std::logic_error: contract violation       */
#define KVS_ERR_RUNTIME 2     /* std::runtime_error: resource/config error  */
#define KVS_ERR_OTHER 3       /* any other exception                        */
#define KVS_ERR_UNSUPPORTED 4 /* entry point not available in this build    */

typedef struct kvs_store kvs_store;

typedef struct {
  double prefill_throughput;
  double decode_base_ms;
  double decode_half_batch;
  int64_t hbm_capacity;
  int64_t kv_bytes_per_token;
  int32_t num_layers;
  int32_t curve_points; /* number of (batch, ms) pairs in curve_batch/curve_ms */
  const int32_t* curve_batch;
  const double* curve_ms;
} kvs_gpu_profile; /* reference costmodel.hpp:17-27 */

typedef struct {
  double pcie_bandwidth;
  double disk_bandwidth;
  double network_bandwidth;
  int64_t per_transfer_latency;
} kvs_link_profile; /* reference costmodel.hpp:29-36 */

typedef struct {
  int32_t node_id;
  int32_t block_tokens;
  int64_t device_capacity;
  int64_t host_capacity;
  int64_t disk_capacity;
  int32_t write_behind;
} kvs_options; /* reference kvstore.hpp:109-116 */

typedef struct {
  uint64_t id;
  int64_t complete_at;
} kvs_scheduled; /* ScheduledTransfer, kvstore.hpp:70-73 */

typedef struct {
  uint32_t session;
  uint16_t layer;
  uint16_t pad_;
  uint32_t block_index;
} kvs_block_key; /* BlockKey, kvstore.hpp:24-28 */

typedef struct {
  int64_t time;
  int32_t node;
  uint32_t session;
  uint16_t layer_lo;
  uint16_t layer_hi;
  int32_t from; /* Tier: 0 device, 1 host, 2 disk */
  int32_t to;
  int32_t reason; /* TransferReason: prefetch, demand, purge, persist, migrate */
  int64_t bytes;
} kvs_record; /* TransferRecord, kvstore.hpp:47-57 */

typedef struct {
  uint32_t session;
  uint16_t layer;
  uint8_t device_layer_ready;
  uint8_t persists_drained;
  uint8_t migration_arrived;
  uint8_t migration_complete;
  uint8_t voided;
  uint8_t pad_;
} kvs_apply_result; /* KvStore::ApplyResult, kvstore.hpp:204-212 */

typedef struct {
  int32_t has_plan; /* 0 when the store declined (std::nullopt) */
  int32_t any_load;
  int64_t decode_start;
  int64_t finish;
  int64_t total_stall;
} kvs_load_plan; /* LoadPlan, kvstore.hpp:77-83; layer_ready via kvs_out_times */

typedef struct {
  int32_t device_layers;
  int32_t staged_layers;
  int32_t scheduled;
} kvs_promote_result; /* PromoteResult, kvstore.hpp:98-102 */

typedef struct {
  int64_t first_step_end;
  int64_t gate_start;
  int64_t stall;
} kvs_gate_result; /* GateResult, kvstore.hpp:85-89 */

typedef struct {
  int64_t device_capacity;
  int64_t device_used;
  int64_t device_free;
  int64_t host_used;
  int64_t disk_used;
  int64_t layer_block_bytes;
} kvs_counters;

typedef struct {
  int64_t cached_tokens;
  int64_t session_bytes;
  int32_t fully_device_resident;
  int32_t has_any_copy;
  int32_t pending_persists;
  int32_t migrating_out;
  int32_t is_active;
  int32_t pad_;
} kvs_session_info;

typedef struct {
  kvs_block_key key;
  int64_t session_bytes;
  const char* session_id; /* evict_order input; output points into the store */
  int32_t pinned;
  int32_t pad_;
} kvs_block_meta; /* BlockMeta, kvstore.hpp:32-37 */

const char* kvs_last_error(void);
/* 1 for the product build, 0 for the oracle build of the same source. */
int kvs_is_product(void);

/* replaces symsim::KvStore::KvStore, kvstore.hpp:118 */
int kvs_create(const kvs_gpu_profile* gpu, const kvs_link_profile* links, const kvs_options* opts,
               kvs_store** out);
void kvs_destroy(kvs_store* s);

/* replaces symsim::register_session, kvstore.hpp:120 */
int kvs_register_session(kvs_store* s, uint32_t session, const char* id, int32_t priority);
/* replaces symsim::finalize_sessions, kvstore.hpp:121 */
int kvs_finalize_sessions(kvs_store* s);

int kvs_get_counters(kvs_store* s, kvs_counters* out);
int kvs_get_session(kvs_store* s, uint32_t session, kvs_session_info* out);
/* replaces symsim::bytes_for_new_blocks, kvstore.hpp:133 */
int kvs_bytes_for_new_blocks(kvs_store* s, uint32_t session, int64_t new_tokens, int64_t* out);
/* replaces symsim::bytes_for_load, kvstore.hpp:135 */
int kvs_bytes_for_load(kvs_store* s, uint32_t session, int64_t* out);
/* replaces symsim::bytes_for_promote, kvstore.hpp:137 */
int kvs_bytes_for_promote(kvs_store* s, uint32_t session, int64_t* out);
/* replaces symsim::reserve_device, kvstore.hpp:139 */
int kvs_reserve_device(kvs_store* s, int64_t bytes);
/* replaces symsim::unreserve_device, kvstore.hpp:140 */
int kvs_unreserve_device(kvs_store* s, int64_t bytes);
/* replaces symsim::set_active, kvstore.hpp:149 */
int kvs_set_active(kvs_store* s, uint32_t session, int32_t active, int64_t now);

/* Scheduled transfers -> kvs_out_scheduled; created keys -> kvs_out_keys. */
/* replaces symsim::append_blocks, kvstore.hpp:157 (kvstore.cpp:202-271) */
int kvs_append_blocks(kvs_store* s, uint32_t session, int64_t new_tokens, int64_t now);
/* replaces symsim::purge_from_device, kvstore.hpp:166 (kvstore.cpp:332-431) */
int kvs_purge_from_device(kvs_store* s, int64_t bytes_needed, int64_t now, int32_t spare_high_priority,
                          int64_t* freed);
/* layer_ready -> kvs_out_times. */
/* replaces symsim::plan_layerwise_load, kvstore.hpp:177 (kvstore.cpp:433-543) */
int kvs_plan_layerwise_load(kvs_store* s, uint32_t session, int64_t now, int64_t compute_per_layer,
                            int32_t reason, kvs_load_plan* out);
/* replaces symsim::promote, kvstore.hpp:183 (kvstore.cpp:545-640) */
int kvs_promote(kvs_store* s, uint32_t session, int64_t now, kvs_promote_result* out);
/* replaces symsim::offload_session, kvstore.hpp:188 (kvstore.cpp:642-708) */
int kvs_offload_session(kvs_store* s, uint32_t session, int64_t now);
/* replaces symsim::release_session, kvstore.hpp:191 (kvstore.cpp:710-736) */
int kvs_release_session(kvs_store* s, uint32_t session, int64_t now);
/* replaces symsim::mark_migrating_out, kvstore.hpp:196 (kvstore.cpp:738-742) */
int kvs_mark_migrating_out(kvs_store* s, uint32_t session);
/* replaces symsim::import_migration, kvstore.hpp:200 (kvstore.cpp:744-789) */
int kvs_import_migration(kvs_store* s, uint32_t session, int64_t tokens, int64_t now);
/* replaces symsim::apply_transfer, kvstore.hpp:213 (kvstore.cpp:816-926) */
int kvs_apply_transfer(kvs_store* s, uint64_t id, int64_t now, kvs_apply_result* out);
/* replaces symsim::void_session_loads, kvstore.hpp:218 */
int kvs_void_session_loads(kvs_store* s, uint32_t session);
/* replaces symsim::void_session_offload, kvstore.hpp:219 */
int kvs_void_session_offload(kvs_store* s, uint32_t session);
/* Candidates in eviction order -> kvs_out_metas. */
/* replaces symsim::evictable_blocks, kvstore.hpp:226 (kvstore.cpp:310-330) */
int kvs_evictable_blocks(kvs_store* s, int32_t spare_high_priority);
/* replaces symsim::check_budgets, kvstore.hpp:228 */
int kvs_check_budgets(kvs_store* s);
/* replaces symsim::device_usage_debug, kvstore.hpp:130 */
int kvs_device_usage_debug(kvs_store* s, char* buf, size_t cap);

/* replaces symsim::ledger, kvstore.hpp:221 */
size_t kvs_ledger_size(kvs_store* s);
int kvs_ledger_copy(kvs_store* s, size_t start, size_t count, kvs_record* out);

size_t kvs_out_scheduled(kvs_store* s, const kvs_scheduled** out);
size_t kvs_out_keys(kvs_store* s, const kvs_block_key** out);
size_t kvs_out_times(kvs_store* s, const int64_t** out);
size_t kvs_out_metas(kvs_store* s, const kvs_block_meta** out);

/* Free functions of the reference API. evict_order writes the permutation of
 * the input indices into `order` (n entries). */
/* replaces symsim::evict_order, kvstore.hpp:43 (kvstore.cpp:34-44) */
int kvs_evict_order(const kvs_block_meta* candidates, size_t n, uint32_t* order);
/* replaces symsim::pipeline_gate, kvstore.hpp:96 (kvstore.cpp:46-59) */
int kvs_pipeline_gate(const int64_t* layer_ready, size_t n, int64_t compute_ready, int64_t step_ns,
                      kvs_gate_result* out);
int kvs_transfer_time(int64_t bytes, int32_t link, const kvs_link_profile* links, int64_t* out);
int kvs_decode_step_time(int32_t batch, const kvs_gpu_profile* gpu, int64_t* out);
int kvs_prefill_time(int64_t tokens, const kvs_gpu_profile* gpu, int64_t* out);
int kvs_kv_bytes_per_layer(int64_t tokens, const kvs_gpu_profile* gpu, int64_t* out);

/* Product-only (KVS_ERR_UNSUPPORTED in the oracle build): residency bits
 * (1 << Tier) of one block. */
int kvs_residency(kvs_store* s, uint32_t session, uint16_t layer, uint32_t block, uint8_t* out);

/* ---- Physical payload (product build only; KVS_ERR_UNSUPPORTED in the
 * oracle build). A payload node gives a store's tier copies real pages
 * (include/symsim/payload.hpp): attach one per store, drive the store as
 * usual, read any block copy back for verification. --------------------- */
typedef struct kvs_cluster kvs_cluster;
typedef struct kvs_payload kvs_payload;

typedef struct {
  int32_t device;
  int32_t num_kv_heads;
  int32_t head_dim;
  int32_t block_tokens;
  int32_t dtype; /* KVX_DTYPE_* */
  int32_t fill_mode;
  uint64_t device_pages;
  uint64_t host_pages;
  uint64_t landing_pages;
  uint64_t disk_pages;
  uint64_t seed;
  int32_t free_running; /* 0: lockstep (move at apply); 1: issue at schedule, complete at apply */
  int32_t pad_;
  const char* disk_path; /* NULL/"": DISK tier in pinned host memory; else the file backing it */
  uint32_t migrate_max_ctas; /* cap on the K3 grid of migration pushes (0 = all SMs) */
  uint32_t pad2_;
} kvs_payload_options;

int kvs_cluster_create(kvs_cluster** out);
void kvs_cluster_destroy(kvs_cluster* c);
int kvs_payload_create(kvs_cluster* c, int32_t node_id, const kvs_payload_options* opts, kvs_payload** out);
void kvs_payload_destroy(kvs_payload* p);
/* Attach (or detach with NULL) a payload node to a store. */
int kvs_attach_payload(kvs_store* s, kvs_payload* p);
/* Copies one block's `tier` copy to host memory (page_bytes); KVS_ERR_LOGIC
 * when the node holds no such copy. */
int kvs_payload_read_block(kvs_payload* p, uint32_t session, uint16_t layer, uint32_t block, int32_t tier,
                           void* out);
/* pool: 0 device, 1 pinned host, 2 landing (HBM), 3 disk. */
int kvs_payload_pages_in_use(kvs_payload* p, int32_t pool, uint64_t* out);
int kvs_payload_pool_of(kvs_payload* p, uint32_t session, uint16_t layer, uint32_t block, int32_t tier,
                        int32_t* out);
int kvs_payload_bytes_moved(kvs_payload* p, uint64_t* out7);
/* out[0] = host ns blocked in apply waiting for the GPU (free-running),
 * out[1] = transfers issued at schedule time, out[2..5] = pages of each pool
 * held by moves issued but not yet applied, out[6] = page allocations that
 * had to wait for freed pages still touched by queued batches (quarantine:
 * a freed page is reused only once every batch queued before the free has
 * completed). */
int kvs_payload_stats(kvs_payload* p, uint64_t* out7);
/* Host ns of the payload's bookkeeping by phase (nested phases counted in
 * their callers too): [0] transfer_posted (issue at schedule time), [1]
 * transfer_retired (apply), [2] issue (enqueue of one batch's copies), [4]
 * id upload, [5] mover launches, [6] batch close (event) — [4..6] inside
 * [2] — [7] page allocation, and [3] returning quarantined pages to the
 * free lists (inside [7]). */
int kvs_payload_host_ns(kvs_payload* p, uint64_t* out8);
/* Process-wide default: every KvStore constructed afterwards gets a payload
 * node (node_id -> device node_id % num_devices) in cluster `c`, built from
 * `tmpl`. Lets unchanged caller stacks (the reference Simulation) run with
 * real pages. NULL clears it. Nodes are owned by the cluster. */
/* DEVICE page ids of blocks [0, n) of (session, layer) into out[n] — the
 * block-table row for kvx_decode_attention; KVS_ERR_LOGIC if any block is not
 * DEVICE-resident. The pool itself: kvs_payload_pool (0 device, 1 host,
 * 2 landing, 3 disk) returns the kvx_pool* the pages live in. */
int kvs_payload_block_table(kvs_payload* p, uint32_t session, uint16_t layer, uint32_t n, uint32_t* out);
int kvs_payload_pool(kvs_payload* p, int32_t pool, void** out);
/* Waits for everything queued on the node's lanes (free-running moves). */
int kvs_payload_synchronize(kvs_payload* p);
/* The cudaStream_t of one of the node's lanes: 0 IN (moves landing in HBM),
 * 1 OUT (HBM -> pinned host), 2 DISK (disk-tier reads and writes), 3 PEER
 * (migration pushes into a peer), 4 FILL (content of created blocks).
 * Callers may order their own work against a lane with events; the payload
 * never waits on caller streams. */
int kvs_payload_stream(kvs_payload* p, int32_t lane, void** out);
int kvs_set_default_payload(kvs_cluster* c, const kvs_payload_options* tmpl, int32_t num_devices);
int kvs_cluster_node(kvs_cluster* c, int32_t node_id, kvs_payload** out);

/* ---- serving traffic and latency aggregates (product only;
 * include/symsim/traffic.hpp). The reference synthesizes closed-loop chat
 * traffic with typing-time think pauses (workload.cpp:260-311) and reports
 * means + steady requests/s (report.cpp:65-76); configs 4 and 5 add Poisson
 * think times, Zipf session popularity and p50 service levels. ---------- */
/* out[i] = turns of session i under Zipf(s): seeded ranking, rank r gets
 * max(min_turns, round(scale / r^s)). */
int kvs_traffic_zipf_turns(uint64_t sessions, double s, double scale, int32_t min_turns, uint64_t seed,
                           int32_t* out);
/* n exponential gaps (ns) with mean mean_s seconds. */
int kvs_traffic_poisson_gaps(uint64_t n, double mean_s, uint64_t seed, int64_t* out);
/* q-quantile with linear interpolation (numpy default). */
int kvs_traffic_percentile(const double* values, uint64_t n, double q, double* out);
/* Highest rps among sweep points with p50 <= slo (0 if none). */
int kvs_traffic_rps_within_slo(const int32_t* users, const double* rps, const double* p50, uint64_t n, double slo,
                               double* out);

#ifdef __cplusplus
}
#endif

#endif /* KVS_H_ */
