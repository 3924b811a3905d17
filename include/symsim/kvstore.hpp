#pragma once
// Per-node tiered KV block store — B200 build.
//
// This header is the drop-in boundary on the host side. Its
// public surface is source-compatible with the reference
// /root/reference/proj/include/symsim/kvstore.hpp:16-229, so the reference's
// callers (Engine, NodeManager, ClusterScheduler, Simulation) compile and run
// against it unchanged (tests/cpp/build_ref_harness.sh does exactly that).
//
// What is new relative to the reference:
//   * the private representation (one flag byte per block, per-session
//     in-flight lists, see kvstore.cpp), re-implemented from SPEC.md:220-329;
//   * a physical backing hook (TierBackend): every residency transition the
//     state machine applies is reported, batched per (session, layer, tier),
//     so a backend can give DEVICE blocks real HBM pages and move their bytes
//     with the kvx_* kernels (include/kvx.h). Without a backend the store is a
//     pure accounting model, exactly like the reference.

#include <cstdint>
#include <functional>
#include <map>
#include <optional>
#include <string>
#include <unordered_map>
#include <vector>

#include "symsim/costmodel.hpp"
#include "symsim/time.hpp"
#include "symsim/workload.hpp"

namespace symsim {

enum class Tier : unsigned { Device = 0, Host = 1, Disk = 2 };
const char* tier_name(Tier t);

enum class TransferReason { Prefetch, Demand, Purge, Persist, Migrate };
const char* reason_name(TransferReason r);

struct BlockKey {
  std::uint32_t session = 0;
  std::uint16_t layer = 0;
  std::uint32_t block_index = 0;
};

// Eviction candidate; session_bytes is the owner's whole-cache footprint.
struct BlockMeta {
  BlockKey key;
  std::string session_id;
  std::int64_t session_bytes = 0;
  bool pinned = false;
};

// Total eviction order: layer desc, session_bytes asc, block_index desc,
// session_id asc. Pinned candidates are rejected.
std::vector<BlockMeta> evict_order(std::vector<BlockMeta> candidates);

// Transfer ledger row; `time` is the completion instant.
struct TransferRecord {
  Ns time = 0;
  int node = 0;
  std::uint32_t session = 0;
  std::uint16_t layer_lo = 0;
  std::uint16_t layer_hi = 0;  // inclusive
  Tier from = Tier::Device;
  Tier to = Tier::Device;
  std::int64_t bytes = 0;
  TransferReason reason = TransferReason::Demand;
};

// FIFO link: completion is fixed when a transfer is enqueued.
struct Channel {
  Ns busy_until = 0;
  Ns enqueue(Ns ready, Ns duration) {
    busy_until = (ready > busy_until ? ready : busy_until) + duration;
    return busy_until;
  }
};

struct ScheduledTransfer {
  std::uint64_t id = 0;  // node-local
  Ns complete_at = 0;
};

struct LoadPlan {
  std::vector<Ns> layer_ready;
  Ns decode_start = 0;
  Ns finish = 0;
  Ns total_stall = 0;
  bool any_load = false;
};

struct GateResult {
  Ns first_step_end = 0;
  Ns gate_start = 0;
  Ns stall = 0;
};

// e(i) = max(e(i-1), layer_ready[i]) + c_i with e(-1) = compute_ready and
// integer c_i summing exactly to step_ns. On the GPU the same recurrence is
// realised physically: decode of layer i waits on layer i's arrival event.
GateResult pipeline_gate(const std::vector<Ns>& layer_ready, Ns compute_ready, Ns step_ns);

struct PromoteResult {
  int device_layers = 0;
  int staged_layers = 0;
  bool scheduled = false;
};

// ---------------------------------------------------------------------------
// Physical backing (B200 extension, not part of the reference API).

// Why a block gained a tier copy; mirrors the transfer kinds plus creation.
enum class BlockEvent : std::uint8_t {
  Created,       // append_blocks: fresh DEVICE block (engine writes its K/V)
  LoadH2D,       // HOST (or landing buffer) -> DEVICE
  LoadDiskHost,  // DISK -> HOST
  HostCopy,      // write-behind DEVICE -> HOST
  DiskWrite,     // write-behind -> DISK
  SwapOut,       // offload / purge flush DEVICE -> HOST
  NetArrive,     // migration from the source node lands here
};
const char* block_event_name(BlockEvent e);

class TierBackend {
 public:
  virtual ~TierBackend() = default;
  // `blocks` gained a copy in `tier` (ascending block indices, one layer).
  // Called after the state machine has decided the transition and before any
  // copy it supersedes is dropped, so the backend can source the bytes.
  virtual void tier_gained(std::uint32_t session, std::uint16_t layer, Tier tier, BlockEvent why,
                           const std::vector<std::uint32_t>& blocks) = 0;
  // `blocks` lost their copy in `tier`; the backend frees the pages.
  virtual void tier_lost(std::uint32_t session, std::uint16_t layer, Tier tier,
                         const std::vector<std::uint32_t>& blocks) = 0;
  // Free-running backends start a transfer's physical move when the store
  // schedules it (its completion time is fixed by the cost model at that
  // point) and finish it when the store applies it; `transfer_retired` comes
  // first in apply_transfer, before the tier_gained/tier_lost reports of that
  // transfer. Lockstep backends ignore both and move at tier_gained time.
  struct TransferInfo {
    std::uint64_t id = 0;
    std::uint32_t session = 0;
    std::uint16_t layer = 0;
    std::uint32_t block_lo = 0, block_hi = 0;  // inclusive
    BlockEvent kind = BlockEvent::LoadH2D;
    Tier to = Tier::Device;
    std::int64_t bytes = 0;
    Ns complete_at = 0;
  };
  virtual void transfer_posted(const TransferInfo& t) { (void)t; }
  virtual void transfer_retired(std::uint64_t id, bool voided) {
    (void)id;
    (void)voided;
  }
  // Migration endpoints: the source froze `session`; this node imports it.
  virtual void migrating_out(std::uint32_t session) { (void)session; }
  virtual void importing(std::uint32_t session, std::int64_t tokens) {
    (void)session;
    (void)tokens;
  }
};

// Process-wide factory consulted by every KvStore constructor when set, so an
// unchanged caller stack (e.g. the reference Simulation) builds stores that
// are physically backed. Pass an empty function to clear it.
using TierBackendFactory = std::function<TierBackend*(int node_id)>;
void set_default_tier_backend_factory(TierBackendFactory factory);

// ---------------------------------------------------------------------------

class KvStore {
 public:
  struct Options {
    int node_id = 0;
    int block_tokens = 16;
    std::int64_t device_capacity = 0;  // 0: gpu.hbm_capacity
    std::int64_t host_capacity = 256'000'000'000;
    std::int64_t disk_capacity = -1;  // -1: unbounded
    bool write_behind = true;
  };

  KvStore(const GpuProfile& gpu, const LinkProfile& links, const Options& opts);

  void register_session(std::uint32_t session, const std::string& id, PriorityClass priority);
  void finalize_sessions();

  // ---- capacity ----
  std::int64_t device_capacity() const { return device_cap_; }
  std::int64_t device_used() const { return used_[0]; }
  std::int64_t device_free() const { return device_cap_ - used_[0]; }
  std::int64_t host_used() const { return used_[1]; }
  std::int64_t disk_used() const { return used_[2]; }
  std::int64_t layer_block_bytes() const { return page_bytes_; }
  std::string device_usage_debug() const;

  std::int64_t bytes_for_new_blocks(std::uint32_t session, std::int64_t new_tokens) const;
  std::int64_t bytes_for_load(std::uint32_t session) const;
  std::int64_t bytes_for_promote(std::uint32_t session) const;

  void reserve_device(std::int64_t bytes);
  void unreserve_device(std::int64_t bytes);

  // ---- cache state ----
  std::int64_t cached_tokens(std::uint32_t session) const;
  std::int64_t session_bytes(std::uint32_t session) const;
  bool fully_device_resident(std::uint32_t session) const;
  bool has_any_copy(std::uint32_t session) const;
  int pending_persists(std::uint32_t session) const;
  bool migrating_out(std::uint32_t session) const;
  void set_active(std::uint32_t session, bool active, Ns now);
  bool is_active(std::uint32_t session) const;

  // ---- engine-side operations ----
  std::vector<BlockKey> append_blocks(std::uint32_t session, std::int64_t new_tokens, Ns now,
                                      std::vector<ScheduledTransfer>& scheduled);
  std::int64_t purge_from_device(std::int64_t bytes_needed, Ns now, bool spare_high_priority,
                                 std::vector<ScheduledTransfer>& scheduled);
  std::optional<LoadPlan> plan_layerwise_load(std::uint32_t session, Ns now,
                                              Ns compute_per_layer, TransferReason reason,
                                              std::vector<ScheduledTransfer>& scheduled);
  PromoteResult promote(std::uint32_t session, Ns now, std::vector<ScheduledTransfer>& scheduled);
  void offload_session(std::uint32_t session, Ns now, std::vector<ScheduledTransfer>& scheduled);
  void release_session(std::uint32_t session, Ns now);

  // ---- migration ----
  void mark_migrating_out(std::uint32_t session);
  std::vector<ScheduledTransfer> import_migration(std::uint32_t session, std::int64_t tokens,
                                                  Ns now);

  // ---- completion dispatch ----
  struct ApplyResult {
    std::uint32_t session = 0;
    std::uint16_t layer = 0;
    bool device_layer_ready = false;
    bool persists_drained = false;
    bool migration_arrived = false;
    bool migration_complete = false;
    bool voided = false;
  };
  ApplyResult apply_transfer(std::uint64_t id, Ns now);

  void void_session_loads(std::uint32_t session);
  void void_session_offload(std::uint32_t session);

  const std::vector<TransferRecord>& ledger() const { return ledger_; }
  std::vector<TransferRecord> take_ledger() { return std::move(ledger_); }

  std::vector<BlockMeta> evictable_blocks(bool spare_high_priority) const;

  void check_budgets() const;

  // ---- B200 extension ----
  void attach_backend(TierBackend* backend) { backend_ = backend; }
  TierBackend* backend() const { return backend_; }
  int num_layers() const { return gpu_.num_layers; }
  int block_tokens() const { return opts_.block_tokens; }
  // Residency bits (1 << Tier) of one block, 0 when absent. Used by the
  // payload verifier to decide which physical copies must exist.
  std::uint8_t residency(std::uint32_t session, std::uint16_t layer, std::uint32_t block) const;
  std::size_t blocks_in_layer(std::uint32_t session, std::uint16_t layer) const;
  std::size_t inflight_transfers() const { return inflight_.size(); }

 private:
  // Per-block flag byte. Bits 0-2 are residency, indexed by Tier.
  static constexpr std::uint8_t kOnDev = 1u << 0;
  static constexpr std::uint8_t kOnHost = 1u << 1;
  static constexpr std::uint8_t kOnDisk = 1u << 2;
  static constexpr std::uint8_t kResidency = kOnDev | kOnHost | kOnDisk;
  static constexpr std::uint8_t kBacked = kOnHost | kOnDisk;
  static constexpr std::uint8_t kDiskPending = 1u << 3;
  static constexpr std::uint8_t kHostPending = 1u << 4;
  static constexpr std::uint8_t kDropOnPersist = 1u << 5;
  static constexpr std::uint8_t kLoadPending = 1u << 6;

  using Layer = std::vector<std::uint8_t>;

  struct Session {
    std::string name;
    PriorityClass priority = PriorityClass::Normal;
    int lex_rank = 0;
    std::int64_t tokens = 0;
    bool active = false;
    bool leaving = false;  // migrating out
    Ns last_use = 0;
    int persists_in_flight = 0;
    int inbound_layers = 0;
    std::vector<Layer> layers;
    std::vector<Ns> load_eta;
    std::vector<Ns> inbound_eta;
  };

  enum class Kind : std::uint8_t { LoadH2D, LoadDiskHost, HostCopy, DiskWrite, SwapOut, NetArrive };

  struct Move {
    std::uint32_t session = 0;
    std::uint16_t layer = 0;
    std::uint32_t lo = 0, hi = 0;  // inclusive block range
    Kind kind = Kind::LoadH2D;
    std::int64_t bytes = 0;
    TransferReason reason = TransferReason::Demand;
    bool voided = false;
    Ns complete_at = 0;
  };

  Session& sess(std::uint32_t session);
  const Session& sess(std::uint32_t session) const;
  std::int64_t blocks_of(const Session& s) const;
  std::int64_t footprint(const Session& s) const;
  bool make_host_room(std::int64_t bytes, Ns now);
  bool evict_host_lru(std::int64_t bytes_needed, Ns now);
  Ns link_done(Channel& ch, Ns ready, std::int64_t bytes, Link link);
  std::uint64_t post(const Move& m, std::vector<ScheduledTransfer>& scheduled);
  void log(Ns time, std::uint32_t session, int layer_lo, int layer_hi, Tier from, Tier to,
           std::int64_t bytes, TransferReason reason);
  void clear_drop_marks(Session& s);
  void report_gain(std::uint32_t session, std::uint16_t layer, Tier tier, BlockEvent why,
                   const std::vector<std::uint32_t>& blocks);
  void report_loss(std::uint32_t session, std::uint16_t layer, Tier tier,
                   const std::vector<std::uint32_t>& blocks);

  GpuProfile gpu_;
  LinkProfile links_;
  Options opts_;
  std::int64_t device_cap_ = 0;
  std::int64_t page_bytes_ = 0;  // one layer of one block
  std::int64_t used_[3] = {0, 0, 0};
  Channel pcie_up_, pcie_down_, disk_in_, disk_out_, net_rx_;
  std::map<std::uint32_t, Session> sessions_;  // ordered: deterministic sweeps
  std::unordered_map<std::uint64_t, Move> inflight_;
  std::uint64_t next_id_ = 1;
  std::vector<TransferRecord> ledger_;
  bool finalized_ = false;
  TierBackend* backend_ = nullptr;
};

}  // namespace symsim
