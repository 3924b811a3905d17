#pragma once
// Physical KV payload behind the tiered store — B200 build.
//
// NodePayload implements TierBackend (kvstore.hpp): it gives every block
// copy the state machine creates a real page and moves the bytes with the
// kvx_* kernels / copy engines (include/kvx.h):
//
//   DEVICE copy  -> a page of this node's HBM pool
//                   Created   : allocated + filled (K5 / the engine's writes)
//                   LoadH2D   : K3 page copy from the HOST copy (landing pool:
//                               HBM->HBM, the device-local "unpack"; pinned
//                               host: copy engines over PCIe) or DISK copy
//   HOST copy    -> a page of the pinned host pool (HostCopy / SwapOut /
//                   LoadDiskHost, copy engines), or — for blocks that arrived
//                   by migration — a page of this GPU's LANDING pool
//                   (NetArrive: K3 kernel on the source GPU storing straight
//                   into it over NVLink / peer memory)
//   DISK copy    -> a page of the disk pool: a file when disk_path is set
//                   (preads / pwrites in stream order, O_DIRECT where the
//                   filesystem allows; HBM <-> file through a pinned bounce
//                   ring per lane), else pinned host memory standing in for
//                   the SSD (copy engines)
//
// Two modes (SURVEY.md §7 hard part 1):
//   lockstep      every move happens inside apply_transfer, synchronously:
//                 the simplest proof that bytes follow the state.
//   free-running  a move is issued on the node's stream when the store
//                 SCHEDULES it (transfer_posted), chained behind in-flight
//                 sources with CUDA events, and completed when the store
//                 applies it (the apply waits on the transfer's event —
//                 "apply_transfer on CUDA-event completion").
//                 The host only blocks if the GPU is behind the cost model's
//                 clock; that wait is accounted in apply_wait_ns().
// Moves run on four lanes (CUDA streams) per node so independent queues
// overlap the way the hardware allows: IN (anything landing in this GPU's
// HBM: fills, LoadH2D), OUT (HBM -> pinned host: SwapOut, HostCopy), DISK
// (DiskWrite, LoadDiskHost: the reference's separate disk queues) and PEER
// (migration pushes this node runs into a peer's landing pool). PCIe is full
// duplex, so an offload and a prefetch proceed at once. Hazards across lanes are tracked per page: every page
// remembers the last (node, lane, batch) that touched it, and a batch waits
// on the events of the other lanes' batches that still touch its pages.
// In both modes the event order is the reference clock's (apply in
// (complete_at, id) order), so block-table state is bit-identical to the
// reference and every copy's bytes can be verified. Migrated layers land in
// receiver-GPU memory while the ledger still says Host (kvstore.cpp:914-923),
// which keeps ledger parity exact (SURVEY.md §7 hard part 2, option 1).

#include <cstdint>
#include <map>
#include <string>
#include <unordered_map>
#include <vector>

#include "kvx.h"
#include "symsim/kvstore.hpp"

namespace symsim {

struct PayloadOptions {
  int device = 0;
  kvx_page_layout layout{8, 128, 16, KVX_DTYPE_BF16};
  std::uint64_t device_pages = 0;   // HBM pool
  std::uint64_t host_pages = 0;     // pinned host pool (HOST tier)
  std::uint64_t landing_pages = 0;  // HBM pool for migrated HOST-tier copies
  std::uint64_t disk_pages = 0;     // DISK tier: pages in disk_path, or pinned host if empty
  std::string disk_path;            // file backing the DISK tier (created / grown; kept)
  std::uint32_t migrate_max_ctas = 0;  // cap on the K3 grid of migration pushes (0 = all SMs)
  std::uint64_t seed = 0;           // content of Created blocks
  int fill_mode = KVX_FILL_VALUES;
  bool free_running = false;
};

class NodePayload;

// Process-wide view of the nodes, so a receiver can find the migration
// source of a session (Simulation::start_migration, simcore.cpp:132-141,
// freezes the source and then imports on the receiver).
class PayloadCluster {
 public:
  void add(NodePayload* node);
  void remove(NodePayload* node);
  NodePayload* node(int id) const;
  std::vector<NodePayload*> nodes() const;
  void note_source(std::uint32_t session, int node);
  int take_source(std::uint32_t session);

 private:
  std::map<int, NodePayload*> nodes_;
  std::map<std::uint32_t, int> sources_;
};

class NodePayload final : public TierBackend {
 public:
  enum Pool : int { kDevicePool = 0, kHostPool = 1, kLandingPool = 2, kDiskPool = 3 };

  NodePayload(PayloadCluster* cluster, int node_id, const PayloadOptions& opts);
  ~NodePayload() override;
  NodePayload(const NodePayload&) = delete;
  NodePayload& operator=(const NodePayload&) = delete;

  void tier_gained(std::uint32_t session, std::uint16_t layer, Tier tier, BlockEvent why,
                   const std::vector<std::uint32_t>& blocks) override;
  void tier_lost(std::uint32_t session, std::uint16_t layer, Tier tier,
                 const std::vector<std::uint32_t>& blocks) override;
  void transfer_posted(const TransferInfo& t) override;
  void transfer_retired(std::uint64_t id, bool voided) override;
  void migrating_out(std::uint32_t session) override;
  void importing(std::uint32_t session, std::int64_t tokens) override;

  int node_id() const { return node_; }
  int device() const { return opts_.device; }
  const PayloadOptions& options() const { return opts_; }
  std::uint64_t page_bytes() const { return page_bytes_; }
  std::uint64_t pages_in_use(Pool p) const;
  // Copies the bytes of one block's copy in `tier` to host memory; false if
  // this node holds no such copy.
  bool read_block(std::uint32_t session, std::uint16_t layer, std::uint32_t block, Tier tier, void* out);
  // DEVICE page ids of blocks [0, n) of (session, layer) — the block-table
  // row a decode-attention launch consumes (kvx_decode_attention). False if
  // any of them is not DEVICE-resident.
  bool device_block_table(std::uint32_t session, std::uint16_t layer, std::uint32_t n, std::uint32_t* out) const;
  // Which pool holds the block's `tier` copy (-1: none).
  int pool_of(std::uint32_t session, std::uint16_t layer, std::uint32_t block, Tier tier) const;
  // Bytes moved per BlockEvent kind since construction.
  const std::uint64_t* bytes_moved() const { return moved_; }
  // Free-running: host nanoseconds spent waiting in apply for the GPU, and
  // the number of transfers issued at schedule time.
  std::uint64_t apply_wait_ns() const { return apply_wait_ns_; }
  std::uint64_t transfers_posted() const { return posted_; }
  // Free-running: pages of `p` held by moves issued but not yet applied.
  std::uint64_t pages_in_flight(Pool p) const;
  kvx_pool* pool(Pool p) const { return pools_[p]; }
  enum LaneId : int { kLaneIn = 0, kLaneOut = 1, kLaneDisk = 2, kLanePeer = 3, kLanes = 4 };
  void* stream(LaneId lane) const { return lanes_[lane].stream; }
  // Batches that had to wait on another lane's batch (page reuse hazards).
  std::uint64_t cross_lane_waits() const { return cross_waits_; }
  void synchronize();

 private:
  struct Ref {
    std::int8_t pool = -1;
    std::uint32_t page = 0;
  };
  struct Copies {
    Ref tier[3];  // indexed by Tier
  };
  // A stream plus the events of its batches still possibly running; batch
  // tickets increase by one per batch.
  struct Lane {
    void* stream = nullptr;
    std::uint64_t next = 1;  // ticket of the next batch
    std::uint64_t done = 0;  // every ticket <= done has completed
    std::vector<std::pair<std::uint64_t, void*>> pending;  // (ticket, event), ascending
    std::uint32_t* d_ids[2] = {nullptr, nullptr};           // page-id scratch for this lane's kernels
    std::size_t d_ids_cap[2] = {0, 0};
    kvx_pool* bounce = nullptr;  // pinned staging between HBM and a file-backed DISK pool
    void retire();
    void* event_for(std::uint64_t ticket);  // nullptr once complete
    void drain();                           // after a stream sync: everything complete
  };
  static constexpr std::size_t kBouncePages = 256;  // per-lane HBM <-> disk-file staging
  struct Fence {  // the last batch that read or wrote a page
    std::int32_t node = -1;
    std::int32_t lane = 0;
    std::uint64_t ticket = 0;
  };
  using Touch = std::pair<NodePayload*, Ref>;  // a page of some node's pool
  void wait_fences(NodePayload& runner, int lane, const std::vector<Touch>& pages);
  void set_fences(NodePayload& runner, int lane, const std::vector<Touch>& pages);
  Fence& fence(const Ref& r) { return fences_[r.pool][r.page]; }

  struct InFlight {  // a free-running move: pages being written by `event`
    int tier = 0;
    std::uint32_t session = 0;
    std::uint16_t layer = 0;
    std::vector<std::uint32_t> blocks;
    std::vector<Ref> pages;
    void* event = nullptr;
  };
  static std::uint64_t key(std::uint32_t s, std::uint16_t l, std::uint32_t b) {
    return (static_cast<std::uint64_t>(s) << 36) | (static_cast<std::uint64_t>(l) << 20) | b;
  }
  std::uint32_t alloc(Pool p);
  void release(const Ref& r);
  Ref best_source(std::uint32_t s, std::uint16_t l, std::uint32_t b, int exclude_tier) const;
  // In-flight copy of a block (fastest tier first): page + the event that
  // completes it; returns false if none.
  bool inflight_source(std::uint32_t s, std::uint16_t l, std::uint32_t b, int exclude_tier, Ref* page,
                       void** event) const;
  // Issues src[i] -> dst[i] copies on the runner's stream, grouped by pools.
  // Queues the moves on the lane the destination implies; returns the lane's stream.
  void* issue(const std::vector<Ref>& src, const std::vector<Ref>& dst, NodePayload& src_node, bool push,
              const std::vector<void*>& waits);
  void move_now(std::uint32_t session, std::uint16_t layer, Tier tier, BlockEvent why,
                const std::vector<std::uint32_t>& blocks);
  std::uint32_t* device_ids(Lane& lane, const std::vector<std::uint32_t>& ids, int slot);
  void check_file_io() const;

  PayloadCluster* cluster_;
  int node_;
  PayloadOptions opts_;
  std::uint64_t page_bytes_ = 0;
  kvx_pool* pools_[4] = {nullptr, nullptr, nullptr, nullptr};
  std::vector<std::uint32_t> free_[4];
  std::unordered_map<std::uint64_t, Copies> blocks_;
  std::map<std::uint32_t, int> import_src_;
  Lane lanes_[kLanes];
  std::vector<Fence> fences_[4];  // per pool page
  std::uint64_t cross_waits_ = 0;
  // Device id scratch lives per lane (Lane::d_ids): reuse is safe without
  // host syncs because uploads and the kernels reading them share the lane's
  // stream. Tag scratch is used by fills, which run on the IN lane.
  void* d_tags_ = nullptr;
  std::size_t d_tags_cap_ = 0;
  std::uint64_t moved_[8] = {0, 0, 0, 0, 0, 0, 0, 0};
  // free-running state
  std::unordered_map<std::uint64_t, InFlight> inflight_;        // by transfer id
  struct InFlightSlot {
    std::uint64_t id;      // transfer
    std::uint32_t index;   // position of the block in that transfer's InFlight lists
  };
  std::unordered_map<std::uint64_t, InFlightSlot> inflight_by_block_;  // key*4+tier -> slot
  std::uint64_t applying_ = 0;
  bool applying_valid_ = false;
  std::uint64_t apply_wait_ns_ = 0;
  std::uint64_t posted_ = 0;
};

}  // namespace symsim
