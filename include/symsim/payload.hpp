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

#include <algorithm>
#include <cstdint>
#include <deque>
#include <initializer_list>
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
  static constexpr int kPools = 4;

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
  // The block-table rows of one layer of a decode step (the GPU engine's
  // quantum, csrc/host/step_executor.cpp): for request i, the DEVICE pages of
  // blocks [0, reqs[i].second) of session reqs[i].first — installed copies,
  // or (free-running) copies a posted load is still moving in — written to
  // out[i * stride ...]. `waits` receives the events of the batches still
  // WRITING any of those pages (fills, layer-wise loads): the decode of the
  // layer waits on exactly those, which is the reference's pipeline gate
  // (kvstore.cpp:46-59) made physical. Reads of the pages (persists,
  // migration pushes) are not waited for. The handles stay valid until the
  // next call that may retire events (any move, apply or sync); collecting
  // every layer's waits first and then issuing them is safe. False if a
  // block has no DEVICE page at all.
  bool decode_rows(const std::vector<std::pair<std::uint32_t, std::uint32_t>>& reqs, std::uint16_t layer,
                   std::uint32_t stride, std::uint32_t* out, std::vector<void*>& waits);
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
  // IN: moves landing in this GPU's HBM (LoadH2D); OUT: HBM -> pinned host
  // (SwapOut, HostCopy); DISK: the disk tier's reads / writes; PEER:
  // migration pushes this node runs into a peer; FILL: K5 content of created
  // blocks (its own lane so a reader of new pages waits for fills only).
  enum LaneId : int { kLaneIn = 0, kLaneOut = 1, kLaneDisk = 2, kLanePeer = 3, kLaneFill = 4, kLanes = 5 };
  void* stream(LaneId lane) const { return lanes_[lane].stream; }
  // Allocations that had to wait (host) for freed pages still read or
  // written by queued batches of some lane (page reuse hazards).
  std::uint64_t cross_lane_waits() const { return quarantine_waits_; }
  // Host ns spent in the payload's bookkeeping, by phase (nested phases are
  // included in their callers').
  enum HostPhase : int {
    kHostPosted = 0,   // transfer_posted (issue at schedule time)
    kHostRetired = 1,  // transfer_retired (apply)
    kHostIssue = 2,    // issue(): enqueue of one batch's copies
    kHostReclaim = 3,  // returning quarantined pages to the free lists
    kHostUpload = 4,   // id staging + upload (inside issue)
    kHostLaunch = 5,   // kvx mover launches (inside issue)
    kHostClose = 6,    // batch event (inside issue)
    kHostAlloc = 7,    // page allocation (includes reclaim)
    kHostPhases = 8
  };
  const std::uint64_t* host_ns() const { return host_ns_; }
  void synchronize();

 private:
  struct Ref {
    std::int8_t pool = -1;
    std::uint32_t page = 0;
  };
  // A block's copies, packed (24 B): slot = pool << 30 | page (kNoPage:
  // none); coming = 1 + the in-flight move (free-running) bringing that tier.
  static constexpr std::uint32_t kNoPage = 0xFFFFFFFFu;
  static std::uint32_t pack(const Ref& r) {
    return r.pool < 0 ? kNoPage : (static_cast<std::uint32_t>(r.pool) << 30) | r.page;
  }
  static Ref unpack(std::uint32_t v) {
    return v == kNoPage ? Ref{} : Ref{static_cast<std::int8_t>(v >> 30), v & 0x3FFFFFFFu};
  }
  struct Copies {
    std::uint32_t slot[3] = {kNoPage, kNoPage, kNoPage};  // indexed by Tier
    std::uint32_t coming[3] = {0, 0, 0};
    Ref tier(int t) const { return unpack(slot[t]); }
    bool empty() const {
      return slot[0] == kNoPage && slot[1] == kNoPage && slot[2] == kNoPage && !coming[0] && !coming[1] &&
             !coming[2];
    }
  };
  // Copies of a (session, layer)'s blocks, indexed by block: one hash lookup
  // per layer, then dense indexing (2,048-block layers at 70B @32K). The
  // FILL-lane ticket of the row's newest created blocks orders readers of
  // those pages behind their content.
  struct Row {
    std::vector<Copies> b;
    std::uint64_t fill_ticket = 0;
  };
  static std::uint64_t row_key(std::uint32_t s, std::uint16_t l) { return (static_cast<std::uint64_t>(s) << 16) | l; }
  const Row* find_row(std::uint32_t s, std::uint16_t l) const;
  const Copies* find(std::uint32_t s, std::uint16_t l, std::uint32_t b) const;
  Row& row(std::uint32_t s, std::uint16_t l) { return rows_[row_key(s, l)]; }
  static Copies& at(Row& r, std::uint32_t b) {
    if (b >= r.b.size()) r.b.resize(static_cast<std::size_t>(b) + 1);
    return r.b[b];
  }
  // Grows the row once to hold every block of `blocks` (not one at() at a time).
  static void presize(Row& r, const std::vector<std::uint32_t>& blocks) {
    if (blocks.empty()) return;
    const std::uint32_t hi = *std::max_element(blocks.begin(), blocks.end());
    if (hi >= r.b.size()) r.b.resize(static_cast<std::size_t>(hi) + 1);
  }
  void drop_row_if_empty(std::uint32_t s, std::uint16_t l);

  // A stream plus the events of its batches still possibly running; batch
  // tickets increase by one per batch and complete in order.
  struct Lane {
    void* stream = nullptr;
    std::uint64_t next = 1;  // ticket of the next batch
    std::uint64_t done = 0;  // every ticket <= done has completed
    std::vector<std::pair<std::uint64_t, void*>> pending;  // (ticket, event), ascending
    std::uint32_t* d_ids = nullptr;  // page-id scratch for this lane's kernels (one batch)
    std::size_t d_ids_cap = 0;
    // Pinned staging for id / tag uploads, so they are true async copies:
    // a region is reused once the batch (ticket) that uploaded it completed.
    std::uint8_t* ring = nullptr;
    std::size_t ring_cap = 0, ring_head = 0;
    struct Region {
      std::size_t begin, end;
      std::uint64_t ticket;
    };
    std::deque<Region> ring_used;  // FIFO
    kvx_pool* bounce = nullptr;  // pinned staging between HBM and a file-backed DISK pool
    void retire();
    void* event_for(std::uint64_t ticket);  // nullptr once complete
    void* find_pending(std::uint64_t ticket) const;  // same, without retiring
    void drain();                           // after a stream sync: everything complete
    std::uint64_t last() const { return next - 1; }
  };
  static constexpr std::size_t kBouncePages = 256;  // per-lane HBM <-> disk-file staging
  struct HostTimer;
  struct NodeCache {
    int ids[8];
    NodePayload* nodes[8];
    int n = 0;
    NodePayload* get(PayloadCluster* cluster, int id);
  };
  // Event of `node`'s `lane` batch `ticket`, or nullptr once it completed.
  void* pending_event(NodePayload* node, int lane, std::uint64_t ticket) const;

  // Freed pages wait in quarantine until every batch issued (on any lane of
  // any node) before they were freed has completed: a page still read by a
  // queued persist or migration push, or still written by a voided move, is
  // never handed to a new writer. This replaces per-page fences: no batch
  // reads or writes per-page hazard state.
  struct Held {
    std::vector<std::pair<std::pair<int, int>, std::uint64_t>> marks;  // ((node, lane), ticket)
    std::vector<Ref> pages;
  };
  void seal_released();
  bool reclaim(bool wait_for_oldest);

  struct InFlight {  // a free-running move: pages being written by `event`
    std::uint64_t id = 0;
    int tier = 0;
    std::uint32_t session = 0;
    std::uint16_t layer = 0;
    std::vector<std::uint32_t> blocks;  // ascending
    std::vector<Ref> pages;
    void* event = nullptr;
  };
  InFlight& flight(std::uint32_t coming) { return flights_[coming - 1]; }
  const InFlight& flight(std::uint32_t coming) const { return flights_[coming - 1]; }
  static Ref flight_page(const InFlight& f, std::uint32_t b);
  static void reset_flight(InFlight& f);
  void give_back(const Ref* pages, std::size_t n);
  std::uint32_t alloc(Pool p);
  void alloc_n(Pool p, std::size_t n, std::vector<std::uint32_t>& out);
  void release(const Ref& r);
  Ref best_source(std::uint32_t s, std::uint16_t l, std::uint32_t b, int exclude_tier) const;
  // In-flight copy of a block (fastest tier first): page + the event that
  // completes it; returns false if none.
  bool inflight_source(std::uint32_t s, std::uint16_t l, std::uint32_t b, int exclude_tier, Ref* page,
                       void** event) const;
  // Issues src[i] -> dst[i] copies on the runner's stream, grouped by pools.
  // Queues the moves on the lane the destination implies (after `waits` and
  // the fill of the source row, `src_fill`); returns the lane's stream.
  void* issue(const std::vector<Ref>& src, const std::vector<Ref>& dst, NodePayload& src_node, bool push,
              const std::vector<void*>& waits, std::uint64_t src_fill);
  // Records the batch just queued on `lane`; returns its ticket.
  std::uint64_t close_batch(int lane);
  void move_now(std::uint32_t session, std::uint16_t layer, Tier tier, BlockEvent why,
                const std::vector<std::uint32_t>& blocks);
  std::uint32_t* upload_ids(Lane& lane, const std::uint32_t* staged, std::size_t n);
  std::uint32_t* device_ids(Lane& lane, const std::vector<std::uint32_t>& ids);
  void* stage(Lane& lane, std::size_t bytes);
  void check_file_io() const;

  PayloadCluster* cluster_;
  int node_;
  PayloadOptions opts_;
  std::uint64_t page_bytes_ = 0;
  kvx_pool* pools_[4] = {nullptr, nullptr, nullptr, nullptr};
  std::vector<std::uint32_t> free_[4];
  std::vector<Ref> released_;      // freed since the last seal
  std::deque<Held> quarantine_;    // sealed groups, FIFO
  std::uint64_t held_[4] = {0, 0, 0, 0};  // pages per pool in released_ + quarantine_
  std::uint64_t quarantine_waits_ = 0;
  std::unordered_map<std::uint64_t, Row> rows_;
  std::map<std::uint32_t, int> import_src_;
  Lane lanes_[kLanes];
  void* d_tags_ = nullptr;  // fill ids + tags (FILL lane)
  std::size_t d_tags_cap_ = 0;
  std::uint64_t moved_[8] = {0, 0, 0, 0, 0, 0, 0, 0};
  // free-running state
  std::vector<InFlight> flights_;              // slots; coming = slot + 1
  std::vector<std::uint32_t> free_flights_;
  std::unordered_map<std::uint64_t, std::uint32_t> flight_of_;  // transfer id -> slot
  std::uint64_t applying_ = 0;
  bool applying_valid_ = false;
  std::uint64_t apply_wait_ns_ = 0;
  std::uint64_t posted_ = 0;
  std::uint64_t host_ns_[kHostPhases] = {};
  std::vector<Ref> scratch_src_;  // transfer_posted scratch (reused)
  std::vector<void*> scratch_waits_;
  std::vector<std::uint32_t> scratch_pages_;
};

}  // namespace symsim
