// NodePayload: physical pages behind KvStore's tier residency.
// See include/symsim/payload.hpp for the tier -> pool mapping and the two
// modes. All CUDA work goes through the kvx C ABI (include/kvx.h); this file
// has no CUDA headers.
//
// Reference anchors for when each copy comes into existence (the hooks fire
// from the re-implemented state machine at exactly these points):
//   Created      append_blocks            kvstore.cpp:221-228
//   HostCopy     write-behind landing     kvstore.cpp:867-880
//   DiskWrite    persist landing          kvstore.cpp:881-900
//   SwapOut      offload / purge flush    kvstore.cpp:901-913
//   LoadDiskHost disk stage landing       kvstore.cpp:862-866
//   LoadH2D      demand / prefetch load   kvstore.cpp:852-861
//   NetArrive    migration layer landing  kvstore.cpp:914-923
//   tier_lost    purge / evict / release  kvstore.cpp:388-393, 293-295, 710-736
// Free-running mode issues each move when the transfer is scheduled
// (add_transfer, kvstore.cpp:180-185) and completes it at apply.
//
// Ordering between lanes, without per-page state on the hot path:
//   * a page installed as a tier copy is complete (lockstep moves sync; a
//     free-running move is installed at apply, after its event) — except a
//     created block, whose fill runs on the FILL lane: readers of a row wait
//     for the row's newest fill ticket;
//   * a page still being moved in (posted, not applied) is only read by
//     moves chained on its event (inflight_source) or by a decode step
//     (decode_rows returns the event);
//   * a freed page goes to quarantine until every batch queued before the
//     free has completed, so no new writer ever races an old reader/writer.

#include "symsim/payload.hpp"

#include <nvtx3/nvToolsExt.h>  // header-only NVTX v3: ranges show per lane in nsys / ncu

#include <algorithm>
#include <chrono>
#include <cstring>
#include <stdexcept>
#include <string>

namespace symsim {

namespace {

void kvx_check(int rc, const char* what) {
  if (rc != KVX_OK) throw std::runtime_error(std::string("payload: ") + what + ": " + kvx_last_error());
}

std::uint64_t now_ns() {
  return static_cast<std::uint64_t>(
      std::chrono::duration_cast<std::chrono::nanoseconds>(std::chrono::steady_clock::now().time_since_epoch())
          .count());
}

const char* const kPoolNames[] = {"device", "host", "landing", "disk"};

}  // namespace

// Host time of the payload's bookkeeping, by phase (kvs_payload_host_ns).
struct NodePayload::HostTimer {
  std::uint64_t& acc;
  std::uint64_t t0;
  explicit HostTimer(std::uint64_t& a) : acc(a), t0(now_ns()) {}
  ~HostTimer() { acc += now_ns() - t0; }
};

// node id -> node for one pass (a cluster lookup per node, not per page).
NodePayload* NodePayload::NodeCache::get(PayloadCluster* cluster, int id) {
  for (int k = 0; k < n; ++k)
    if (ids[k] == id) return nodes[k];
  NodePayload* p = cluster ? cluster->node(id) : nullptr;
  if (n < 8) {
    ids[n] = id;
    nodes[n++] = p;
  }
  return p;
}

// ---------------------------------------------------------------------------
// cluster registry

void PayloadCluster::add(NodePayload* node) { nodes_[node->node_id()] = node; }

void PayloadCluster::remove(NodePayload* node) {
  const auto it = nodes_.find(node->node_id());
  if (it != nodes_.end() && it->second == node) nodes_.erase(it);
}

std::vector<NodePayload*> PayloadCluster::nodes() const {
  std::vector<NodePayload*> out;
  for (const auto& e : nodes_) out.push_back(e.second);
  return out;
}

NodePayload* PayloadCluster::node(int id) const {
  const auto it = nodes_.find(id);
  return it == nodes_.end() ? nullptr : it->second;
}

void PayloadCluster::note_source(std::uint32_t session, int node) { sources_[session] = node; }

int PayloadCluster::take_source(std::uint32_t session) {
  const auto it = sources_.find(session);
  if (it == sources_.end()) return -1;
  const int n = it->second;
  sources_.erase(it);
  return n;
}

// ---------------------------------------------------------------------------
// lanes

// Retires completed batches from the front (they complete in ticket order).
void NodePayload::Lane::retire() {
  std::size_t k = 0;
  while (k < pending.size() && kvx_event_query(pending[k].second) == KVX_OK) {
    done = pending[k].first;
    kvx_event_destroy(pending[k].second);
    ++k;
  }
  pending.erase(pending.begin(), pending.begin() + static_cast<std::ptrdiff_t>(k));
}

void* NodePayload::Lane::event_for(std::uint64_t ticket) {
  if (ticket <= done) return nullptr;
  retire();
  return find_pending(ticket);
}

// Like event_for, but without retiring (destroying) completed events: a
// caller collecting several lanes' events before using them all keeps every
// handle alive this way.
void* NodePayload::Lane::find_pending(std::uint64_t ticket) const {
  if (ticket <= done) return nullptr;
  const auto it = std::lower_bound(pending.begin(), pending.end(), std::make_pair(ticket, static_cast<void*>(nullptr)),
                                   [](const auto& a, const auto& b) { return a.first < b.first; });
  return it != pending.end() && it->first == ticket ? it->second : nullptr;
}

void NodePayload::Lane::drain() {
  for (auto& e : pending) kvx_event_destroy(e.second);
  pending.clear();
  done = next - 1;
}

void* NodePayload::pending_event(NodePayload* node, int lane, std::uint64_t ticket) const {
  return node ? node->lanes_[lane].event_for(ticket) : nullptr;
}

std::uint64_t NodePayload::close_batch(int lane) {
  const HostTimer timer(host_ns_[kHostClose]);
  Lane& L = lanes_[lane];
  L.retire();  // keeps the pending list short on lanes nobody waits on
  void* ev = nullptr;
  kvx_check(kvx_event_create(&ev), "event");
  kvx_check(kvx_event_record(ev, L.stream), "event record");
  const std::uint64_t ticket = L.next++;
  L.pending.emplace_back(ticket, ev);
  return ticket;
}

// ---------------------------------------------------------------------------
// node: pools, pages, scratch

NodePayload::NodePayload(PayloadCluster* cluster, int node_id, const PayloadOptions& opts)
    : cluster_(cluster), node_(node_id), opts_(opts) {
  page_bytes_ = kvx_page_bytes(&opts_.layout);
  if (page_bytes_ == 0) throw std::runtime_error("payload: empty page layout");
  for (Lane& L : lanes_) {
    kvx_check(kvx_stream_create(opts_.device, &L.stream), "stream");
    // Upload staging up front: pinned allocations cost milliseconds, not
    // something to pay inside the first moves.
    void* p = nullptr;
    L.ring_cap = std::size_t{4} << 20;
    kvx_check(kvx_host_alloc(L.ring_cap, &p), "upload ring");
    L.ring = static_cast<std::uint8_t*>(p);
    L.d_ids_cap = std::size_t{1} << 16;
    kvx_check(kvx_malloc(opts_.device, L.d_ids_cap * sizeof(std::uint32_t), &p), "id scratch");
    L.d_ids = static_cast<std::uint32_t*>(p);
  }
  const std::uint64_t counts[4] = {opts_.device_pages, opts_.host_pages, opts_.landing_pages, opts_.disk_pages};
  for (int p = 0; p < 4; ++p) {
    if (counts[p] == 0) continue;
    if (counts[p] > 0x3FFFFFFFull) throw std::runtime_error("payload: a pool holds at most 2^30 pages");
    if (p == kDevicePool || p == kLandingPool)
      kvx_check(kvx_pool_create(opts_.device, counts[p], page_bytes_, &pools_[p]), "device pool");
    else if (p == kDiskPool && !opts_.disk_path.empty())
      kvx_check(kvx_pool_create_file(opts_.disk_path.c_str(), counts[p], page_bytes_, &pools_[p]), "disk file");
    else
      kvx_check(kvx_pool_create_host(counts[p], page_bytes_, &pools_[p]), "host pool");
    free_[p].resize(counts[p]);
    // LIFO free list handing out low page ids first.
    for (std::uint64_t i = 0; i < counts[p]; ++i) free_[p][i] = static_cast<std::uint32_t>(counts[p] - 1 - i);
  }
  if (cluster_) cluster_->add(this);
}

NodePayload::~NodePayload() {
  // Peers may have queued pushes into our landing pool: let them land first.
  if (cluster_) {
    cluster_->remove(this);
    for (NodePayload* n : cluster_->nodes()) n->synchronize();
  }
  for (Lane& L : lanes_)
    if (L.stream) kvx_stream_synchronize(L.stream);
  for (InFlight& f : flights_) kvx_event_destroy(f.event);
  for (auto*& p : pools_)
    if (p) kvx_pool_destroy(p);
  for (Lane& L : lanes_) {
    L.drain();
    kvx_free(L.d_ids);
    kvx_host_free(L.ring);
    if (L.bounce) kvx_pool_destroy(L.bounce);
    kvx_stream_destroy(L.stream);
  }
  kvx_free(d_tags_);
}

void NodePayload::synchronize() {
  for (Lane& L : lanes_) {
    kvx_check(kvx_stream_synchronize(L.stream), "sync");
    L.drain();
  }
}

std::uint64_t NodePayload::pages_in_use(Pool p) const {
  const std::uint64_t total = pools_[p] ? kvx_pool_num_pages(pools_[p]) : 0;
  return total - free_[p].size() - held_[p];
}

std::uint64_t NodePayload::pages_in_flight(Pool p) const {
  std::uint64_t n = 0;
  for (const auto& e : flight_of_)
    for (const Ref& r : flights_[e.second].pages) n += r.pool == p;
  return n;
}

// ---------------------------------------------------------------------------
// free pages and quarantine

void NodePayload::release(const Ref& r) {
  if (r.pool < 0) return;
  released_.push_back(r);
  ++held_[r.pool];
}

// Returns held pages to their free lists (each list grows once; per-page
// push_back dominated reclaim on 2,048-page layers). Order within a pool is
// the order of `pages`, as one push_back at a time would leave it.
void NodePayload::give_back(const Ref* pages, std::size_t n) {
  std::size_t count[kPools] = {};
  for (std::size_t i = 0; i < n; ++i) ++count[pages[i].pool];
  std::uint32_t* out[kPools] = {};
  for (int p = 0; p < kPools; ++p) {
    if (!count[p]) continue;
    const std::size_t at = free_[p].size();
    free_[p].resize(at + count[p]);
    out[p] = free_[p].data() + at;
    held_[p] -= count[p];
  }
  for (std::size_t i = 0; i < n; ++i) *out[pages[i].pool]++ = pages[i].page;
}

// Closes the group of pages freed so far: they may be reused once every
// batch queued until now, on any lane of any node, has completed.
void NodePayload::seal_released() {
  if (released_.empty()) return;
  Held h;
  auto mark = [&h](const NodePayload& n) {
    for (int l = 0; l < kLanes; ++l)
      if (n.lanes_[l].last() > n.lanes_[l].done) h.marks.push_back({{n.node_, l}, n.lanes_[l].last()});
  };
  if (cluster_)
    for (const NodePayload* n : cluster_->nodes()) mark(*n);
  else
    mark(*this);
  if (h.marks.empty()) {  // nothing queued anywhere: free now
    give_back(released_.data(), released_.size());
  } else {
    h.pages.assign(released_.begin(), released_.end());  // released_ keeps its capacity
    quarantine_.push_back(std::move(h));
  }
  released_.clear();
}

// Returns quarantined groups whose batches have all completed (FIFO: later
// groups were sealed later, so they are never ready before earlier ones).
// With `wait_for_oldest`, blocks on the oldest group first. True if any
// group was returned.
bool NodePayload::reclaim(bool wait_for_oldest) {
  const HostTimer timer(host_ns_[kHostReclaim]);
  bool any = false;
  NodeCache owners;
  while (!quarantine_.empty()) {
    Held& h = quarantine_.front();
    bool ready = true;
    for (const auto& m : h.marks) {
      NodePayload* owner = m.first.first == node_ ? this : owners.get(cluster_, m.first.first);
      if (!owner) continue;  // gone, and synchronized on its way out
      Lane& L = owner->lanes_[m.first.second];
      if (m.second <= L.done) continue;
      void* ev = L.event_for(m.second);
      if (!ev) continue;
      if (!wait_for_oldest) {
        ready = false;
        break;
      }
      kvx_check(kvx_event_synchronize(ev), "quarantine wait");
      L.retire();
    }
    if (!ready) break;
    give_back(h.pages.data(), h.pages.size());
    quarantine_.pop_front();
    any = true;
    wait_for_oldest = false;
  }
  return any;
}

// n pages at once from the free list's top (same order as n alloc() calls),
// taking back quarantined pages as needed.
void NodePayload::alloc_n(Pool p, std::size_t n, std::vector<std::uint32_t>& out) {
  const HostTimer timer(host_ns_[kHostAlloc]);
  std::vector<std::uint32_t>& fl = free_[p];
  if (fl.size() < n) {
    seal_released();
    reclaim(false);
    bool waited = false;
    while (fl.size() < n && !quarantine_.empty()) {
      reclaim(true);
      waited = true;
    }
    if (waited) ++quarantine_waits_;
  }
  if (fl.size() < n)
    throw std::runtime_error(std::string("payload: node ") + std::to_string(node_) + " " + kPoolNames[p] +
                             " pool exhausted");
  out.insert(out.end(), fl.rbegin(), fl.rbegin() + static_cast<std::ptrdiff_t>(n));
  fl.resize(fl.size() - n);
}

std::uint32_t NodePayload::alloc(Pool p) {
  std::vector<std::uint32_t> one;
  alloc_n(p, 1, one);
  return one[0];
}

// Re-deals a batch's freshly allocated pages (one pool) in ascending order:
// the free list is LIFO, so pages released in ascending order come back
// descending; ascending destinations pair with ascending sources into long
// runs of consecutive ids, which the copy engines move as one copy each.
void sort_pages(std::vector<std::uint32_t>& pages) { std::sort(pages.begin(), pages.end()); }

// ---------------------------------------------------------------------------
// uploads

void* NodePayload::stage(Lane& L, std::size_t bytes) {
  const std::size_t need = (std::max<std::size_t>(bytes, 1) + 255) & ~static_cast<std::size_t>(255);
  if (need > L.ring_cap) {
    // Grow: every upload staged so far must have been consumed first.
    if (L.ring) {
      kvx_check(kvx_stream_synchronize(L.stream), "sync");
      L.retire();
      kvx_host_free(L.ring);
      L.ring = nullptr;
    }
    L.ring_used.clear();
    L.ring_head = 0;
    L.ring_cap = std::max<std::size_t>(need * 4, std::size_t{4} << 20);
    void* p = nullptr;
    kvx_check(kvx_host_alloc(L.ring_cap, &p), "upload ring");
    L.ring = static_cast<std::uint8_t*>(p);
  }
  std::size_t begin = L.ring_head;
  if (begin + need > L.ring_cap) begin = 0;
  const std::size_t end = begin + need;
  // Regions of completed batches are free; an overlapping live one is waited
  // for (rare: the ring holds many batches).
  while (!L.ring_used.empty() && L.ring_used.front().ticket <= L.done) L.ring_used.pop_front();
  std::uint64_t wait = 0;
  for (const Lane::Region& r : L.ring_used)
    if (r.begin < end && begin < r.end) wait = std::max(wait, r.ticket);
  if (wait) {
    if (void* ev = L.event_for(wait)) kvx_check(kvx_event_synchronize(ev), "upload ring wait");
    L.retire();
    while (!L.ring_used.empty() && L.ring_used.front().ticket <= L.done) L.ring_used.pop_front();
  }
  L.ring_used.push_back(Lane::Region{begin, end, L.next});
  L.ring_head = end;
  return L.ring + begin;
}

// The lane's device id scratch filled from `n` ids already staged in its
// pinned ring (one async copy; same-stream order protects the scratch).
std::uint32_t* NodePayload::upload_ids(Lane& L, const std::uint32_t* staged, std::size_t n) {
  if (n > L.d_ids_cap) {
    kvx_check(kvx_stream_synchronize(L.stream), "sync");  // queued kernels may still read it
    kvx_free(L.d_ids);
    L.d_ids = nullptr;
    L.d_ids_cap = std::max<std::size_t>(n * 2, 8192);
    void* p = nullptr;
    kvx_check(kvx_malloc(opts_.device, L.d_ids_cap * sizeof(std::uint32_t), &p), "id scratch");
    L.d_ids = static_cast<std::uint32_t*>(p);
  }
  kvx_check(kvx_memcpy_async(L.d_ids, staged, n * sizeof(std::uint32_t), L.stream), "ids upload");
  return L.d_ids;
}

std::uint32_t* NodePayload::device_ids(Lane& L, const std::vector<std::uint32_t>& ids) {
  auto* host = static_cast<std::uint32_t*>(stage(L, ids.size() * sizeof(std::uint32_t)));
  std::memcpy(host, ids.data(), ids.size() * sizeof(std::uint32_t));
  return upload_ids(L, host, ids.size());
}

// ---------------------------------------------------------------------------
// lookups

const NodePayload::Row* NodePayload::find_row(std::uint32_t s, std::uint16_t l) const {
  const auto it = rows_.find(row_key(s, l));
  return it == rows_.end() ? nullptr : &it->second;
}

const NodePayload::Copies* NodePayload::find(std::uint32_t s, std::uint16_t l, std::uint32_t b) const {
  const Row* r = find_row(s, l);
  return r && b < r->b.size() ? &r->b[b] : nullptr;
}

void NodePayload::drop_row_if_empty(std::uint32_t s, std::uint16_t l) {
  const auto it = rows_.find(row_key(s, l));
  if (it == rows_.end()) return;
  for (const Copies& c : it->second.b)
    if (!c.empty()) return;
  rows_.erase(it);
}

// Best existing copy of a block on this node, fastest tier first, skipping
// `exclude_tier` (the tier being created).
NodePayload::Ref NodePayload::best_source(std::uint32_t s, std::uint16_t l, std::uint32_t b,
                                          int exclude_tier) const {
  const Copies* c = find(s, l, b);
  if (!c) return Ref{};
  for (int t = 0; t < 3; ++t)
    if (t != exclude_tier && c->slot[t] != kNoPage) return c->tier(t);
  return Ref{};
}

NodePayload::Ref NodePayload::flight_page(const InFlight& f, std::uint32_t b) {
  const auto pos = std::lower_bound(f.blocks.begin(), f.blocks.end(), b);  // f.blocks ascends
  return f.pages[static_cast<std::size_t>(pos - f.blocks.begin())];
}

// Empties a finished flight slot but keeps its vectors' capacity: the next
// posting into the slot refills them without a fresh allocation (2,048-block
// layers at 70B @32K).
void NodePayload::reset_flight(InFlight& f) {
  f.id = 0;
  f.tier = 0;
  f.session = 0;
  f.layer = 0;
  f.blocks.clear();
  f.pages.clear();
  f.event = nullptr;
}

bool NodePayload::inflight_source(std::uint32_t s, std::uint16_t l, std::uint32_t b, int exclude_tier, Ref* page,
                                  void** event) const {
  const Copies* c = find(s, l, b);
  if (!c) return false;
  for (int t = 0; t < 3; ++t) {
    if (t == exclude_tier || !c->coming[t]) continue;
    const InFlight& f = flight(c->coming[t]);
    *page = flight_page(f, b);
    *event = f.event;
    return true;
  }
  return false;
}

bool NodePayload::device_block_table(std::uint32_t session, std::uint16_t layer, std::uint32_t n,
                                     std::uint32_t* out) const {
  if (n == 0) return true;
  const Row* r = find_row(session, layer);
  if (!r || r->b.size() < n) return false;
  for (std::uint32_t b = 0; b < n; ++b) {
    const Ref p = r->b[b].tier(0);
    if (p.pool != kDevicePool) return false;
    out[b] = p.page;
  }
  return true;
}

bool NodePayload::decode_rows(const std::vector<std::pair<std::uint32_t, std::uint32_t>>& reqs, std::uint16_t layer,
                              std::uint32_t stride, std::uint32_t* out, std::vector<void*>& waits) {
  std::uint64_t fill = 0;  // newest fill among the rows (the FILL lane completes in order)
  const std::size_t first_wait = waits.size();
  // A batch already complete on the GPU needs no wait (and an empty wait
  // list lets the step replay as a CUDA graph): queried once per event.
  void* last_checked = nullptr;
  auto add_wait = [&](void* ev) {
    if (std::find(waits.begin() + static_cast<std::ptrdiff_t>(first_wait), waits.end(), ev) != waits.end()) return;
    if (kvx_event_query(ev) == KVX_OK) return;
    waits.push_back(ev);
  };
  for (std::size_t i = 0; i < reqs.size(); ++i) {
    const std::uint32_t n = reqs[i].second;
    if (n == 0) continue;
    const Row* r = find_row(reqs[i].first, layer);
    if (!r || r->b.size() < n) return false;
    fill = std::max(fill, r->fill_ticket);
    std::uint32_t* dst = out + i * stride;
    for (std::uint32_t b = 0; b < n; ++b) {
      const Copies& c = r->b[b];
      if (c.slot[0] != kNoPage && (c.slot[0] >> 30) == static_cast<std::uint32_t>(kDevicePool)) {
        dst[b] = c.slot[0] & 0x3FFFFFFFu;
        continue;
      }
      if (!c.coming[0]) return false;
      const InFlight& f = flight(c.coming[0]);  // a load still landing: wait for exactly that move
      dst[b] = flight_page(f, b).page;
      if (f.event != last_checked) {
        last_checked = f.event;
        add_wait(f.event);
      }
    }
  }
  // No retiring here: the executor collects all layers' waits before issuing
  // them, so handles found for earlier layers must stay alive.
  if (void* ev = fill ? lanes_[kLaneFill].find_pending(fill) : nullptr) add_wait(ev);
  return true;
}

int NodePayload::pool_of(std::uint32_t s, std::uint16_t l, std::uint32_t b, Tier tier) const {
  const Copies* c = find(s, l, b);
  return c ? c->tier(static_cast<int>(tier)).pool : -1;
}

// ---------------------------------------------------------------------------
// moves

// Queues src[i] -> dst[i] (dst in this node's pools) grouped by (source pool,
// destination pool). HBM<->HBM pairs use the SM/TMA page mover with device id
// lists; anything touching pinned host memory uses the copy engines. With
// `push` the work runs on the source node's PEER lane and stores into this
// node's memory (the NVLink / peer path of a migration); otherwise on this
// node's IN lane (destination in HBM), DISK lane (disk-tier source or
// destination) or OUT lane (HBM -> host). The batch first waits on `waits`
// and on the source row's fill (ticket `src_fill` of the source node's FILL
// lane); destination pages come from the free lists, so nothing queued can
// still be touching them.
void* NodePayload::issue(const std::vector<Ref>& src, const std::vector<Ref>& dst, NodePayload& src_node, bool push,
                         const std::vector<void*>& waits, std::uint64_t src_fill) {
  const HostTimer timer(host_ns_[kHostIssue]);
  NodePayload& runner = push ? src_node : *this;
  const int dp0 = dst.empty() ? static_cast<int>(kDevicePool) : dst[0].pool;
  const bool from_disk = std::any_of(src.begin(), src.end(), [](const Ref& r) { return r.pool == kDiskPool; });
  const int lane = push                                           ? kLanePeer
                   : (dp0 == kDevicePool || dp0 == kLandingPool) ? kLaneIn
                   : (dp0 == kDiskPool || from_disk)             ? kLaneDisk
                                                                 : kLaneOut;
  Lane& L = runner.lanes_[lane];
  static const char* const kLaneNames[] = {"kvs:IN", "kvs:OUT", "kvs:DISK", "kvs:PEER", "kvs:FILL"};
  nvtxRangePushA(kLaneNames[lane]);  // host-side enqueue of this batch (NVTX, SURVEY.md §5 tracing)
  struct PopRange {
    ~PopRange() { nvtxRangePop(); }
  } pop_range;
  for (void* ev : waits) kvx_check(kvx_stream_wait_event(L.stream, ev), "stream wait");
  if (void* ev = src_fill ? src_node.lanes_[kLaneFill].event_for(src_fill) : nullptr)
    kvx_check(kvx_stream_wait_event(L.stream, ev), "fill wait");
  auto hbm = [](int p) { return p == kDevicePool || p == kLandingPool; };
  // Common case: one (source pool, destination pool) pair, HBM on both
  // sides — the ids go straight into the pinned ring, one upload, one mover.
  bool uniform = !src.empty();
  for (std::size_t i = 1; i < src.size() && uniform; ++i)
    uniform = src[i].pool == src[0].pool && dst[i].pool == dst[0].pool;
  if (uniform && hbm(src[0].pool) && hbm(dst[0].pool)) {
    const std::size_t n = src.size();
    std::uint32_t* d_ids = nullptr;
    {
      const HostTimer up(host_ns_[kHostUpload]);
      auto* h = static_cast<std::uint32_t*>(runner.stage(L, 2 * n * sizeof(std::uint32_t)));
      for (std::size_t i = 0; i < n; ++i) h[i] = src[i].page;
      for (std::size_t i = 0; i < n; ++i) h[n + i] = dst[i].page;
      d_ids = runner.upload_ids(L, h, 2 * n);
    }
    {
      const HostTimer launch_timer(host_ns_[kHostLaunch]);
      kvx_check(kvx_copy_pages_capped(src_node.pools_[src[0].pool], d_ids, pools_[dst[0].pool], d_ids + n, n,
                                      KVX_COPY_AUTO, push ? src_node.opts_.migrate_max_ctas : 0u, L.stream),
                "page copy");
    }
    runner.close_batch(lane);
    return L.stream;
  }
  // General case: bucket by pool pair; the id lists of every HBM<->HBM
  // bucket go up in ONE staged upload.
  std::vector<std::uint32_t> bucket_ids[16][2];
  for (std::size_t i = 0; i < src.size(); ++i) {
    const int k = src[i].pool * 4 + dst[i].pool;
    bucket_ids[k][0].push_back(src[i].page);
    bucket_ids[k][1].push_back(dst[i].page);
  }
  std::size_t offsets[16][2] = {};
  std::vector<std::uint32_t> staged;
  for (int k = 0; k < 16; ++k)
    if (!bucket_ids[k][0].empty() && hbm(k / 4) && hbm(k % 4))
      for (int side = 0; side < 2; ++side) {
        offsets[k][side] = staged.size();
        staged.insert(staged.end(), bucket_ids[k][side].begin(), bucket_ids[k][side].end());
      }
  const std::uint32_t* d_staged = nullptr;
  if (!staged.empty()) {
    const HostTimer up(host_ns_[kHostUpload]);
    d_staged = runner.device_ids(L, staged);
  }
  const HostTimer launch_timer(host_ns_[kHostLaunch]);
  for (int sp = 0; sp < 4; ++sp)
    for (int dp = 0; dp < 4; ++dp) {
      const std::vector<std::uint32_t>& s_ids = bucket_ids[sp * 4 + dp][0];
      const std::vector<std::uint32_t>& d_ids = bucket_ids[sp * 4 + dp][1];
      if (s_ids.empty()) continue;
      kvx_pool* from = src_node.pools_[sp];
      kvx_pool* to = pools_[dp];
      // A file pool on either side (the source node's DISK copy may be a file
      // even when ours is not) with HBM on the other goes through a bounce.
      const bool file_side = kvx_pool_file_direct(from) >= 0 || kvx_pool_file_direct(to) >= 0;
      const bool file_hop = file_side && (hbm(sp) || hbm(dp));
      if (hbm(sp) && hbm(dp)) {
        const std::uint32_t* ds = d_staged + offsets[sp * 4 + dp][0];
        const std::uint32_t* dd = d_staged + offsets[sp * 4 + dp][1];
        kvx_check(kvx_copy_pages_capped(from, ds, to, dd, s_ids.size(), KVX_COPY_AUTO,
                                        push ? src_node.opts_.migrate_max_ctas : 0u, L.stream),
                  "page copy");
      } else if (file_hop) {
        // HBM <-> file: through this lane's pinned bounce pages, a chunk at a
        // time; stream order keeps each chunk's file I/O ahead of the copy
        // that refills the bounce pages.
        if (!L.bounce) kvx_check(kvx_pool_create_host(kBouncePages, page_bytes_, &L.bounce), "bounce pool");
        for (std::size_t at = 0; at < s_ids.size(); at += kBouncePages) {
          const std::size_t k = std::min<std::size_t>(kBouncePages, s_ids.size() - at);
          std::vector<std::uint32_t> b_ids(k);
          for (std::size_t i = 0; i < k; ++i) b_ids[i] = static_cast<std::uint32_t>(i);
          kvx_check(kvx_copy_pages(from, s_ids.data() + at, L.bounce, b_ids.data(), k, KVX_COPY_CE, L.stream),
                    "disk hop (in)");
          kvx_check(kvx_copy_pages(L.bounce, b_ids.data(), to, d_ids.data() + at, k, KVX_COPY_CE, L.stream),
                    "disk hop (out)");
        }
      } else {
        kvx_check(kvx_copy_pages(from, s_ids.data(), to, d_ids.data(), s_ids.size(), KVX_COPY_CE, L.stream),
                  "copy-engine copy");
      }
    }
  runner.close_batch(lane);
  return L.stream;
}

// ---------------------------------------------------------------------------
// residency transitions

void NodePayload::tier_gained(std::uint32_t session, std::uint16_t layer, Tier tier, BlockEvent why,
                              const std::vector<std::uint32_t>& blocks) {
  const int t = static_cast<int>(tier);
  moved_[static_cast<int>(why)] += blocks.size() * page_bytes_;

  if (why == BlockEvent::Created) {
    Row& r = row(session, layer);
    presize(r, blocks);
    for (std::uint32_t b : blocks) {
      Copies& c = at(r, b);
      release(c.tier(t));
      c.slot[t] = kNoPage;
    }
    std::vector<std::uint32_t> pages;
    alloc_n(kDevicePool, blocks.size(), pages);
    sort_pages(pages);
    // One staged upload carries the page ids and their (session, layer,
    // block) tags; the fill runs on the FILL lane.
    const std::size_t id_bytes = pages.size() * sizeof(std::uint32_t);
    const std::size_t tag_off = (id_bytes + 15) & ~static_cast<std::size_t>(15);
    const std::size_t bytes = tag_off + blocks.size() * sizeof(kvx_block_tag);
    Lane& L = lanes_[kLaneFill];
    auto* host = static_cast<std::uint8_t*>(stage(L, bytes));
    std::memcpy(host, pages.data(), id_bytes);
    auto* tags = reinterpret_cast<kvx_block_tag*>(host + tag_off);
    for (std::size_t i = 0; i < blocks.size(); ++i) {
      r.b[blocks[i]].slot[t] = pack(Ref{kDevicePool, pages[i]});
      tags[i] = kvx_block_tag{session, layer, blocks[i]};
    }
    if (bytes > d_tags_cap_) {
      if (d_tags_) kvx_check(kvx_stream_synchronize(L.stream), "sync");
      kvx_free(d_tags_);
      d_tags_cap_ = std::max<std::size_t>(bytes * 2, 65536);
      kvx_check(kvx_malloc(opts_.device, d_tags_cap_, &d_tags_), "tag scratch");
    }
    kvx_check(kvx_memcpy_async(d_tags_, host, bytes, L.stream), "ids + tags upload");
    const auto* d_pages = static_cast<const std::uint32_t*>(d_tags_);
    const auto* d_tags = reinterpret_cast<const kvx_block_tag*>(static_cast<const std::uint8_t*>(d_tags_) + tag_off);
    kvx_check(kvx_fill_pages(pools_[kDevicePool], d_pages, d_tags, pages.size(), opts_.seed, &opts_.layout,
                             opts_.fill_mode, L.stream),
              "fill");
    r.fill_ticket = close_batch(kLaneFill);
    if (!opts_.free_running) synchronize();
    return;
  }

  if (!opts_.free_running || !applying_valid_) {
    move_now(session, layer, tier, why, blocks);
    return;
  }

  // Free-running: the move was issued when the transfer was scheduled and
  // has completed (transfer_retired waited on it). Install the pages of the
  // blocks the state machine says gained the tier; return the rest.
  const std::uint32_t slot = flight_of_.at(applying_);
  InFlight& f = flights_[slot];
  applying_valid_ = false;
  std::vector<std::uint32_t> missing;
  Row& r = row(session, layer);
  presize(r, blocks);
  if (blocks.size() == f.blocks.size() &&
      std::equal(blocks.begin(), blocks.end(), f.blocks.begin())) {  // the usual case: every posted block gained
    Copies* const rb = r.b.data();
    const Ref* const fp = f.pages.data();
    for (std::size_t i = 0; i < blocks.size(); ++i) {
      Copies& c = rb[blocks[i]];
      if (c.slot[t] != kNoPage) release(c.tier(t));
      c.slot[t] = pack(fp[i]);
    }
    kvx_event_destroy(f.event);
    reset_flight(f);
    flight_of_.erase(applying_);
    free_flights_.push_back(slot);
    return;
  }
  std::size_t cursor = 0;  // both lists usually ascend: a merge walk, bisection otherwise
  for (std::uint32_t b : blocks) {
    std::size_t i = cursor;
    if (i >= f.blocks.size() || f.blocks[i] != b) {
      const auto pos = std::lower_bound(f.blocks.begin(), f.blocks.end(), b);
      i = static_cast<std::size_t>(pos - f.blocks.begin());
    }
    if (i >= f.blocks.size() || f.blocks[i] != b) {
      missing.push_back(b);  // its source appeared only after scheduling
      continue;
    }
    cursor = i + 1;
    Copies& c = at(r, b);
    release(c.tier(t));
    c.slot[t] = pack(f.pages[i]);
    f.pages[i] = Ref{};  // installed; release() skips it below
  }
  for (const Ref& p : f.pages) release(p);
  kvx_event_destroy(f.event);
  reset_flight(f);
  flight_of_.erase(applying_);
  free_flights_.push_back(slot);
  if (!missing.empty()) move_now(session, layer, tier, why, missing);
}

// Lockstep move: choose each block's source now, copy, wait.
void NodePayload::move_now(std::uint32_t session, std::uint16_t layer, Tier tier, BlockEvent why,
                           const std::vector<std::uint32_t>& blocks) {
  if (blocks.empty()) return;
  const int t = static_cast<int>(tier);
  Pool dest = kDevicePool;
  NodePayload* src_node = this;
  bool push = false;
  if (tier == Tier::Host) dest = why == BlockEvent::NetArrive ? kLandingPool : kHostPool;
  if (tier == Tier::Disk) dest = kDiskPool;
  if (why == BlockEvent::NetArrive) {
    const auto it = import_src_.find(session);
    if (it == import_src_.end() || !cluster_ || !cluster_->node(it->second))
      throw std::runtime_error("payload: migration layer arrived with no known source node");
    src_node = cluster_->node(it->second);
    push = true;
  }
  std::vector<Ref> src, dst;
  Row& r = row(session, layer);
  presize(r, blocks);
  for (std::uint32_t b : blocks) {
    const Ref from = src_node->best_source(session, layer, b, src_node == this ? t : -1);
    if (from.pool < 0)
      throw std::runtime_error("payload: no source copy for session " + std::to_string(session) + " layer " +
                               std::to_string(layer) + " block " + std::to_string(b) + " (" +
                               block_event_name(why) + ")");
    Copies& c = at(r, b);
    release(c.tier(t));
    c.slot[t] = kNoPage;
    src.push_back(from);
  }
  std::vector<std::uint32_t> pages;
  alloc_n(dest, blocks.size(), pages);
  sort_pages(pages);
  for (std::size_t i = 0; i < blocks.size(); ++i) {
    const Ref d{static_cast<std::int8_t>(dest), pages[i]};
    at(r, blocks[i]).slot[t] = pack(d);
    dst.push_back(d);
  }
  const Row* sr = src_node->find_row(session, layer);
  issue(src, dst, *src_node, push, {}, sr ? sr->fill_ticket : 0);
  (push ? *src_node : *this).synchronize();
  check_file_io();
}

// Sticky file-pool I/O errors (kvx_pool_io_error) of this node and of every
// node it may read from, raised before a move's pages are installed.
void NodePayload::check_file_io() const {
  auto check = [](const NodePayload& n) {
    const kvx_pool* disk = n.pools_[kDiskPool];
    if (const int e = disk ? kvx_pool_io_error(disk) : 0)
      throw std::runtime_error("payload: node " + std::to_string(n.node_) + " disk-tier file I/O failed (errno " +
                               std::to_string(e) + "); the move's pages are not valid");
  };
  check(*this);
  if (cluster_)
    for (const NodePayload* n : cluster_->nodes())
      if (n != this) check(*n);
}

void NodePayload::tier_lost(std::uint32_t session, std::uint16_t layer, Tier tier,
                            const std::vector<std::uint32_t>& blocks) {
  const int t = static_cast<int>(tier);
  const auto it = rows_.find(row_key(session, layer));
  if (it == rows_.end()) return;
  const std::size_t base = released_.size();
  released_.resize(base + blocks.size());
  Ref* const out = released_.data() + base;
  std::size_t n = 0;
  Copies* const rb = it->second.b.data();
  const std::size_t rn = it->second.b.size();
  for (const std::uint32_t b : blocks) {
    if (b >= rn || rb[b].slot[t] == kNoPage) continue;
    const Ref r = rb[b].tier(t);  // release(), inlined
    out[n++] = r;
    ++held_[r.pool];
    rb[b].slot[t] = kNoPage;
  }
  released_.resize(base + n);
  drop_row_if_empty(session, layer);
}

// ---------------------------------------------------------------------------
// free-running: issue at schedule time, complete at apply

void NodePayload::transfer_posted(const TransferInfo& tr) {
  if (!opts_.free_running) return;
  const int t = static_cast<int>(tr.to);
  Pool dest = kDevicePool;
  if (tr.to == Tier::Host) dest = tr.kind == BlockEvent::NetArrive ? kLandingPool : kHostPool;
  if (tr.to == Tier::Disk) dest = kDiskPool;
  NodePayload* src_node = this;
  bool push = false;
  if (tr.kind == BlockEvent::NetArrive) {
    const auto it = import_src_.find(tr.session);
    if (it == import_src_.end() || !cluster_ || !cluster_->node(it->second)) return;  // apply falls back
    src_node = cluster_->node(it->second);
    push = true;
  }
  const HostTimer timer(host_ns_[kHostPosted]);
  std::uint32_t slot;
  if (!free_flights_.empty()) {
    slot = free_flights_.back();
    free_flights_.pop_back();
  } else {
    slot = static_cast<std::uint32_t>(flights_.size());
    flights_.emplace_back();
  }
  InFlight& f = flights_[slot];
  f.id = tr.id;
  f.tier = t;
  f.session = tr.session;
  f.layer = tr.layer;
  f.blocks.clear();
  f.pages.clear();
  // Per-posting scratch is kept across calls: fresh 16-100 KB buffers per
  // layer cost more in allocation and first-touch faults than the work.
  std::vector<Ref>& src = scratch_src_;
  std::vector<void*>& waits = scratch_waits_;
  std::vector<std::uint32_t>& pages = scratch_pages_;
  src.clear();
  waits.clear();
  pages.clear();
  const Row* have = find_row(tr.session, tr.layer);
  const Row* srow = src_node->find_row(tr.session, tr.layer);
  const int exclude = src_node == this ? t : -1;
  const std::size_t span = static_cast<std::size_t>(tr.block_hi - tr.block_lo + 1);
  // Written through raw pointers into buffers sized for the whole span, then
  // trimmed: per-element push_back costs several times the loop body on
  // 2,048-block layers.
  src.resize(span);
  f.blocks.resize(span);
  Ref* const sp = src.data();
  std::uint32_t* const bp = f.blocks.data();
  std::size_t n = 0;
  const Copies* const hv = have ? have->b.data() : nullptr;
  const std::size_t hn = have ? have->b.size() : 0;
  const Copies* const sv = srow ? srow->b.data() : nullptr;
  const std::size_t sn = srow ? srow->b.size() : 0;
  for (std::uint64_t b64 = tr.block_lo; b64 <= tr.block_hi; ++b64) {
    const auto b = static_cast<std::uint32_t>(b64);
    if (b < hn && (hv[b].slot[t] != kNoPage || hv[b].coming[t])) continue;  // already there / already coming
    if (b >= sn) continue;
    const Copies& sc = sv[b];
    const int k = (exclude != 0 && sc.slot[0] != kNoPage)   ? 0
                  : (exclude != 1 && sc.slot[1] != kNoPage) ? 1
                  : (exclude != 2 && sc.slot[2] != kNoPage) ? 2
                                                            : -1;
    Ref from;
    if (k >= 0) {
      from = sc.tier(k);
    } else {  // chained behind a move still in flight on the source side
      void* ev = nullptr;
      if (!src_node->inflight_source(tr.session, tr.layer, b, exclude, &from, &ev)) continue;
      if (waits.empty() || waits.back() != ev) waits.push_back(ev);
    }
    sp[n] = from;
    bp[n] = b;
    ++n;
  }
  src.resize(n);
  f.blocks.resize(n);
  if (f.blocks.empty()) {
    free_flights_.push_back(slot);
    return;
  }
  alloc_n(dest, f.blocks.size(), pages);
  // Ascending pages only matter for copy-engine runs (host / disk pools);
  // the HBM movers take any permutation.
  if (dest == kHostPool || dest == kDiskPool) sort_pages(pages);
  f.pages.resize(pages.size());  // the flight's pages are the move's destinations
  {
    Ref* const fp = f.pages.data();
    const std::uint32_t* const pg = pages.data();
    for (std::size_t i = 0; i < pages.size(); ++i) fp[i] = Ref{static_cast<std::int8_t>(dest), pg[i]};
  }
  std::sort(waits.begin(), waits.end());
  waits.erase(std::unique(waits.begin(), waits.end()), waits.end());
  void* lane_stream = issue(src, f.pages, *src_node, push, waits, srow ? srow->fill_ticket : 0);
  kvx_check(kvx_event_create(&f.event), "event");
  kvx_check(kvx_event_record(f.event, lane_stream), "event record");
  {
    Row& r = row(tr.session, tr.layer);
    if (r.b.size() <= f.blocks.back()) r.b.resize(static_cast<std::size_t>(f.blocks.back()) + 1);  // ascending
    Copies* const rb = r.b.data();
    for (const std::uint32_t b : f.blocks) rb[b].coming[t] = slot + 1;
  }
  moved_[7] += f.blocks.size() * page_bytes_;  // bytes issued ahead of their apply
  flight_of_.emplace(tr.id, slot);
  ++posted_;
}

void NodePayload::transfer_retired(std::uint64_t id, bool voided) {
  const HostTimer timer(host_ns_[kHostRetired]);
  applying_valid_ = false;
  if (!opts_.free_running) return;
  const auto it = flight_of_.find(id);
  if (it == flight_of_.end()) return;
  const std::uint32_t slot = it->second;
  InFlight& f = flights_[slot];
  if (kvx_event_query(f.event) == KVX_NOT_READY) {  // the GPU is behind the model clock
    const std::uint64_t t0 = now_ns();
    nvtxRangePushA("kvs:apply_wait");
    kvx_check(kvx_event_synchronize(f.event), "event sync");
    nvtxRangePop();
    apply_wait_ns_ += now_ns() - t0;
  }
  // A failed pread / pwrite does not fail the stream (host callback): check
  // the file pools before the store installs these pages as valid.
  if (!voided) check_file_io();
  const auto rt = rows_.find(row_key(f.session, f.layer));
  if (rt != rows_.end()) {
    Copies* const rb = rt->second.b.data();
    const std::size_t rn = rt->second.b.size();
    const int ft = f.tier;
    for (const std::uint32_t b : f.blocks)
      if (b < rn && rb[b].coming[ft] == slot + 1) rb[b].coming[ft] = 0;
  }
  if (voided) {
    for (const Ref& r : f.pages) release(r);
    kvx_event_destroy(f.event);
    const std::uint32_t s = f.session;
    const std::uint16_t l = f.layer;
    reset_flight(f);
    flight_of_.erase(it);
    free_flights_.push_back(slot);
    drop_row_if_empty(s, l);
    return;
  }
  applying_ = id;
  applying_valid_ = true;
}

// ---------------------------------------------------------------------------
// migration endpoints, verification

void NodePayload::migrating_out(std::uint32_t session) {
  if (cluster_) cluster_->note_source(session, node_);
}

void NodePayload::importing(std::uint32_t session, std::int64_t /*tokens*/) {
  const int src = cluster_ ? cluster_->take_source(session) : -1;
  if (src >= 0) import_src_[session] = src;
  if (src >= 0 && cluster_->node(src) && cluster_->node(src)->device() != opts_.device)
    kvx_check(kvx_enable_peer_access(cluster_->node(src)->device(), opts_.device), "peer access");
}

bool NodePayload::read_block(std::uint32_t session, std::uint16_t layer, std::uint32_t block, Tier tier, void* out) {
  const Copies* c = find(session, layer, block);
  if (!c) return false;
  const Ref r = c->tier(static_cast<int>(tier));
  if (r.pool < 0) return false;
  synchronize();
  kvx_check(kvx_read_page(pools_[r.pool], r.page, out), "read page");
  return true;
}

}  // namespace symsim
