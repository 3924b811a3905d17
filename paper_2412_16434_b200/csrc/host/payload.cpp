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

#include "symsim/payload.hpp"

#include <nvtx3/nvToolsExt.h>  // header-only NVTX v3: ranges show per lane in nsys / ncu

#include <algorithm>
#include <chrono>
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

}  // namespace

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
// lanes and per-page fences

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

// Make `runner`'s lane wait for every other lane's batch still touching
// `pages` (reads and writes alike: WAR, RAW and WAW are all covered).
void NodePayload::wait_fences(NodePayload& runner, int lane, const std::vector<Touch>& pages) {
  // A lane completes its batches in ticket order, so waiting for the newest
  // ticket seen per foreign lane covers every page fenced by that lane.
  std::vector<std::pair<Lane*, std::uint64_t>> need;
  for (const Touch& t : pages) {
    const Fence& f = t.first->fence(t.second);
    if (f.ticket == 0 || (f.node == runner.node_ && f.lane == lane)) continue;  // same stream: ordered
    NodePayload* owner = f.node == runner.node_ ? &runner
                         : f.node == node_      ? this
                         : cluster_             ? cluster_->node(f.node)
                                                : nullptr;
    if (!owner) continue;  // that node is gone, and synchronized on its way out
    Lane* L = &owner->lanes_[f.lane];
    auto it = std::find_if(need.begin(), need.end(), [L](const auto& e) { return e.first == L; });
    if (it == need.end())
      need.emplace_back(L, f.ticket);
    else
      it->second = std::max(it->second, f.ticket);
  }
  bool waited = false;
  for (const auto& [L, ticket] : need)
    if (void* ev = L->event_for(ticket)) {  // nullptr: already complete
      kvx_check(kvx_stream_wait_event(runner.lanes_[lane].stream, ev), "stream wait");
      waited = true;
    }
  if (waited) ++cross_waits_;
}

// Close the batch just queued on `runner`'s lane: one event, and every page
// it touched now points at it.
void NodePayload::set_fences(NodePayload& runner, int lane, const std::vector<Touch>& pages) {
  Lane& L = runner.lanes_[lane];
  L.retire();  // keeps the pending list short on lanes nobody waits on
  void* ev = nullptr;
  kvx_check(kvx_event_create(&ev), "event");
  kvx_check(kvx_event_record(ev, L.stream), "event record");
  const std::uint64_t ticket = L.next++;
  L.pending.emplace_back(ticket, ev);
  for (const Touch& t : pages) t.first->fence(t.second) = Fence{runner.node_, lane, ticket};
}

// ---------------------------------------------------------------------------
// node: pools, pages, scratch

NodePayload::NodePayload(PayloadCluster* cluster, int node_id, const PayloadOptions& opts)
    : cluster_(cluster), node_(node_id), opts_(opts) {
  page_bytes_ = kvx_page_bytes(&opts_.layout);
  if (page_bytes_ == 0) throw std::runtime_error("payload: empty page layout");
  for (Lane& L : lanes_) kvx_check(kvx_stream_create(opts_.device, &L.stream), "stream");
  const std::uint64_t counts[4] = {opts_.device_pages, opts_.host_pages, opts_.landing_pages, opts_.disk_pages};
  for (int p = 0; p < 4; ++p) {
    if (counts[p] == 0) continue;
    if (p == kDevicePool || p == kLandingPool)
      kvx_check(kvx_pool_create(opts_.device, counts[p], page_bytes_, &pools_[p]), "device pool");
    else if (p == kDiskPool && !opts_.disk_path.empty())
      kvx_check(kvx_pool_create_file(opts_.disk_path.c_str(), counts[p], page_bytes_, &pools_[p]), "disk file");
    else
      kvx_check(kvx_pool_create_host(counts[p], page_bytes_, &pools_[p]), "host pool");
    free_[p].resize(counts[p]);
    fences_[p].resize(counts[p]);
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
  for (auto& entry : inflight_) kvx_event_destroy(entry.second.event);
  for (auto*& p : pools_)
    if (p) kvx_pool_destroy(p);
  for (Lane& L : lanes_) {
    L.drain();
    for (auto* d : L.d_ids) kvx_free(d);
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
  return total - free_[p].size();
}

std::uint64_t NodePayload::pages_in_flight(Pool p) const {
  std::uint64_t n = 0;
  for (const auto& entry : inflight_)
    for (const Ref& r : entry.second.pages) n += r.pool == p;
  return n;
}

std::uint32_t NodePayload::alloc(Pool p) {
  if (free_[p].empty()) {
    static const char* const kNames[] = {"device", "host", "landing", "disk"};
    throw std::runtime_error(std::string("payload: node ") + std::to_string(node_) + " " + kNames[p] +
                             " pool exhausted");
  }
  const std::uint32_t page = free_[p].back();
  free_[p].pop_back();
  return page;
}

// Re-deals a batch's freshly allocated pages (one pool) in ascending order:
// the free list is LIFO, so pages released in ascending order come back
// descending; ascending destinations pair with ascending sources into long
// runs of consecutive ids, which the copy engines move as one copy each.
void sort_pages(std::vector<std::uint32_t>& pages) { std::sort(pages.begin(), pages.end()); }

// A freed page may still be read by queued work; its fence makes any later
// writer on another lane wait for that work, so no host sync is needed.
void NodePayload::release(const Ref& r) {
  if (r.pool >= 0) free_[r.pool].push_back(r.page);
}

std::uint32_t* NodePayload::device_ids(Lane& lane, const std::vector<std::uint32_t>& ids, int slot) {
  if (ids.size() > lane.d_ids_cap[slot]) {
    if (lane.d_ids[slot]) {
      kvx_check(kvx_stream_synchronize(lane.stream), "sync");  // queued kernels may still read it
      kvx_free(lane.d_ids[slot]);
    }
    lane.d_ids[slot] = nullptr;
    const std::size_t cap = std::max<std::size_t>(ids.size(), 4096);
    void* p = nullptr;
    kvx_check(kvx_malloc(opts_.device, cap * sizeof(std::uint32_t), &p), "id scratch");
    lane.d_ids[slot] = static_cast<std::uint32_t*>(p);
    lane.d_ids_cap[slot] = cap;
  }
  kvx_check(kvx_memcpy_async(lane.d_ids[slot], ids.data(), ids.size() * sizeof(std::uint32_t), lane.stream),
            "ids upload");
  return lane.d_ids[slot];
}

// Best existing copy of a block on this node, fastest tier first, skipping
// `exclude_tier` (the tier being created).
NodePayload::Ref NodePayload::best_source(std::uint32_t s, std::uint16_t l, std::uint32_t b,
                                          int exclude_tier) const {
  const auto it = blocks_.find(key(s, l, b));
  if (it == blocks_.end()) return Ref{};
  for (int t = 0; t < 3; ++t)
    if (t != exclude_tier && it->second.tier[t].pool >= 0) return it->second.tier[t];
  return Ref{};
}

bool NodePayload::inflight_source(std::uint32_t s, std::uint16_t l, std::uint32_t b, int exclude_tier, Ref* page,
                                  void** event) const {
  for (int t = 0; t < 3; ++t) {
    if (t == exclude_tier) continue;
    const auto it = inflight_by_block_.find(key(s, l, b) * 4 + t);
    if (it == inflight_by_block_.end()) continue;
    const InFlight& f = inflight_.at(it->second.id);
    *page = f.pages[it->second.index];  // the slot recorded at posting: O(1)
    *event = f.event;
    return true;
  }
  return false;
}

bool NodePayload::device_block_table(std::uint32_t session, std::uint16_t layer, std::uint32_t n,
                                     std::uint32_t* out) const {
  for (std::uint32_t b = 0; b < n; ++b) {
    const auto it = blocks_.find(key(session, layer, b));
    if (it == blocks_.end() || it->second.tier[0].pool != kDevicePool) return false;
    out[b] = it->second.tier[0].page;
  }
  return true;
}

int NodePayload::pool_of(std::uint32_t s, std::uint16_t l, std::uint32_t b, Tier tier) const {
  const auto it = blocks_.find(key(s, l, b));
  return it == blocks_.end() ? -1 : it->second.tier[static_cast<int>(tier)].pool;
}

// Queues src[i] -> dst[i] (dst in this node's pools, all in one pool)
// grouped by (source pool, destination pool). HBM<->HBM pairs use the SM/TMA
// page mover with device id lists; anything touching pinned host memory uses
// the copy engines. With `push` the work runs on the source node's PEER lane
// and stores into this node's memory (the NVLink / peer path of a
// migration); otherwise on this node's IN lane (destination in HBM), DISK
// lane (disk-tier source or destination) or OUT lane (HBM -> host). The batch first waits on `waits` and on
// the fences of every page it touches.
void* NodePayload::issue(const std::vector<Ref>& src, const std::vector<Ref>& dst, NodePayload& src_node, bool push,
                         const std::vector<void*>& waits) {
  NodePayload& runner = push ? src_node : *this;
  const int dp0 = dst.empty() ? static_cast<int>(kDevicePool) : dst[0].pool;
  const bool from_disk = std::any_of(src.begin(), src.end(), [](const Ref& r) { return r.pool == kDiskPool; });
  const int lane = push                                           ? kLanePeer
                   : (dp0 == kDevicePool || dp0 == kLandingPool) ? kLaneIn
                   : (dp0 == kDiskPool || from_disk)             ? kLaneDisk
                                                                 : kLaneOut;
  Lane& L = runner.lanes_[lane];
  static const char* const kLaneNames[] = {"kvs:IN", "kvs:OUT", "kvs:DISK", "kvs:PEER"};
  nvtxRangePushA(kLaneNames[lane]);  // host-side enqueue of this batch (NVTX, SURVEY.md §5 tracing)
  struct PopRange {
    ~PopRange() { nvtxRangePop(); }
  } pop_range;
  std::vector<Touch> touched;
  touched.reserve(src.size() + dst.size());
  for (const Ref& r : src) touched.emplace_back(&src_node, r);
  for (const Ref& r : dst) touched.emplace_back(this, r);
  for (void* ev : waits) kvx_check(kvx_stream_wait_event(L.stream, ev), "stream wait");
  wait_fences(runner, lane, touched);
  for (int sp = 0; sp < 4; ++sp)
    for (int dp = 0; dp < 4; ++dp) {
      std::vector<std::uint32_t> s_ids, d_ids;
      for (std::size_t i = 0; i < src.size(); ++i)
        if (src[i].pool == sp && dst[i].pool == dp) {
          s_ids.push_back(src[i].page);
          d_ids.push_back(dst[i].page);
        }
      if (s_ids.empty()) continue;
      kvx_pool* from = src_node.pools_[sp];
      kvx_pool* to = pools_[dp];
      const bool on_device = (sp == kDevicePool || sp == kLandingPool) && (dp == kDevicePool || dp == kLandingPool);
      // A file pool on either side (the source node's DISK copy may be a file
      // even when ours is not) with HBM on the other goes through a bounce.
      const bool file_side = kvx_pool_file_direct(from) >= 0 || kvx_pool_file_direct(to) >= 0;
      const bool hbm_side = sp == kDevicePool || sp == kLandingPool || dp == kDevicePool || dp == kLandingPool;
      const bool file_hop = file_side && hbm_side;
      if (on_device) {
        const std::uint32_t* ds = runner.device_ids(L, s_ids, 0);
        const std::uint32_t* dd = runner.device_ids(L, d_ids, 1);
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
  set_fences(runner, lane, touched);
  return L.stream;
}

// ---------------------------------------------------------------------------
// residency transitions

void NodePayload::tier_gained(std::uint32_t session, std::uint16_t layer, Tier tier, BlockEvent why,
                              const std::vector<std::uint32_t>& blocks) {
  const int t = static_cast<int>(tier);
  moved_[static_cast<int>(why)] += blocks.size() * page_bytes_;

  if (why == BlockEvent::Created) {
    std::vector<std::uint32_t> pages;
    std::vector<kvx_block_tag> tags;
    std::vector<Touch> touched;
    for (std::uint32_t b : blocks) {
      Copies& c = blocks_[key(session, layer, b)];
      release(c.tier[t]);
      c.tier[t] = Ref{};
    }
    for (std::size_t i = 0; i < blocks.size(); ++i) pages.push_back(alloc(kDevicePool));
    sort_pages(pages);
    for (std::size_t i = 0; i < blocks.size(); ++i) {
      Copies& c = blocks_[key(session, layer, blocks[i])];
      c.tier[t] = Ref{kDevicePool, pages[i]};
      tags.push_back(kvx_block_tag{session, layer, blocks[i]});
      touched.emplace_back(this, c.tier[t]);
    }
    Lane& L = lanes_[kLaneIn];
    wait_fences(*this, kLaneIn, touched);
    const std::uint32_t* d_pages = device_ids(L, pages, 0);
    if (tags.size() * sizeof(kvx_block_tag) > d_tags_cap_) {
      if (d_tags_) kvx_check(kvx_stream_synchronize(L.stream), "sync");
      kvx_free(d_tags_);
      d_tags_cap_ = std::max<std::size_t>(tags.size() * sizeof(kvx_block_tag), 65536);
      kvx_check(kvx_malloc(opts_.device, d_tags_cap_, &d_tags_), "tag scratch");
    }
    kvx_check(kvx_memcpy_async(d_tags_, tags.data(), tags.size() * sizeof(kvx_block_tag), L.stream), "tags upload");
    kvx_check(kvx_fill_pages(pools_[kDevicePool], d_pages, static_cast<const kvx_block_tag*>(d_tags_), pages.size(),
                             opts_.seed, &opts_.layout, opts_.fill_mode, L.stream),
              "fill");
    set_fences(*this, kLaneIn, touched);
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
  InFlight f = std::move(inflight_.at(applying_));
  inflight_.erase(applying_);
  applying_valid_ = false;
  std::vector<bool> used(f.blocks.size(), false);
  std::vector<std::uint32_t> missing;
  // f.blocks ascends (posted over block_lo..block_hi in order), so each
  // gained block is found by bisection: O(n log n) per layer, not O(n^2)
  // (2,048-block layers at Llama-3.1-70B @32K).
  for (std::uint32_t b : blocks) {
    const auto pos = std::lower_bound(f.blocks.begin(), f.blocks.end(), b);
    const std::size_t i = static_cast<std::size_t>(pos - f.blocks.begin());
    if (pos == f.blocks.end() || *pos != b) {
      missing.push_back(b);  // its source appeared only after scheduling
      continue;
    }
    Copies& c = blocks_[key(session, layer, b)];
    release(c.tier[t]);
    c.tier[t] = f.pages[i];
    used[i] = true;
  }
  for (std::size_t i = 0; i < f.blocks.size(); ++i)
    if (!used[i]) release(f.pages[i]);
  kvx_event_destroy(f.event);
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
  for (std::uint32_t b : blocks) {
    const Ref from = src_node->best_source(session, layer, b, src_node == this ? t : -1);
    if (from.pool < 0)
      throw std::runtime_error("payload: no source copy for session " + std::to_string(session) + " layer " +
                               std::to_string(layer) + " block " + std::to_string(b) + " (" +
                               block_event_name(why) + ")");
    Copies& c = blocks_[key(session, layer, b)];
    release(c.tier[t]);
    c.tier[t] = Ref{};
    src.push_back(from);
  }
  std::vector<std::uint32_t> pages;
  for (std::size_t i = 0; i < blocks.size(); ++i) pages.push_back(alloc(dest));
  sort_pages(pages);
  for (std::size_t i = 0; i < blocks.size(); ++i) {
    Copies& c = blocks_[key(session, layer, blocks[i])];
    c.tier[t] = Ref{static_cast<std::int8_t>(dest), pages[i]};
    dst.push_back(c.tier[t]);
  }
  issue(src, dst, *src_node, push, {});
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
  for (std::uint32_t b : blocks) {
    const auto it = blocks_.find(key(session, layer, b));
    if (it == blocks_.end()) continue;
    release(it->second.tier[t]);
    it->second.tier[t] = Ref{};
    const Copies& c = it->second;
    if (c.tier[0].pool < 0 && c.tier[1].pool < 0 && c.tier[2].pool < 0) blocks_.erase(it);
  }
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
  InFlight f;
  f.tier = t;
  f.session = tr.session;
  f.layer = tr.layer;
  std::vector<Ref> src, dst;
  std::vector<void*> waits;
  for (std::uint64_t b64 = tr.block_lo; b64 <= tr.block_hi; ++b64) {
    const auto b = static_cast<std::uint32_t>(b64);
    const auto have = blocks_.find(key(tr.session, tr.layer, b));
    if (have != blocks_.end() && have->second.tier[t].pool >= 0) continue;  // already there
    if (inflight_by_block_.count(key(tr.session, tr.layer, b) * 4 + t)) continue;  // already coming
    const int exclude = src_node == this ? t : -1;
    Ref from = src_node->best_source(tr.session, tr.layer, b, exclude);
    if (from.pool < 0) {  // chained behind a move still in flight on the source side
      void* ev = nullptr;
      if (!src_node->inflight_source(tr.session, tr.layer, b, exclude, &from, &ev)) continue;
      waits.push_back(ev);
    }
    src.push_back(from);
    f.blocks.push_back(b);
  }
  if (f.blocks.empty()) return;
  std::vector<std::uint32_t> pages;
  for (std::size_t i = 0; i < f.blocks.size(); ++i) pages.push_back(alloc(dest));
  sort_pages(pages);
  for (std::uint32_t pg : pages) {
    dst.push_back(Ref{static_cast<std::int8_t>(dest), pg});
    f.pages.push_back(dst.back());
  }
  // Sources still being written by another move are chained explicitly (and
  // by their fences); recycled destination pages wait on their fences.
  std::sort(waits.begin(), waits.end());
  waits.erase(std::unique(waits.begin(), waits.end()), waits.end());
  void* lane_stream = issue(src, dst, *src_node, push, waits);
  kvx_check(kvx_event_create(&f.event), "event");
  kvx_check(kvx_event_record(f.event, lane_stream), "event record");
  for (std::size_t i = 0; i < f.blocks.size(); ++i)
    inflight_by_block_[key(tr.session, tr.layer, f.blocks[i]) * 4 + t] = InFlightSlot{tr.id, static_cast<std::uint32_t>(i)};
  moved_[7] += f.blocks.size() * page_bytes_;  // bytes issued ahead of their apply
  inflight_.emplace(tr.id, std::move(f));
  ++posted_;
}

void NodePayload::transfer_retired(std::uint64_t id, bool voided) {
  applying_valid_ = false;
  if (!opts_.free_running) return;
  const auto it = inflight_.find(id);
  if (it == inflight_.end()) return;
  InFlight& f = it->second;
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
  // Later moves touching these pages are ordered by the pages' fences.
  for (std::uint32_t b : f.blocks) {
    const auto k = key(f.session, f.layer, b) * 4 + f.tier;
    const auto jt = inflight_by_block_.find(k);
    if (jt != inflight_by_block_.end() && jt->second.id == id) inflight_by_block_.erase(jt);
  }
  if (voided) {
    for (const Ref& r : f.pages) release(r);
    kvx_event_destroy(f.event);
    inflight_.erase(it);
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
  const auto it = blocks_.find(key(session, layer, block));
  if (it == blocks_.end()) return false;
  const Ref r = it->second.tier[static_cast<int>(tier)];
  if (r.pool < 0) return false;
  synchronize();
  kvx_check(kvx_read_page(pools_[r.pool], r.page, out), "read page");
  return true;
}

}  // namespace symsim
