// Tiered KV block store — B200 build, host state machine.
//
// Re-implemented from the module spec and
// the reference tests; every public operation reproduces the reference
// KvStore's observable behaviour bit for bit (returned values, scheduled
// transfer ids and completion times, ledger rows, counters, exceptions), which
// tests/test_state_parity.py checks against the reference compiled as the
// oracle (oracle/_ref). Reference anchors are given per function as
// kvstore.cpp:<lines> (= /root/reference/proj/src/kvstore.cpp).
//
// Representation differs from the reference: one flag byte per block
// (residency bits indexed by Tier plus the four pending markers), tier
// counters in an array indexed by Tier, and optional physical backing through
// TierBackend, which receives every residency transition batched per
// (session, layer, tier) so device pages and their bytes follow the state.

#include "symsim/kvstore.hpp"

#include <algorithm>
#include <mutex>
#include <stdexcept>

namespace symsim {

namespace {

std::mutex& factory_mutex() {
  static std::mutex m;
  return m;
}
TierBackendFactory& factory_slot() {
  static TierBackendFactory f;
  return f;
}

bool evicts_before(const BlockMeta& a, const BlockMeta& b) {
  if (a.key.layer != b.key.layer) return a.key.layer > b.key.layer;
  if (a.session_bytes != b.session_bytes) return a.session_bytes < b.session_bytes;
  if (a.key.block_index != b.key.block_index) return a.key.block_index > b.key.block_index;
  return a.session_id < b.session_id;
}

}  // namespace

void set_default_tier_backend_factory(TierBackendFactory factory) {
  std::lock_guard<std::mutex> lock(factory_mutex());
  factory_slot() = std::move(factory);
}

const char* tier_name(Tier t) {
  switch (t) {
    case Tier::Device: return "device";
    case Tier::Host: return "host";
    case Tier::Disk: return "disk";
  }
  return "?";
}

const char* reason_name(TransferReason r) {
  static const char* const kNames[] = {"prefetch", "demand", "purge", "persist", "migrate"};
  const auto i = static_cast<unsigned>(r);
  return i < 5 ? kNames[i] : "?";
}

const char* block_event_name(BlockEvent e) {
  static const char* const kNames[] = {"created",   "load_h2d", "load_disk_host", "host_copy",
                                       "disk_write", "swap_out", "net_arrive"};
  const auto i = static_cast<unsigned>(e);
  return i < 7 ? kNames[i] : "?";
}

// kvstore.cpp:34-44 — total order; the comparator is the spec's key tuple.
std::vector<BlockMeta> evict_order(std::vector<BlockMeta> candidates) {
  if (std::any_of(candidates.begin(), candidates.end(), [](const BlockMeta& m) { return m.pinned; }))
    throw std::runtime_error("evict_order: pinned block in candidate set");
  std::sort(candidates.begin(), candidates.end(), evicts_before);
  return candidates;
}

// kvstore.cpp:46-59 — the compute increment of layer i is the exact integer
// share floor((i+1)S/L) - floor(iS/L), so the increments sum to S.
GateResult pipeline_gate(const std::vector<Ns>& layer_ready, Ns compute_ready, Ns step_ns) {
  if (layer_ready.empty()) throw std::runtime_error("pipeline_gate: no layers");
  const auto n = static_cast<std::int64_t>(layer_ready.size());
  Ns end = compute_ready;
  Ns prev_share = 0;
  for (std::int64_t i = 0; i < n; ++i) {
    const Ns share = (i + 1) * step_ns / n;
    end = std::max(end, layer_ready[static_cast<std::size_t>(i)]) + (share - prev_share);
    prev_share = share;
  }
  GateResult g;
  g.first_step_end = end;
  g.gate_start = end - step_ns;
  g.stall = std::max<Ns>(0, end - (compute_ready + step_ns));
  return g;
}

// ---------------------------------------------------------------------------
// construction, registry

KvStore::KvStore(const GpuProfile& gpu, const LinkProfile& links, const Options& opts)
    : gpu_(gpu), links_(links), opts_(opts) {
  gpu_.validate();
  links_.validate();
  if (opts_.block_tokens <= 0) throw std::runtime_error("kvstore: block_tokens must be positive");
  device_cap_ = opts_.device_capacity > 0 ? opts_.device_capacity : gpu_.hbm_capacity;
  page_bytes_ = kv_bytes_per_layer(opts_.block_tokens, gpu_);
  std::lock_guard<std::mutex> lock(factory_mutex());
  if (factory_slot()) backend_ = factory_slot()(opts_.node_id);
}

void KvStore::register_session(std::uint32_t session, const std::string& id, PriorityClass priority) {
  if (finalized_) throw std::logic_error("kvstore: register after finalize");
  Session& s = sessions_[session];
  if (backend_)  // re-registration discards any block table the session had
    for (std::size_t l = 0; l < s.layers.size(); ++l) {
      std::vector<std::uint32_t> lost[3];
      for (std::size_t b = 0; b < s.layers[l].size(); ++b)
        for (unsigned t = 0; t < 3; ++t)
          if (s.layers[l][b] & (1u << t)) lost[t].push_back(static_cast<std::uint32_t>(b));
      for (unsigned t = 0; t < 3; ++t) report_loss(session, static_cast<std::uint16_t>(l), Tier(t), lost[t]);
    }
  s.name = id;
  s.priority = priority;
  const auto layers = static_cast<std::size_t>(gpu_.num_layers);
  s.layers.assign(layers, Layer{});
  s.load_eta.assign(layers, 0);
  s.inbound_eta.assign(layers, 0);
}

// kvstore.cpp:81-88 — lexicographic rank over (id, index).
void KvStore::finalize_sessions() {
  std::vector<std::pair<std::string, std::uint32_t>> order;
  order.reserve(sessions_.size());
  for (const auto& [idx, s] : sessions_) order.emplace_back(s.name, idx);
  std::sort(order.begin(), order.end());
  int rank = 0;
  for (const auto& entry : order) sessions_[entry.second].lex_rank = rank++;
  finalized_ = true;
}

KvStore::Session& KvStore::sess(std::uint32_t session) {
  const auto it = sessions_.find(session);
  if (it == sessions_.end()) throw std::logic_error("kvstore: unknown session");
  return it->second;
}

const KvStore::Session& KvStore::sess(std::uint32_t session) const {
  const auto it = sessions_.find(session);
  if (it == sessions_.end()) throw std::logic_error("kvstore: unknown session");
  return it->second;
}

std::int64_t KvStore::blocks_of(const Session& s) const {
  // int-valued like the reference's blocks_per_layer (kvstore.cpp:102-104)
  return static_cast<int>((s.tokens + opts_.block_tokens - 1) / opts_.block_tokens);
}

std::int64_t KvStore::footprint(const Session& s) const {
  return blocks_of(s) * gpu_.num_layers * page_bytes_;
}

// ---------------------------------------------------------------------------
// small helpers

Ns KvStore::link_done(Channel& ch, Ns ready, std::int64_t bytes, Link link) {
  return ch.enqueue(ready, transfer_time(bytes, link, links_));
}

std::uint64_t KvStore::post(const Move& m, std::vector<ScheduledTransfer>& scheduled) {
  const std::uint64_t id = next_id_++;
  scheduled.push_back(ScheduledTransfer{id, m.complete_at});
  inflight_.emplace(id, m);
  if (backend_) {
    static const BlockEvent kEvent[] = {BlockEvent::LoadH2D,   BlockEvent::LoadDiskHost, BlockEvent::HostCopy,
                                        BlockEvent::DiskWrite, BlockEvent::SwapOut,      BlockEvent::NetArrive};
    static const Tier kTo[] = {Tier::Device, Tier::Host, Tier::Host, Tier::Disk, Tier::Host, Tier::Host};
    TierBackend::TransferInfo info;
    info.id = id;
    info.session = m.session;
    info.layer = m.layer;
    info.block_lo = m.lo;
    info.block_hi = m.hi;
    info.kind = kEvent[static_cast<int>(m.kind)];
    info.to = kTo[static_cast<int>(m.kind)];
    info.bytes = m.bytes;
    info.complete_at = m.complete_at;
    backend_->transfer_posted(info);
  }
  return id;
}

void KvStore::log(Ns time, std::uint32_t session, int layer_lo, int layer_hi, Tier from, Tier to,
                  std::int64_t bytes, TransferReason reason) {
  TransferRecord r;
  r.time = time;
  r.node = opts_.node_id;
  r.session = session;
  r.layer_lo = static_cast<std::uint16_t>(layer_lo);
  r.layer_hi = static_cast<std::uint16_t>(layer_hi);
  r.from = from;
  r.to = to;
  r.bytes = bytes;
  r.reason = reason;
  ledger_.push_back(r);
}

void KvStore::clear_drop_marks(Session& s) {
  for (Layer& lay : s.layers)
    for (std::uint8_t& f : lay) f = static_cast<std::uint8_t>(f & ~kDropOnPersist);
}

void KvStore::report_gain(std::uint32_t session, std::uint16_t layer, Tier tier, BlockEvent why,
                          const std::vector<std::uint32_t>& blocks) {
  // Reported even when empty for applied transfers: a free-running backend
  // must learn that none of its in-flight pages were wanted.
  if (backend_ && (!blocks.empty() || why != BlockEvent::Created))
    backend_->tier_gained(session, layer, tier, why, blocks);
}

void KvStore::report_loss(std::uint32_t session, std::uint16_t layer, Tier tier,
                          const std::vector<std::uint32_t>& blocks) {
  if (backend_ && !blocks.empty()) backend_->tier_lost(session, layer, tier, blocks);
}

// Ensures `bytes` more fit in HOST, evicting LRU host copies (that also have
// a DISK copy) when they do not. kvstore.cpp:237-238 and its siblings.
bool KvStore::make_host_room(std::int64_t bytes, Ns now) {
  if (used_[1] + bytes <= opts_.host_capacity) return true;
  return evict_host_lru(bytes - (opts_.host_capacity - used_[1]), now);
}

// kvstore.cpp:273-308 — whole idle sessions, least recently used first; a
// session qualifies when nothing is in flight toward HOST/DEVICE for it and
// it has at least one block persisted on both HOST and DISK.
bool KvStore::evict_host_lru(std::int64_t bytes_needed, Ns now) {
  if (bytes_needed <= 0) return true;
  std::vector<std::pair<Ns, std::uint32_t>> victims;
  for (const auto& [idx, s] : sessions_) {
    if (s.active || s.leaving || s.inbound_layers > 0) continue;
    std::uint8_t seen_any = 0;
    bool doubly_backed = false;
    for (const Layer& lay : s.layers)
      for (std::uint8_t f : lay) {
        seen_any |= f;
        doubly_backed = doubly_backed || (f & kBacked) == kBacked;
      }
    if (!(seen_any & (kHostPending | kLoadPending)) && doubly_backed) victims.emplace_back(s.last_use, idx);
  }
  std::sort(victims.begin(), victims.end());
  std::int64_t freed = 0;
  for (const auto& victim : victims) {
    const std::uint32_t idx = victim.second;
    Session& s = sessions_[idx];
    std::int64_t got = 0;
    for (std::size_t l = 0; l < s.layers.size(); ++l) {
      std::vector<std::uint32_t> dropped;
      Layer& lay = s.layers[l];
      std::uint8_t* const f = lay.data();  // locals: byte stores would force reloads through `lay`
      const std::size_t nb = lay.size();
      const std::int64_t pb = page_bytes_;
      for (std::size_t b = 0; b < nb; ++b)
        if ((f[b] & kBacked) == kBacked) {
          f[b] = static_cast<std::uint8_t>(f[b] & ~kOnHost);
          got += pb;
          if (backend_) dropped.push_back(static_cast<std::uint32_t>(b));
        }
      report_loss(idx, static_cast<std::uint16_t>(l), Tier::Host, dropped);
    }
    if (got > 0) {
      used_[1] -= got;
      freed += got;
      log(now, idx, 0, gpu_.num_layers - 1, Tier::Host, Tier::Disk, got, TransferReason::Purge);
    }
    if (freed >= bytes_needed) return true;
  }
  return freed >= bytes_needed;
}

// ---------------------------------------------------------------------------
// queries

std::int64_t KvStore::cached_tokens(std::uint32_t session) const { return sess(session).tokens; }
std::int64_t KvStore::session_bytes(std::uint32_t session) const { return footprint(sess(session)); }
bool KvStore::has_any_copy(std::uint32_t session) const { return sess(session).tokens > 0; }
int KvStore::pending_persists(std::uint32_t session) const { return sess(session).persists_in_flight; }
bool KvStore::migrating_out(std::uint32_t session) const { return sess(session).leaving; }
bool KvStore::is_active(std::uint32_t session) const { return sess(session).active; }

bool KvStore::fully_device_resident(std::uint32_t session) const {
  const Session& s = sess(session);
  if (s.tokens == 0) return false;
  for (const Layer& lay : s.layers)
    if (std::any_of(lay.begin(), lay.end(), [](std::uint8_t f) { return !(f & kOnDev); })) return false;
  return true;
}

std::uint8_t KvStore::residency(std::uint32_t session, std::uint16_t layer, std::uint32_t block) const {
  const Session& s = sess(session);
  if (layer >= s.layers.size() || block >= s.layers[layer].size()) return 0;
  return static_cast<std::uint8_t>(s.layers[layer][block] & kResidency);
}

std::size_t KvStore::blocks_in_layer(std::uint32_t session, std::uint16_t layer) const {
  const Session& s = sess(session);
  return layer < s.layers.size() ? s.layers[layer].size() : 0;
}

void KvStore::set_active(std::uint32_t session, bool active, Ns now) {
  Session& s = sess(session);
  s.active = active;
  s.last_use = now;
  if (!active) return;
  clear_drop_marks(s);  // wanted again: cancel deferred drops and demotions
  void_session_offload(session);
}

std::int64_t KvStore::bytes_for_new_blocks(std::uint32_t session, std::int64_t new_tokens) const {
  const Session& s = sess(session);
  const std::int64_t bt = opts_.block_tokens;
  const std::int64_t grown = (s.tokens + new_tokens + bt - 1) / bt - (s.tokens + bt - 1) / bt;
  return grown * gpu_.num_layers * page_bytes_;
}

std::int64_t KvStore::bytes_for_load(std::uint32_t session) const {
  std::int64_t n = 0;
  for (const Layer& lay : sess(session).layers)
    n += std::count_if(lay.begin(), lay.end(), [](std::uint8_t f) { return !(f & (kOnDev | kLoadPending)); });
  return n * page_bytes_;
}

std::int64_t KvStore::bytes_for_promote(std::uint32_t session) const { return bytes_for_load(session); }

void KvStore::reserve_device(std::int64_t bytes) {
  if (bytes < 0) throw std::logic_error("kvstore: negative reservation");
  if (used_[0] + bytes > device_cap_) throw std::logic_error("kvstore: device reservation overflows capacity");
  used_[0] += bytes;
}

void KvStore::unreserve_device(std::int64_t bytes) {
  if (bytes < 0 || bytes > used_[0]) throw std::logic_error("kvstore: bad unreserve");
  used_[0] -= bytes;
}

// ---------------------------------------------------------------------------
// append (kvstore.cpp:202-271)

std::vector<BlockKey> KvStore::append_blocks(std::uint32_t session, std::int64_t new_tokens, Ns now,
                                             std::vector<ScheduledTransfer>& scheduled) {
  if (new_tokens <= 0) throw std::logic_error("append_blocks: token count must be positive");
  Session& s = sess(session);
  if (s.leaving) throw std::logic_error("append_blocks: session is migrating out");
  s.last_use = now;
  const auto first = static_cast<std::uint32_t>(blocks_of(s));
  s.tokens += new_tokens;
  const auto last = static_cast<std::uint32_t>(blocks_of(s));
  std::vector<BlockKey> created;
  if (first == last) return created;

  const std::int64_t fresh = last - first;
  const int layers = gpu_.num_layers;
  used_[0] += fresh * layers * page_bytes_;
  if (used_[0] > device_cap_)
    throw std::logic_error("append_blocks: device capacity exceeded (missing reservation)");

  created.reserve(static_cast<std::size_t>(fresh * layers));
  std::vector<std::uint32_t> range;
  if (backend_)
    for (std::uint32_t b = first; b < last; ++b) range.push_back(b);
  for (int l = 0; l < layers; ++l) {
    Layer& lay = s.layers[static_cast<std::size_t>(l)];
    lay.resize(last);
    std::vector<std::uint32_t> lost[3];
    std::uint8_t* const f = lay.data();
    const bool track = backend_ != nullptr;
    for (std::uint32_t b = first; b < last; ++b) {
      if (track)
        for (unsigned t = 1; t < 3; ++t)
          if (f[b] & (1u << t)) lost[t].push_back(b);
      f[b] = static_cast<std::uint8_t>((f[b] & ~kResidency) | kOnDev);
      created.push_back(BlockKey{session, static_cast<std::uint16_t>(l), b});
    }
    if (!backend_) continue;
    report_loss(session, static_cast<std::uint16_t>(l), Tier::Host, lost[1]);
    report_loss(session, static_cast<std::uint16_t>(l), Tier::Disk, lost[2]);
    report_gain(session, static_cast<std::uint16_t>(l), Tier::Device, BlockEvent::Created, range);
  }

  if (!opts_.write_behind) return created;
  // Write-behind: per layer one D2H copy of the new range, then a disk write
  // chained behind it (or issued directly when HOST has no room).
  const std::int64_t bytes = fresh * page_bytes_;
  for (int l = 0; l < layers; ++l) {
    Layer& lay = s.layers[static_cast<std::size_t>(l)];
    Move m;
    m.session = session;
    m.layer = static_cast<std::uint16_t>(l);
    m.lo = first;
    m.hi = last - 1;
    m.bytes = bytes;
    m.reason = TransferReason::Persist;
    Ns disk_ready = now;
    if (make_host_room(bytes, now)) {
      m.kind = Kind::HostCopy;
      m.complete_at = link_done(pcie_down_, now, bytes, Link::PcieD2H);
      used_[1] += bytes;
      std::uint8_t* const f = lay.data();
      for (std::uint32_t b = first; b < last; ++b) f[b] |= kHostPending;
      disk_ready = m.complete_at;
      post(m, scheduled);
    }
    m.kind = Kind::DiskWrite;
    m.complete_at = link_done(disk_out_, disk_ready, bytes, Link::DiskWrite);
    std::uint8_t* const fd = lay.data();
    for (std::uint32_t b = first; b < last; ++b) fd[b] |= kDiskPending;
    s.persists_in_flight += 1;
    post(m, scheduled);
  }
  return created;
}

// ---------------------------------------------------------------------------
// eviction (kvstore.cpp:310-431)

std::vector<BlockMeta> KvStore::evictable_blocks(bool spare_high_priority) const {
  std::vector<BlockMeta> out;
  for (const auto& [idx, s] : sessions_) {
    if (s.active || s.leaving) continue;
    if (spare_high_priority && s.priority == PriorityClass::High) continue;
    const std::int64_t fp = footprint(s);
    for (std::size_t l = 0; l < s.layers.size(); ++l)
      for (std::size_t b = 0; b < s.layers[l].size(); ++b) {
        const std::uint8_t f = s.layers[l][b];
        if (!(f & kOnDev) || (f & kDropOnPersist)) continue;
        BlockMeta m;
        m.key = BlockKey{idx, static_cast<std::uint16_t>(l), static_cast<std::uint32_t>(b)};
        m.session_id = s.name;
        m.session_bytes = fp;
        out.push_back(std::move(m));
      }
  }
  return evict_order(std::move(out));
}

std::int64_t KvStore::purge_from_device(std::int64_t bytes_needed, Ns now, bool spare_high_priority,
                                        std::vector<ScheduledTransfer>& scheduled) {
  if (bytes_needed <= 0) return 0;

  // Eviction order without materialising every block: one entry per
  // (session, layer) holding a droppable DEVICE block, sorted on the order's
  // leading keys; entries tied on (layer, footprint) interleave block by
  // block, highest index first, lexicographic rank breaking the tie.
  struct Run {
    std::uint16_t layer;
    std::int64_t fp;
    int rank;
    std::uint32_t session;
  };
  std::vector<Run> runs;
  for (const auto& [idx, s] : sessions_) {
    if (s.active || s.leaving) continue;
    if (spare_high_priority && s.priority == PriorityClass::High) continue;
    const std::int64_t fp = footprint(s);
    for (std::size_t l = 0; l < s.layers.size(); ++l) {
      const Layer& lay = s.layers[l];
      if (std::any_of(lay.begin(), lay.end(), [](std::uint8_t f) { return (f & kOnDev) && !(f & kDropOnPersist); }))
        runs.push_back(Run{static_cast<std::uint16_t>(l), fp, s.lex_rank, idx});
    }
  }
  std::sort(runs.begin(), runs.end(), [](const Run& a, const Run& b) {
    if (a.layer != b.layer) return a.layer > b.layer;
    if (a.fp != b.fp) return a.fp < b.fp;
    return a.rank < b.rank;
  });

  std::int64_t freed = 0;
  for (std::size_t head = 0; head < runs.size() && freed < bytes_needed;) {
    std::size_t tail = head + 1;
    while (tail < runs.size() && runs[tail].layer == runs[head].layer && runs[tail].fp == runs[head].fp) ++tail;
    const std::size_t width = tail - head;
    int deepest = 0;
    for (std::size_t k = head; k < tail; ++k)
      deepest = std::max(deepest, static_cast<int>(sessions_[runs[k].session].layers[runs[k].layer].size()));
    std::vector<std::int64_t> instant(width, 0);
    std::vector<std::vector<std::uint32_t>> dropped(width);

    for (int b = deepest - 1; b >= 0 && freed < bytes_needed; --b) {
      for (std::size_t k = head; k < tail && freed < bytes_needed; ++k) {
        Session& s = sessions_[runs[k].session];
        Layer& lay = s.layers[runs[k].layer];
        if (b >= static_cast<int>(lay.size())) continue;
        std::uint8_t& f = lay[static_cast<std::size_t>(b)];
        if (!(f & kOnDev) || (f & kDropOnPersist)) continue;
        if (f & kBacked) {
          // Another tier holds it: dropping DEVICE residency moves no bytes.
          f = static_cast<std::uint8_t>(f & ~kOnDev);
          used_[0] -= page_bytes_;
          freed += page_bytes_;
          instant[k - head] += page_bytes_;
          if (backend_) dropped[k - head].push_back(static_cast<std::uint32_t>(b));
        } else if (opts_.write_behind) {
          f |= kDropOnPersist;  // its persist is in flight; drop when it lands
        } else {
          if (!make_host_room(page_bytes_, now)) continue;
          Move m;
          m.session = runs[k].session;
          m.layer = runs[k].layer;
          m.lo = m.hi = static_cast<std::uint32_t>(b);
          m.kind = Kind::SwapOut;
          m.bytes = page_bytes_;
          m.reason = TransferReason::Purge;
          m.complete_at = link_done(pcie_down_, now, page_bytes_, Link::PcieD2H);
          used_[1] += page_bytes_;
          f |= kHostPending | kDropOnPersist;
          post(m, scheduled);
        }
      }
    }
    for (std::size_t k = head; k < tail; ++k) {
      if (instant[k - head] == 0) continue;
      const Layer& lay = sessions_[runs[k].session].layers[runs[k].layer];
      if (backend_) {
        std::vector<std::uint32_t> ascending(dropped[k - head].rbegin(), dropped[k - head].rend());
        report_loss(runs[k].session, runs[k].layer, Tier::Device, ascending);
      }
      const bool on_host = std::any_of(lay.begin(), lay.end(), [](std::uint8_t f) { return (f & kOnHost) != 0; });
      log(now, runs[k].session, runs[k].layer, runs[k].layer, Tier::Device, on_host ? Tier::Host : Tier::Disk,
          instant[k - head], TransferReason::Purge);
    }
    head = tail;
  }
  return freed;
}

// ---------------------------------------------------------------------------
// loads toward DEVICE (kvstore.cpp:433-640)

std::optional<LoadPlan> KvStore::plan_layerwise_load(std::uint32_t session, Ns now, Ns compute_per_layer,
                                                     TransferReason reason,
                                                     std::vector<ScheduledTransfer>& scheduled) {
  Session& s = sess(session);
  s.last_use = now;
  const int layers = gpu_.num_layers;
  LoadPlan plan;
  plan.layer_ready.assign(static_cast<std::size_t>(layers), now);
  if (s.tokens == 0) {
    plan.decode_start = now;
    plan.finish = now + static_cast<Ns>(layers) * compute_per_layer;
    return plan;
  }
  clear_drop_marks(s);

  // Dry run: bytes to reserve, and every block with no source at all.
  // (Counters are locals: stores through uint8_t flags alias any member.)
  std::int64_t need_blocks = 0;
  std::string missing;
  for (int l = 0; l < layers; ++l) {
    const Layer& lay = s.layers[static_cast<std::size_t>(l)];
    const bool inbound = s.inbound_eta[static_cast<std::size_t>(l)] != 0;
    for (std::size_t b = 0; b < lay.size(); ++b) {
      if (lay[b] & (kOnDev | kLoadPending)) continue;
      ++need_blocks;
      if (!(lay[b] & kBacked) && !inbound) missing += " " + std::to_string(l) + ":" + std::to_string(b);
    }
  }
  const std::int64_t need = need_blocks * page_bytes_;
  if (!missing.empty())
    throw std::runtime_error("plan_layerwise_load: session " + s.name + " missing layer:block" + missing);
  if (need > device_cap_ - used_[0]) return std::nullopt;
  used_[0] += need;

  for (int l = 0; l < layers; ++l) {
    const auto li = static_cast<std::size_t>(l);
    Layer& lay = s.layers[li];
    const Ns ready = s.load_eta[li] > 0 ? std::max(now, s.load_eta[li]) : now;
    std::int64_t src_blocks[3] = {0, 0, 0};  // [host, disk, inbound]
    std::uint32_t lo = 0, hi = 0;
    bool any = false;
    {
      std::uint8_t* const p = lay.data();
      const std::size_t nb = lay.size();
      std::int64_t host = 0, disk = 0, inbound = 0;
      for (std::size_t b = 0; b < nb; ++b) {
        const std::uint8_t f = p[b];
        if (f & (kOnDev | kLoadPending)) continue;
        if (!any) lo = static_cast<std::uint32_t>(b);
        hi = static_cast<std::uint32_t>(b);
        any = true;
        p[b] = static_cast<std::uint8_t>(f | kLoadPending);
        host += (f & kOnHost) != 0;
        disk += !(f & kOnHost) && (f & kOnDisk);
        inbound += !(f & (kOnHost | kOnDisk));
      }
      src_blocks[0] = host;
      src_blocks[1] = disk;
      src_blocks[2] = inbound;
    }
    const std::int64_t src_bytes[3] = {src_blocks[0] * page_bytes_, src_blocks[1] * page_bytes_,
                                       src_blocks[2] * page_bytes_};
    if (!any) {
      plan.layer_ready[li] = ready;
      continue;
    }
    plan.any_load = true;

    Move m;
    m.session = session;
    m.layer = static_cast<std::uint16_t>(l);
    m.lo = lo;
    m.hi = hi;
    m.reason = reason;
    Ns up_ready = now;
    if (src_bytes[1] > 0) {  // DISK blocks stage through HOST
      if (!make_host_room(src_bytes[1], now))
        throw std::runtime_error("kvstore: host tier too small to stage a layer from disk");
      m.kind = Kind::LoadDiskHost;
      m.bytes = src_bytes[1];
      m.complete_at = link_done(disk_in_, now, src_bytes[1], Link::DiskRead);
      used_[1] += src_bytes[1];
      post(m, scheduled);
      up_ready = std::max(up_ready, m.complete_at);
    }
    if (src_bytes[2] > 0) up_ready = std::max(up_ready, s.inbound_eta[li]);  // wait for the migration
    m.kind = Kind::LoadH2D;
    m.bytes = src_bytes[0] + src_bytes[1] + src_bytes[2];
    m.complete_at = link_done(pcie_up_, up_ready, m.bytes, Link::PcieH2D);
    post(m, scheduled);
    s.load_eta[li] = m.complete_at;
    plan.layer_ready[li] = std::max(ready, m.complete_at);
  }

  plan.decode_start = plan.layer_ready[0];
  Ns end = now;
  for (Ns r : plan.layer_ready) end = std::max(end, r) + compute_per_layer;
  plan.finish = end;
  plan.total_stall = std::max<Ns>(0, end - (now + static_cast<Ns>(layers) * compute_per_layer));
  return plan;
}

PromoteResult KvStore::promote(std::uint32_t session, Ns now, std::vector<ScheduledTransfer>& scheduled) {
  Session& s = sess(session);
  s.last_use = now;
  PromoteResult res;
  if (s.tokens == 0) return res;
  clear_drop_marks(s);

  bool device_full = false;
  for (int l = 0; l < gpu_.num_layers; ++l) {
    const auto li = static_cast<std::size_t>(l);
    Layer& lay = s.layers[li];
    std::int64_t host_blocks = 0, disk_blocks = 0;
    std::uint32_t lo = 0, hi = 0;
    bool any = false;
    for (std::size_t b = 0; b < lay.size(); ++b) {
      const std::uint8_t f = lay[b];
      if ((f & (kOnDev | kLoadPending)) || !(f & kBacked)) continue;  // inbound: demand path
      if (!any) lo = static_cast<std::uint32_t>(b);
      hi = static_cast<std::uint32_t>(b);
      any = true;
      ++((f & kOnHost) ? host_blocks : disk_blocks);
    }
    const std::int64_t host_bytes = host_blocks * page_bytes_, disk_bytes = disk_blocks * page_bytes_;
    if (!any) {
      if (!device_full) ++res.device_layers;
      continue;
    }
    const std::int64_t bytes = host_bytes + disk_bytes;
    Move m;
    m.session = session;
    m.layer = static_cast<std::uint16_t>(l);
    m.lo = lo;
    m.hi = hi;
    m.reason = TransferReason::Prefetch;

    if (device_full || used_[0] + bytes > device_cap_) {
      // No DEVICE room from here on: at least lift DISK-only blocks to HOST.
      device_full = true;
      if (disk_bytes == 0 || !make_host_room(disk_bytes, now)) continue;
      m.kind = Kind::LoadDiskHost;
      m.bytes = disk_bytes;
      m.complete_at = link_done(disk_in_, now, disk_bytes, Link::DiskRead);
      used_[1] += disk_bytes;
      post(m, scheduled);
      ++res.staged_layers;
      res.scheduled = true;
      continue;
    }
    used_[0] += bytes;
    Ns up_ready = now;
    if (disk_bytes > 0) {
      if (!make_host_room(disk_bytes, now))
        throw std::runtime_error("kvstore: host tier too small to stage a layer from disk");
      m.kind = Kind::LoadDiskHost;
      m.bytes = disk_bytes;
      m.complete_at = link_done(disk_in_, now, disk_bytes, Link::DiskRead);
      used_[1] += disk_bytes;
      post(m, scheduled);
      up_ready = m.complete_at;
    }
    m.kind = Kind::LoadH2D;
    m.bytes = bytes;
    m.complete_at = link_done(pcie_up_, up_ready, bytes, Link::PcieH2D);
    {
      std::uint8_t* const p = lay.data();
      for (std::uint32_t b = lo; b <= hi; ++b)
        if (!(p[b] & kOnDev)) p[b] |= kLoadPending;
    }
    post(m, scheduled);
    s.load_eta[li] = m.complete_at;
    ++res.device_layers;
    res.scheduled = true;
  }
  return res;
}

// ---------------------------------------------------------------------------
// offload / release / migration (kvstore.cpp:642-789)

void KvStore::offload_session(std::uint32_t session, Ns now, std::vector<ScheduledTransfer>& scheduled) {
  Session& s = sess(session);
  s.last_use = now;
  std::int64_t unbacked_blocks = 0;
  for (const Layer& lay : s.layers)
    for (std::uint8_t f : lay) unbacked_blocks += (f & kOnDev) && !(f & kBacked);
  const std::int64_t unbacked = unbacked_blocks * page_bytes_;
  if (unbacked > 0 && !make_host_room(unbacked, now)) {
    // HOST cannot take it: drop the cache outright (from == to marks a drop).
    const std::int64_t dropped = footprint(s);
    release_session(session, now);
    log(now, session, 0, gpu_.num_layers - 1, Tier::Device, Tier::Device, dropped, TransferReason::Purge);
    return;
  }
  for (std::size_t l = 0; l < s.layers.size(); ++l) {
    Layer& lay = s.layers[l];
    std::int64_t copy = 0, demoted = 0;
    std::uint32_t lo = 0, hi = 0;
    bool any = false;
    std::vector<std::uint32_t> gone;
    {
      std::uint8_t* const p = lay.data();
      const std::size_t nb = lay.size();
      const std::int64_t pb = page_bytes_;
      const bool track = backend_ != nullptr;
      for (std::size_t b = 0; b < nb; ++b) {
        const std::uint8_t f = p[b];
        if (!(f & kOnDev)) continue;
        if (f & kBacked) {
          p[b] = static_cast<std::uint8_t>(f & ~kOnDev);
          demoted += pb;
          if (track) gone.push_back(static_cast<std::uint32_t>(b));
        } else {
          if (!any) lo = static_cast<std::uint32_t>(b);
          hi = static_cast<std::uint32_t>(b);
          any = true;
          copy += pb;
        }
      }
      used_[0] -= demoted;
    }
    report_loss(session, static_cast<std::uint16_t>(l), Tier::Device, gone);
    if (demoted > 0)
      log(now, session, static_cast<int>(l), static_cast<int>(l), Tier::Device, Tier::Host, demoted,
          TransferReason::Purge);
    if (!any || !make_host_room(copy, now)) continue;
    Move m;
    m.session = session;
    m.layer = static_cast<std::uint16_t>(l);
    m.lo = lo;
    m.hi = hi;
    m.kind = Kind::SwapOut;
    m.bytes = copy;
    m.reason = TransferReason::Persist;
    m.complete_at = link_done(pcie_down_, now, copy, Link::PcieD2H);
    used_[1] += copy;
    std::uint8_t* const p = lay.data();
    for (std::uint32_t b = lo; b <= hi; ++b)
      if ((p[b] & kOnDev) && !(p[b] & kBacked)) p[b] |= kHostPending | kDropOnPersist;
    post(m, scheduled);
  }
}

void KvStore::release_session(std::uint32_t session, Ns now) {
  Session& s = sess(session);
  void_session_loads(session);
  void_session_offload(session);
  for (auto& entry : inflight_)
    if (entry.second.session == session) entry.second.voided = true;
  std::int64_t held[3] = {0, 0, 0};
  for (std::size_t l = 0; l < s.layers.size(); ++l) {
    std::int64_t count[3] = {0, 0, 0};
    std::vector<std::uint32_t> lost[3];
    for (std::size_t b = 0; b < s.layers[l].size(); ++b) {
      const std::uint8_t f = s.layers[l][b];
      count[0] += f & kOnDev;
      count[1] += (f & kOnHost) >> 1;
      count[2] += (f & kOnDisk) >> 2;
      if (backend_)
        for (unsigned t = 0; t < 3; ++t)
          if (f & (1u << t)) lost[t].push_back(static_cast<std::uint32_t>(b));
    }
    for (unsigned t = 0; t < 3; ++t) {
      held[t] += count[t] * page_bytes_;
      report_loss(session, static_cast<std::uint16_t>(l), Tier(t), lost[t]);
    }
    s.layers[l].clear();
  }
  for (unsigned t = 0; t < 3; ++t) used_[t] -= held[t];
  s.tokens = 0;
  s.active = false;
  s.leaving = false;
  s.persists_in_flight = 0;
  s.inbound_layers = 0;
  std::fill(s.load_eta.begin(), s.load_eta.end(), 0);
  std::fill(s.inbound_eta.begin(), s.inbound_eta.end(), 0);
  s.last_use = now;
}

void KvStore::mark_migrating_out(std::uint32_t session) {
  Session& s = sess(session);
  if (s.leaving) throw std::runtime_error("kvstore: session already migrating");
  s.leaving = true;
  if (backend_) backend_->migrating_out(session);
}

std::vector<ScheduledTransfer> KvStore::import_migration(std::uint32_t session, std::int64_t tokens, Ns now) {
  Session& s = sess(session);
  if (s.tokens != 0) throw std::logic_error("import_migration: session already present");
  s.tokens = tokens;
  const std::int64_t nblocks = blocks_of(s);
  const std::int64_t layer_bytes = nblocks * page_bytes_;
  std::vector<ScheduledTransfer> out;
  s.last_use = now;
  if (backend_) backend_->importing(session, tokens);
  for (int l = 0; l < gpu_.num_layers; ++l) {
    const auto li = static_cast<std::size_t>(l);
    s.layers[li].assign(static_cast<std::size_t>(nblocks), 0);
    if (!make_host_room(layer_bytes, now))
      throw std::runtime_error("kvstore: host tier too small to receive a migrating cache");
    Move m;
    m.session = session;
    m.layer = static_cast<std::uint16_t>(l);
    m.lo = 0;
    m.hi = static_cast<std::uint32_t>(nblocks - 1);
    m.kind = Kind::NetArrive;
    m.bytes = layer_bytes;
    m.reason = TransferReason::Migrate;
    m.complete_at = link_done(net_rx_, now, layer_bytes, Link::Network);
    used_[1] += layer_bytes;
    s.inbound_eta[li] = m.complete_at;
    post(m, out);
    if (opts_.write_behind) {
      const Ns arrived = m.complete_at;
      m.kind = Kind::DiskWrite;
      m.reason = TransferReason::Persist;
      m.complete_at = link_done(disk_out_, arrived, layer_bytes, Link::DiskWrite);
      s.persists_in_flight += 1;
      for (std::uint8_t& f : s.layers[li]) f |= kDiskPending;
      post(m, out);
    }
  }
  s.inbound_layers = gpu_.num_layers;
  return out;
}

void KvStore::void_session_loads(std::uint32_t session) {
  Session& s = sess(session);
  for (auto& entry : inflight_) {
    Move& m = entry.second;
    if (m.session == session && (m.kind == Kind::LoadH2D || m.kind == Kind::LoadDiskHost)) m.voided = true;
  }
  std::fill(s.load_eta.begin(), s.load_eta.end(), 0);
  for (Layer& lay : s.layers)
    for (std::uint8_t& f : lay) f = static_cast<std::uint8_t>(f & ~kLoadPending);
}

void KvStore::void_session_offload(std::uint32_t session) {
  Session& s = sess(session);
  for (auto& entry : inflight_) {
    Move& m = entry.second;
    if (m.session != session || m.kind != Kind::SwapOut || m.voided) continue;
    m.voided = true;
    if (m.layer >= s.layers.size()) continue;
    Layer& lay = s.layers[m.layer];
    std::uint8_t* const p = lay.data();
    const std::uint64_t z = std::min<std::uint64_t>(static_cast<std::uint64_t>(m.hi) + 1, lay.size());
    for (std::uint64_t b = m.lo; b < z; ++b) p[b] = static_cast<std::uint8_t>(p[b] & ~(kHostPending | kDropOnPersist));
  }
}

// ---------------------------------------------------------------------------
// completion dispatch (kvstore.cpp:816-926)

KvStore::ApplyResult KvStore::apply_transfer(std::uint64_t id, Ns now) {
  const auto it = inflight_.find(id);
  if (it == inflight_.end()) throw std::logic_error("kvstore: unknown transfer id");
  const Move m = it->second;
  inflight_.erase(it);

  ApplyResult res;
  res.session = m.session;
  res.layer = m.layer;
  if (backend_) backend_->transfer_retired(id, m.voided);
  if (m.voided) {  // return the schedule-time reservation; the bytes are discarded
    if (m.kind == Kind::LoadH2D) used_[0] -= m.bytes;
    else if (m.kind != Kind::DiskWrite) used_[1] -= m.bytes;
    res.voided = true;
    return res;
  }

  Session& s = sess(m.session);
  if (m.layer >= s.layers.size() || s.layers[m.layer].empty())
    throw std::logic_error("kvstore: transfer for missing blocks");
  Layer& lay = s.layers[m.layer];
  const std::uint64_t stop = std::min<std::uint64_t>(static_cast<std::uint64_t>(m.hi) + 1, lay.size());

  std::vector<std::uint32_t> gained, dev_dropped;
  const bool track = backend_ != nullptr;  // hoisted: flag stores alias members
  std::uint8_t* const flags = lay.data();
  // Byte-flag loops below work on local copies of the bounds and the base
  // pointer: a uint8_t store may alias anything reached through a reference,
  // which would force a reload per element and block vectorisation.
  const std::uint64_t lo = m.lo;
  // Sets `bit` on every block of the range, remembering which ones are new.
  auto gain_bit = [&](std::uint8_t bit, std::uint8_t clear) {
    std::uint8_t* const f = flags;
    const std::uint64_t a = lo, z = stop;
    if (track)
      for (std::uint64_t b = a; b < z; ++b)
        if (!(f[b] & bit)) gained.push_back(static_cast<std::uint32_t>(b));
    const std::uint8_t keep = static_cast<std::uint8_t>(~clear);
    for (std::uint64_t b = a; b < z; ++b) f[b] = static_cast<std::uint8_t>((f[b] | bit) & keep);
  };
  // Completes a deferred drop: DEVICE residency leaves once a persist lands.
  auto settle_drop = [&]() {
    std::uint8_t* const f = flags;
    const std::uint64_t a = lo, z = stop;
    std::int64_t n = 0;
    constexpr std::uint8_t both = kDropOnPersist | kOnDev;
    if (track) {
      for (std::uint64_t b = a; b < z; ++b)
        if ((f[b] & both) == both) {
          f[b] = static_cast<std::uint8_t>(f[b] & ~both);
          ++n;
          dev_dropped.push_back(static_cast<std::uint32_t>(b));
        }
    } else {
      for (std::uint64_t b = a; b < z; ++b) {
        const bool hit = (f[b] & both) == both;
        n += hit;
        f[b] = static_cast<std::uint8_t>(hit ? f[b] & ~both : f[b]);
      }
    }
    used_[0] -= n * page_bytes_;
  };

  switch (m.kind) {
    case Kind::LoadH2D:
      gain_bit(kOnDev, kLoadPending);
      report_gain(m.session, m.layer, Tier::Device, BlockEvent::LoadH2D, gained);
      s.load_eta[m.layer] = 0;
      log(now, m.session, m.layer, m.layer, Tier::Host, Tier::Device, m.bytes, m.reason);
      res.device_layer_ready = true;
      break;
    case Kind::LoadDiskHost:
      gain_bit(kOnHost, 0);
      report_gain(m.session, m.layer, Tier::Host, BlockEvent::LoadDiskHost, gained);
      log(now, m.session, m.layer, m.layer, Tier::Disk, Tier::Host, m.bytes, m.reason);
      break;
    case Kind::HostCopy:
      gain_bit(kOnHost, kHostPending);
      report_gain(m.session, m.layer, Tier::Host, BlockEvent::HostCopy, gained);
      settle_drop();
      report_loss(m.session, m.layer, Tier::Device, dev_dropped);
      log(now, m.session, m.layer, m.layer, Tier::Device, Tier::Host, m.bytes, TransferReason::Persist);
      break;
    case Kind::DiskWrite:
      if (opts_.disk_capacity >= 0 && used_[2] + m.bytes > opts_.disk_capacity)
        throw std::runtime_error("kvstore: disk tier capacity exceeded");
      used_[2] += m.bytes;
      gain_bit(kOnDisk, kDiskPending);
      report_gain(m.session, m.layer, Tier::Disk, BlockEvent::DiskWrite, gained);
      settle_drop();
      report_loss(m.session, m.layer, Tier::Device, dev_dropped);
      log(now, m.session, m.layer, m.layer, Tier::Host, Tier::Disk, m.bytes, TransferReason::Persist);
      if (--s.persists_in_flight < 0) throw std::logic_error("kvstore: persist count underflow");
      res.persists_drained = s.persists_in_flight == 0;
      break;
    case Kind::SwapOut:
      gain_bit(kOnHost, kHostPending);
      report_gain(m.session, m.layer, Tier::Host, BlockEvent::SwapOut, gained);
      {
        std::uint8_t* const f = flags;
        const std::uint64_t a = lo, z = stop;
        std::int64_t n = 0;
        for (std::uint64_t b = a; b < z; ++b) {
          if (f[b] & kOnDev) {
            ++n;
            if (track) dev_dropped.push_back(static_cast<std::uint32_t>(b));
          }
          f[b] = static_cast<std::uint8_t>(f[b] & ~(kOnDev | kDropOnPersist));
        }
        used_[0] -= n * page_bytes_;
      }
      report_loss(m.session, m.layer, Tier::Device, dev_dropped);
      log(now, m.session, m.layer, m.layer, Tier::Device, Tier::Host, m.bytes, m.reason);
      break;
    case Kind::NetArrive:
      gain_bit(kOnHost, 0);
      report_gain(m.session, m.layer, Tier::Host, BlockEvent::NetArrive, gained);
      s.inbound_eta[m.layer] = 0;
      s.inbound_layers -= 1;
      log(now, m.session, m.layer, m.layer, Tier::Host, Tier::Host, m.bytes, TransferReason::Migrate);
      res.migration_arrived = true;
      res.migration_complete = s.inbound_layers == 0;
      break;
  }
  return res;
}

// ---------------------------------------------------------------------------
// diagnostics

std::string KvStore::device_usage_debug() const {
  // Same buckets and format as the reference diagnostic (kvstore.cpp:928-950),
  // which the reference Engine embeds in its device-pressure error message.
  std::int64_t bytes[4] = {0, 0, 0, 0};  // active, migrating, offloading, idle
  int count[4] = {0, 0, 0, 0};
  for (const auto& [idx, s] : sessions_) {
    std::int64_t dev = 0, dropping = 0;
    for (const Layer& lay : s.layers)
      for (std::uint8_t f : lay)
        if (f & kOnDev) {
          dev += page_bytes_;
          if (f & kDropOnPersist) dropping += page_bytes_;
        }
    if (dev == 0) continue;
    const int bucket = s.active ? 0 : s.leaving ? 1 : (dropping == dev ? 2 : 3);
    bytes[bucket] += dev;
    count[bucket] += 1;
  }
  static const char* const kLabel[] = {"active=", " migrating=", " offloading=", " idle="};
  std::string out;
  for (int i = 0; i < 4; ++i)
    out += kLabel[i] + std::to_string(bytes[i] / 1000000) + "MB/" + std::to_string(count[i]);
  return out;
}

void KvStore::check_budgets() const {
  if (used_[0] < 0 || used_[0] > device_cap_) throw std::logic_error("kvstore: device budget out of range");
  if (used_[1] < 0 || used_[1] > opts_.host_capacity) throw std::logic_error("kvstore: host budget out of range");
  if (used_[2] < 0 || (opts_.disk_capacity >= 0 && used_[2] > opts_.disk_capacity))
    throw std::logic_error("kvstore: disk budget out of range");
}

}  // namespace symsim
