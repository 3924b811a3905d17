#pragma once
// Physical KV payload behind the tiered store — B200 build.
//
// NodePayload implements TierBackend (kvstore.hpp): it gives every block
// copy the state machine creates a real page and moves the bytes with the
// kvx_* kernels / copy engines (include/kvx.h) at the moment the reference
// semantics say the copy comes into existence:
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
//   DISK copy    -> a page of the disk pool (pinned host memory standing in
//                   for the SSD tier; copy engines)
//
// This is the "lockstep" mode of SURVEY.md §7 hard part 1: the event order is
// the reference clock's (apply_transfer in (complete_at, id) order) and every
// physical move is complete before the call returns, so block-table state is
// bit-identical to the reference and every copy's bytes can be verified.
// Migrated layers land in receiver-GPU memory while the ledger still says
// Host (kvstore.cpp:914-923), which keeps ledger parity exact (SURVEY.md §7
// hard part 2, option 1): the follow-up LoadH2D becomes an HBM->HBM copy.

#include <cstdint>
#include <map>
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
  std::uint64_t disk_pages = 0;     // DISK tier stand-in (pinned host)
  std::uint64_t seed = 0;           // content of Created blocks
  int fill_mode = KVX_FILL_VALUES;
};

class NodePayload;

// Process-wide view of the nodes, so a receiver can find the migration
// source of a session (Simulation::start_migration, simcore.cpp:132-141,
// freezes the source and then imports on the receiver).
class PayloadCluster {
 public:
  void add(NodePayload* node);
  NodePayload* node(int id) const;
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
  // Which pool holds the block's `tier` copy (-1: none).
  int pool_of(std::uint32_t session, std::uint16_t layer, std::uint32_t block, Tier tier) const;
  // Bytes moved per BlockEvent kind since construction.
  const std::uint64_t* bytes_moved() const { return moved_; }
  kvx_pool* pool(Pool p) const { return pools_[p]; }
  void* stream() const { return stream_; }

 private:
  struct Ref {
    std::int8_t pool = -1;
    std::uint32_t page = 0;
  };
  struct Copies {
    Ref tier[3];  // indexed by Tier
  };
  static std::uint64_t key(std::uint32_t s, std::uint16_t l, std::uint32_t b) {
    return (static_cast<std::uint64_t>(s) << 36) | (static_cast<std::uint64_t>(l) << 20) | b;
  }
  std::uint32_t alloc(Pool p);
  void release(const Ref& r);
  Ref best_source(std::uint32_t s, std::uint16_t l, std::uint32_t b, int exclude_tier) const;
  // Copies src pages -> dst pages (grouped by source pool) and waits.
  void move(std::vector<Ref>& src, const std::vector<Ref>& dst, NodePayload& src_node, bool push_from_source);
  std::uint32_t* device_ids(const std::vector<std::uint32_t>& ids, int slot);

  PayloadCluster* cluster_;
  int node_;
  PayloadOptions opts_;
  std::uint64_t page_bytes_ = 0;
  kvx_pool* pools_[4] = {nullptr, nullptr, nullptr, nullptr};
  std::vector<std::uint32_t> free_[4];
  std::unordered_map<std::uint64_t, Copies> blocks_;
  std::map<std::uint32_t, int> import_src_;
  void* stream_ = nullptr;
  std::uint32_t* d_ids_[2] = {nullptr, nullptr};
  std::size_t d_ids_cap_[2] = {0, 0};
  void* d_tags_ = nullptr;
  std::size_t d_tags_cap_ = 0;
  std::uint64_t moved_[8] = {0, 0, 0, 0, 0, 0, 0, 0};
};

}  // namespace symsim
