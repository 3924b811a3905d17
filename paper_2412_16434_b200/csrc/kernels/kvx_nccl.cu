// K3 over NCCL: a migration's pages moved with ncclSend / ncclRecv — the
// collective-library variant of the reference's per-layer NetArrive
// (kvstore.cpp:753-769, SURVEY.md §8b "kvx_migrate(..., mode{CE, SM_FUSED,
// NCCL})"). Per chunk (one migration layer): K1 packs the chunk's pages into
// a staging slot, one NCCL group sends it to the receiver and receives the
// peer's chunk into the other slot, K2 unpacks what arrived. The page movers
// are this library's kernels; the transfer is NCCL's.
//
// NCCL is resolved at run time (dlopen "libnccl.so.2"): inside a PyTorch
// process that is the NCCL torch already loaded; libkvx itself has no link
// dependency on it and loads where NCCL is absent (every call then fails with
// KVX_ERR_UNSUPPORTED).

#include <dlfcn.h>

#include <algorithm>
#include <cstring>
#include <mutex>

#include "kvx_common.cuh"

namespace kvx {
namespace {

// The subset of nccl.h used here (ABI-stable since NCCL 2.0).
using ncclComm_t = void*;
constexpr int kNcclInt8 = 0;  // ncclInt8 / ncclChar
using FnSend = int (*)(const void*, size_t, int, int, ncclComm_t, cudaStream_t);
using FnRecv = int (*)(void*, size_t, int, int, ncclComm_t, cudaStream_t);
using FnGroup = int (*)();
using FnErr = const char* (*)(int);
using FnUid = int (*)(void*);
using FnDestroy = int (*)(ncclComm_t);

struct Uid128 {
  char bytes[128];
};
using FnInitRank = int (*)(ncclComm_t*, int, Uid128, int);

struct Nccl {
  FnSend send = nullptr;
  FnRecv recv = nullptr;
  FnGroup group_start = nullptr, group_end = nullptr;
  FnErr error = nullptr;
  FnUid unique_id = nullptr;
  FnInitRank init_rank = nullptr;
  FnDestroy destroy = nullptr;
  bool ok = false;
};

const Nccl& nccl() {
  static Nccl n;
  static std::once_flag once;
  std::call_once(once, [] {
    void* h = dlopen("libnccl.so.2", RTLD_NOW | RTLD_GLOBAL);
    if (!h) h = dlopen("libnccl.so", RTLD_NOW | RTLD_GLOBAL);
    if (!h) return;
    n.send = reinterpret_cast<FnSend>(dlsym(h, "ncclSend"));
    n.recv = reinterpret_cast<FnRecv>(dlsym(h, "ncclRecv"));
    n.group_start = reinterpret_cast<FnGroup>(dlsym(h, "ncclGroupStart"));
    n.group_end = reinterpret_cast<FnGroup>(dlsym(h, "ncclGroupEnd"));
    n.error = reinterpret_cast<FnErr>(dlsym(h, "ncclGetErrorString"));
    n.unique_id = reinterpret_cast<FnUid>(dlsym(h, "ncclGetUniqueId"));
    n.init_rank = reinterpret_cast<FnInitRank>(dlsym(h, "ncclCommInitRank"));
    n.destroy = reinterpret_cast<FnDestroy>(dlsym(h, "ncclCommDestroy"));
    n.ok = n.send && n.recv && n.group_start && n.group_end && n.error && n.unique_id && n.init_rank && n.destroy;
  });
  return n;
}

int need_nccl(const char* who) {
  if (nccl().ok) return KVX_OK;
  set_error(std::string(who) + ": NCCL (libnccl.so.2) is not available in this process");
  return KVX_ERR_UNSUPPORTED;
}

int nccl_fail(int r, const char* who) {
  set_error(std::string(who) + ": " + (nccl().error ? nccl().error(r) : "NCCL error") + " (" + std::to_string(r) +
            ")");
  return KVX_ERR_CUDA;
}

}  // namespace
}  // namespace kvx

extern "C" {

int kvx_nccl_get_unique_id(void* id128) {
  if (!id128) return kvx::fail_arg("kvx_nccl_get_unique_id: null out");
  if (int rc = kvx::need_nccl("kvx_nccl_get_unique_id")) return rc;
  kvx::Uid128 id{};
  if (int r = kvx::nccl().unique_id(&id)) return kvx::nccl_fail(r, "kvx_nccl_get_unique_id");
  std::memcpy(id128, id.bytes, 128);
  return KVX_OK;
}

int kvx_nccl_comm_init_rank(void** comm, int nranks, const void* id128, int rank, int device) {
  if (!comm || !id128 || nranks <= 0 || rank < 0 || rank >= nranks)
    return kvx::fail_arg("kvx_nccl_comm_init_rank: bad arguments");
  if (int rc = kvx::need_nccl("kvx_nccl_comm_init_rank")) return rc;
  kvx::DeviceGuard guard(device);
  kvx::Uid128 id{};
  std::memcpy(id.bytes, id128, 128);
  if (int r = kvx::nccl().init_rank(comm, nranks, id, rank)) return kvx::nccl_fail(r, "kvx_nccl_comm_init_rank");
  return KVX_OK;
}

int kvx_nccl_comm_destroy(void* comm) {
  if (!comm) return KVX_OK;
  if (int rc = kvx::need_nccl("kvx_nccl_comm_destroy")) return rc;
  if (int r = kvx::nccl().destroy(comm)) return kvx::nccl_fail(r, "kvx_nccl_comm_destroy");
  return KVX_OK;
}

uint64_t kvx_migrate_nccl_staging_bytes(uint64_t page_bytes, uint64_t pages_per_chunk) {
  return 2 * page_bytes * pages_per_chunk;
}

int kvx_migrate_nccl(const kvx_pool* send_pool, const uint32_t* d_send_ids, uint64_t n_send, int send_peer,
                     kvx_pool* recv_pool, const uint32_t* d_recv_ids, uint64_t n_recv, int recv_peer,
                     uint64_t pages_per_chunk, void* comm, void* d_staging, uint64_t staging_bytes, void* stream) {
  const bool sending = n_send > 0, receiving = n_recv > 0;
  if (!sending && !receiving) return KVX_OK;
  if (!comm || !d_staging || pages_per_chunk == 0) return kvx::fail_arg("kvx_migrate_nccl: null comm / staging");
  if ((sending && (!send_pool || !d_send_ids || send_peer < 0)) ||
      (receiving && (!recv_pool || !d_recv_ids || recv_peer < 0)))
    return kvx::fail_arg("kvx_migrate_nccl: a side with pages needs its pool, ids and peer");
  const uint64_t pb = sending ? send_pool->page_bytes : recv_pool->page_bytes;
  if (sending && receiving && send_pool->page_bytes != recv_pool->page_bytes)
    return kvx::fail_arg("kvx_migrate_nccl: page size mismatch");
  if (staging_bytes < kvx_migrate_nccl_staging_bytes(pb, pages_per_chunk))
    return kvx::fail_arg("kvx_migrate_nccl: staging smaller than 2 x pages_per_chunk pages");
  if (int rc = kvx::need_nccl("kvx_migrate_nccl")) return rc;
  const kvx::Nccl& N = kvx::nccl();
  const cudaStream_t st = kvx::as_stream(stream);
  uint8_t* out_slot = static_cast<uint8_t*>(d_staging);
  uint8_t* in_slot = out_slot + pb * pages_per_chunk;
  const uint64_t chunks_send = (n_send + pages_per_chunk - 1) / pages_per_chunk;
  const uint64_t chunks_recv = (n_recv + pages_per_chunk - 1) / pages_per_chunk;
  const uint64_t chunks = chunks_send > chunks_recv ? chunks_send : chunks_recv;
  for (uint64_t c = 0; c < chunks; ++c) {
    const uint64_t s0 = c * pages_per_chunk, r0 = c * pages_per_chunk;
    const uint64_t ns = s0 < n_send ? std::min(pages_per_chunk, n_send - s0) : 0;
    const uint64_t nr = r0 < n_recv ? std::min(pages_per_chunk, n_recv - r0) : 0;
    if (ns)
      if (int rc = kvx_pack(send_pool, d_send_ids + s0, ns, out_slot, KVX_COPY_AUTO, stream)) return rc;
    if (int r = N.group_start()) return kvx::nccl_fail(r, "kvx_migrate_nccl: ncclGroupStart");
    if (ns)
      if (int r = N.send(out_slot, ns * pb, kvx::kNcclInt8, send_peer, comm, st))
        return kvx::nccl_fail(r, "kvx_migrate_nccl: ncclSend");
    if (nr)
      if (int r = N.recv(in_slot, nr * pb, kvx::kNcclInt8, recv_peer, comm, st))
        return kvx::nccl_fail(r, "kvx_migrate_nccl: ncclRecv");
    if (int r = N.group_end()) return kvx::nccl_fail(r, "kvx_migrate_nccl: ncclGroupEnd");
    if (nr)
      if (int rc = kvx_unpack(recv_pool, d_recv_ids + r0, nr, in_slot, KVX_COPY_AUTO, stream)) return rc;
  }
  return KVX_OK;
}

}  // extern "C"
