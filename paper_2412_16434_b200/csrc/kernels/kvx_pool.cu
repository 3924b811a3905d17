// Page pools and the error channel of the kvx C ABI (include/kvx.h).
//
// A pool is a flat array of equal-size pages. A DEVICE pool is one cudaMalloc
// in HBM; a HOST pool is pinned, device-mapped host memory (the HOST tier's
// physical backing, reachable by kernels over PCIe); a pool can also wrap
// caller memory or a peer GPU's pool opened through CUDA IPC, which is how a
// migration kernel on the source GPU stores straight into the receiver's
// pages over NVLink (SURVEY.md §5 "Distributed communication backend").

#include <cstdio>
#include <cstring>
#include <mutex>
#include <string>
#include <vector>

#include "kvx_common.cuh"

namespace kvx {

namespace {
thread_local std::string g_error;
}

void set_error(const std::string& msg) { g_error = msg; }

int fail_cuda(cudaError_t e, const char* what) {
  g_error = std::string(what) + ": " + cudaGetErrorName(e) + " (" + cudaGetErrorString(e) + ")";
  return KVX_ERR_CUDA;
}

int fail_arg(const char* what) {
  g_error = what;
  return KVX_ERR_ARG;
}

int sm_count(int device) {
  static std::mutex mu;
  static std::vector<int> cache;
  std::lock_guard<std::mutex> lock(mu);
  if (device < 0) device = 0;
  if (static_cast<int>(cache.size()) <= device) cache.resize(device + 1, 0);
  if (cache[device] == 0) {
    int n = 0;
    if (cudaDeviceGetAttribute(&n, cudaDevAttrMultiProcessorCount, device) != cudaSuccess || n <= 0) n = 148;
    cache[device] = n;
  }
  return cache[device];
}

}  // namespace kvx

extern "C" {

const char* kvx_last_error(void) { return kvx::g_error.c_str(); }

int kvx_version(void) { return 1; }

uint64_t kvx_page_bytes(const kvx_page_layout* l) {
  if (!l) return 0;
  const uint64_t elt = l->dtype == KVX_DTYPE_BF16 ? 2 : 4;
  return 2ull * l->num_kv_heads * l->block_tokens * l->head_dim * elt;
}

int kvx_pool_create(int device, uint64_t num_pages, uint64_t page_bytes, kvx_pool** out) {
  if (!out || num_pages == 0 || page_bytes == 0 || page_bytes % 16 != 0)
    return kvx::fail_arg("kvx_pool_create: need num_pages > 0 and page_bytes a positive multiple of 16");
  int prev = 0;
  KVX_CUDA_TRY(cudaGetDevice(&prev), "kvx_pool_create: cudaGetDevice");
  KVX_CUDA_TRY(cudaSetDevice(device), "kvx_pool_create: cudaSetDevice");
  void* p = nullptr;
  const cudaError_t e = cudaMalloc(&p, num_pages * page_bytes);
  cudaSetDevice(prev);
  if (e != cudaSuccess) return kvx::fail_cuda(e, "kvx_pool_create: cudaMalloc");
  auto* pool = new kvx_pool;
  pool->base = static_cast<uint8_t*>(p);
  pool->num_pages = num_pages;
  pool->page_bytes = page_bytes;
  pool->device = device;
  pool->owned = true;
  *out = pool;
  return KVX_OK;
}

int kvx_pool_create_host(uint64_t num_pages, uint64_t page_bytes, kvx_pool** out) {
  if (!out || num_pages == 0 || page_bytes == 0 || page_bytes % 16 != 0)
    return kvx::fail_arg("kvx_pool_create_host: need num_pages > 0 and page_bytes a positive multiple of 16");
  void* p = nullptr;
  KVX_CUDA_TRY(cudaHostAlloc(&p, num_pages * page_bytes, cudaHostAllocMapped | cudaHostAllocPortable),
               "kvx_pool_create_host: cudaHostAlloc");
  auto* pool = new kvx_pool;
  pool->base = static_cast<uint8_t*>(p);
  pool->num_pages = num_pages;
  pool->page_bytes = page_bytes;
  pool->device = -1;
  pool->owned = true;
  pool->host = true;
  *out = pool;
  return KVX_OK;
}

int kvx_pool_wrap(int device, void* base, uint64_t num_pages, uint64_t page_bytes, kvx_pool** out) {
  if (!out || !base || num_pages == 0 || page_bytes == 0 || page_bytes % 16 != 0 ||
      reinterpret_cast<uintptr_t>(base) % 16 != 0)
    return kvx::fail_arg("kvx_pool_wrap: need a 16-B aligned base and page_bytes a positive multiple of 16");
  auto* pool = new kvx_pool;
  pool->base = static_cast<uint8_t*>(base);
  pool->num_pages = num_pages;
  pool->page_bytes = page_bytes;
  pool->device = device;
  pool->host = device < 0;
  *out = pool;
  return KVX_OK;
}

int kvx_pool_destroy(kvx_pool* pool) {
  if (!pool) return KVX_OK;
  cudaError_t e = cudaSuccess;
  if (pool->ipc) e = cudaIpcCloseMemHandle(pool->base);
  else if (pool->owned && pool->host) e = cudaFreeHost(pool->base);
  else if (pool->owned) e = cudaFree(pool->base);
  delete pool;
  if (e != cudaSuccess) return kvx::fail_cuda(e, "kvx_pool_destroy");
  return KVX_OK;
}

void* kvx_pool_base(const kvx_pool* pool) { return pool ? pool->base : nullptr; }
uint64_t kvx_pool_num_pages(const kvx_pool* pool) { return pool ? pool->num_pages : 0; }
uint64_t kvx_pool_page_bytes(const kvx_pool* pool) { return pool ? pool->page_bytes : 0; }
int kvx_pool_device(const kvx_pool* pool) { return pool ? pool->device : -1; }

int kvx_pool_ipc_export(const kvx_pool* pool, void* handle64) {
  if (!pool || !handle64 || pool->host) return kvx::fail_arg("kvx_pool_ipc_export: need a DEVICE pool");
  static_assert(sizeof(cudaIpcMemHandle_t) == 64, "IPC handle size");
  cudaIpcMemHandle_t h;
  KVX_CUDA_TRY(cudaIpcGetMemHandle(&h, pool->base), "kvx_pool_ipc_export: cudaIpcGetMemHandle");
  std::memcpy(handle64, &h, 64);
  return KVX_OK;
}

int kvx_pool_ipc_open(int device, const void* handle64, uint64_t num_pages, uint64_t page_bytes, kvx_pool** out) {
  if (!out || !handle64 || num_pages == 0 || page_bytes % 16 != 0) return kvx::fail_arg("kvx_pool_ipc_open: bad args");
  cudaIpcMemHandle_t h;
  std::memcpy(&h, handle64, 64);
  int prev = 0;
  KVX_CUDA_TRY(cudaGetDevice(&prev), "kvx_pool_ipc_open: cudaGetDevice");
  KVX_CUDA_TRY(cudaSetDevice(device), "kvx_pool_ipc_open: cudaSetDevice");
  void* p = nullptr;
  const cudaError_t e = cudaIpcOpenMemHandle(&p, h, cudaIpcMemLazyEnablePeerAccess);
  cudaSetDevice(prev);
  if (e != cudaSuccess) return kvx::fail_cuda(e, "kvx_pool_ipc_open: cudaIpcOpenMemHandle");
  auto* pool = new kvx_pool;
  pool->base = static_cast<uint8_t*>(p);
  pool->num_pages = num_pages;
  pool->page_bytes = page_bytes;
  pool->device = device;
  pool->ipc = true;
  *out = pool;
  return KVX_OK;
}

int kvx_enable_peer_access(int device, int peer) {
  if (device == peer) return KVX_OK;
  int can = 0;
  KVX_CUDA_TRY(cudaDeviceCanAccessPeer(&can, device, peer), "kvx_enable_peer_access: cudaDeviceCanAccessPeer");
  if (!can) return kvx::fail_arg("kvx_enable_peer_access: devices cannot access each other");
  int prev = 0;
  KVX_CUDA_TRY(cudaGetDevice(&prev), "kvx_enable_peer_access: cudaGetDevice");
  KVX_CUDA_TRY(cudaSetDevice(device), "kvx_enable_peer_access: cudaSetDevice");
  cudaError_t e = cudaDeviceEnablePeerAccess(peer, 0);
  cudaSetDevice(prev);
  if (e == cudaErrorPeerAccessAlreadyEnabled) {
    cudaGetLastError();
    e = cudaSuccess;
  }
  if (e != cudaSuccess) return kvx::fail_cuda(e, "kvx_enable_peer_access: cudaDeviceEnablePeerAccess");
  return KVX_OK;
}

}  // extern "C"

extern "C" {

int kvx_stream_create(int device, void** out) {
  if (!out) return kvx::fail_arg("kvx_stream_create: null out");
  int prev = 0;
  KVX_CUDA_TRY(cudaGetDevice(&prev), "kvx_stream_create: cudaGetDevice");
  KVX_CUDA_TRY(cudaSetDevice(device), "kvx_stream_create: cudaSetDevice");
  cudaStream_t s = nullptr;
  const cudaError_t e = cudaStreamCreateWithFlags(&s, cudaStreamNonBlocking);
  cudaSetDevice(prev);
  if (e != cudaSuccess) return kvx::fail_cuda(e, "kvx_stream_create");
  *out = s;
  return KVX_OK;
}

int kvx_stream_destroy(void* stream) {
  if (stream) KVX_CUDA_TRY(cudaStreamDestroy(static_cast<cudaStream_t>(stream)), "kvx_stream_destroy");
  return KVX_OK;
}

int kvx_stream_synchronize(void* stream) {
  KVX_CUDA_TRY(cudaStreamSynchronize(static_cast<cudaStream_t>(stream)), "kvx_stream_synchronize");
  return KVX_OK;
}

int kvx_malloc(int device, uint64_t bytes, void** out) {
  if (!out) return kvx::fail_arg("kvx_malloc: null out");
  int prev = 0;
  KVX_CUDA_TRY(cudaGetDevice(&prev), "kvx_malloc: cudaGetDevice");
  KVX_CUDA_TRY(cudaSetDevice(device), "kvx_malloc: cudaSetDevice");
  const cudaError_t e = cudaMalloc(out, bytes ? bytes : 1);
  cudaSetDevice(prev);
  if (e != cudaSuccess) return kvx::fail_cuda(e, "kvx_malloc");
  return KVX_OK;
}

int kvx_free(void* ptr) {
  if (ptr) KVX_CUDA_TRY(cudaFree(ptr), "kvx_free");
  return KVX_OK;
}

int kvx_memcpy_async(void* dst, const void* src, uint64_t bytes, void* stream) {
  if (bytes == 0) return KVX_OK;
  KVX_CUDA_TRY(cudaMemcpyAsync(dst, src, bytes, cudaMemcpyDefault, static_cast<cudaStream_t>(stream)),
               "kvx_memcpy_async");
  return KVX_OK;
}

int kvx_read_page(const kvx_pool* pool, uint64_t page, void* host_out) {
  if (!pool || !host_out || page >= pool->num_pages) return kvx::fail_arg("kvx_read_page: bad page");
  KVX_CUDA_TRY(cudaMemcpy(host_out, pool->base + page * pool->page_bytes, pool->page_bytes, cudaMemcpyDefault),
               "kvx_read_page");
  return KVX_OK;
}

}  // extern "C"

extern "C" {

int kvx_event_create(void** out) {
  if (!out) return kvx::fail_arg("kvx_event_create: null out");
  cudaEvent_t e = nullptr;
  KVX_CUDA_TRY(cudaEventCreateWithFlags(&e, cudaEventDisableTiming), "kvx_event_create");
  *out = e;
  return KVX_OK;
}

int kvx_event_destroy(void* event) {
  if (event) KVX_CUDA_TRY(cudaEventDestroy(static_cast<cudaEvent_t>(event)), "kvx_event_destroy");
  return KVX_OK;
}

int kvx_event_record(void* event, void* stream) {
  KVX_CUDA_TRY(cudaEventRecord(static_cast<cudaEvent_t>(event), static_cast<cudaStream_t>(stream)), "kvx_event_record");
  return KVX_OK;
}

int kvx_event_synchronize(void* event) {
  KVX_CUDA_TRY(cudaEventSynchronize(static_cast<cudaEvent_t>(event)), "kvx_event_synchronize");
  return KVX_OK;
}

int kvx_event_query(void* event) {
  const cudaError_t e = cudaEventQuery(static_cast<cudaEvent_t>(event));
  if (e == cudaErrorNotReady) return KVX_NOT_READY;
  KVX_CUDA_TRY(e, "kvx_event_query");
  return KVX_OK;
}

int kvx_stream_wait_event(void* stream, void* event) {
  KVX_CUDA_TRY(cudaStreamWaitEvent(static_cast<cudaStream_t>(stream), static_cast<cudaEvent_t>(event), 0),
               "kvx_stream_wait_event");
  return KVX_OK;
}

}  // extern "C"
