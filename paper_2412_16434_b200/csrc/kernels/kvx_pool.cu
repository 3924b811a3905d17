// Page pools and the error channel of the kvx C ABI (include/kvx.h).
//
// A pool is a flat array of equal-size pages. A DEVICE pool is one cudaMalloc
// in HBM; a HOST pool is pinned, device-mapped host memory (the HOST tier's
// physical backing, reachable by kernels over PCIe); a pool can also wrap
// caller memory or a peer GPU's pool opened through CUDA IPC, which is how a
// migration kernel on the source GPU stores straight into the receiver's
// pages over NVLink (SURVEY.md §5 "Distributed communication backend").

#include <fcntl.h>
#include <sys/stat.h>
#include <unistd.h>

#include <cerrno>
#include <cstdlib>
#include <cstdio>
#include <cstring>
#include <mutex>
#include <string>
#include <thread>
#include <vector>

#include <unordered_map>
#include "kvx_common.cuh"

namespace kvx {

namespace {
thread_local std::string g_error;
}

void set_error(const std::string& msg) { g_error = msg; }

namespace {
std::atomic<uint64_t> g_launches{0}, g_library_launches{0};
}
void note_launch(uint64_t n) { g_launches.fetch_add(n, std::memory_order_relaxed); }
void note_library_launch(uint64_t n) { g_library_launches.fetch_add(n, std::memory_order_relaxed); }

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

int check_io(const kvx_pool* pool, const char* who) {
  if (!pool || pool->fd < 0) return KVX_OK;
  const int e = pool->io_errno.load();
  if (e == 0) return KVX_OK;
  g_error = std::string(who) + ": disk-tier file I/O failed earlier: " + std::strerror(e);
  return KVX_ERR_IO;
}

namespace {

constexpr uint64_t kIoThreads = 8;  // concurrent preads / pwrites per large job

struct FileJob {
  kvx_pool* pool;
  std::vector<FileRun> runs;
  bool write;
};

// Whole-run pread/pwrite with retry on short transfers; the first failure is
// recorded on the pool (sticky) and later runs are skipped.
void do_run(kvx_pool* p, const FileRun& r, bool write) {
  uint64_t done = 0;
  while (done < r.bytes && p->io_errno.load() == 0) {
    const ssize_t n = write ? ::pwrite(p->fd, r.host + done, r.bytes - done, static_cast<off_t>(r.offset + done))
                            : ::pread(p->fd, r.host + done, r.bytes - done, static_cast<off_t>(r.offset + done));
    if (n < 0 && errno == EINTR) continue;
    if (n <= 0) {
      int expected = 0;
      p->io_errno.compare_exchange_strong(expected, n < 0 ? errno : EIO);
      return;
    }
    done += static_cast<uint64_t>(n);
  }
}

// Big jobs fan out over a few threads (queue depth for the SSD); the
// callback returns — and the stream proceeds — only when all runs are done.
void run_file_job(void* arg) {
  FileJob* job = static_cast<FileJob*>(arg);
  kvx_pool* p = job->pool;
  uint64_t total = 0;
  for (const FileRun& r : job->runs) total += r.bytes;
  const int threads = static_cast<int>(std::min<uint64_t>(kIoThreads, std::max<uint64_t>(1, total >> 22)));
  if (threads <= 1 || job->runs.size() < 2) {
    for (const FileRun& r : job->runs) do_run(p, r, job->write);
  } else {
    std::atomic<size_t> next{0};
    auto worker = [&] {
      for (size_t i = next++; i < job->runs.size(); i = next++) do_run(p, job->runs[i], job->write);
    };
    std::vector<std::thread> pool;
    for (int t = 1; t < threads; ++t) pool.emplace_back(worker);
    worker();
    for (auto& t : pool) t.join();
  }
  delete job;
}

}  // namespace

// The I/O runs as a host callback in stream order: after everything queued
// before it on `stream` (e.g. the copy that filled the host pages it writes),
// before everything queued after it (e.g. the copy that reads what it loaded).
int enqueue_file_io(kvx_pool* file, std::vector<FileRun> runs, bool write, cudaStream_t stream, const char* who) {
  if (int rc = check_io(file, who)) return rc;
  if (runs.empty()) return KVX_OK;
  auto* job = new FileJob{file, std::move(runs), write};
  const cudaError_t e = cudaLaunchHostFunc(stream, run_file_job, job);
  if (e != cudaSuccess) {
    delete job;
    return fail_cuda(e, who);
  }
  return KVX_OK;
}

}  // namespace kvx

extern "C" {

const char* kvx_last_error(void) { return kvx::g_error.c_str(); }

int kvx_version(void) { return 1; }

uint64_t kvx_launch_count(void) { return kvx::g_launches.load(std::memory_order_relaxed); }
uint64_t kvx_library_launch_count(void) { return kvx::g_library_launches.load(std::memory_order_relaxed); }

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

int kvx_pool_create_file(const char* path, uint64_t num_pages, uint64_t page_bytes, kvx_pool** out) {
  if (!out || !path || num_pages == 0 || page_bytes == 0 || page_bytes % 4096 != 0)
    return kvx::fail_arg("kvx_pool_create_file: need a path, num_pages > 0 and page_bytes a multiple of 4096");
  bool direct = true;
  int fd = ::open(path, O_RDWR | O_CREAT | O_DIRECT, 0600);
  if (fd < 0 && errno == EINVAL) {  // filesystem without O_DIRECT (e.g. tmpfs): buffered I/O
    direct = false;
    fd = ::open(path, O_RDWR | O_CREAT, 0600);
  }
  if (fd < 0) {
    kvx::set_error(std::string("kvx_pool_create_file: open ") + path + ": " + std::strerror(errno));
    return KVX_ERR_IO;
  }
  const uint64_t bytes = num_pages * page_bytes;
  struct stat st {};
  if (::fstat(fd, &st) != 0 || (static_cast<uint64_t>(st.st_size) < bytes && ::ftruncate(fd, static_cast<off_t>(bytes)) != 0)) {
    kvx::set_error(std::string("kvx_pool_create_file: size ") + path + ": " + std::strerror(errno));
    ::close(fd);
    return KVX_ERR_IO;
  }
  auto* pool = new kvx_pool;
  pool->num_pages = num_pages;
  pool->page_bytes = page_bytes;
  pool->device = -1;
  pool->host = true;
  pool->fd = fd;
  pool->direct = direct;
  *out = pool;
  return KVX_OK;
}

int kvx_pool_file_direct(const kvx_pool* pool) { return pool && pool->fd >= 0 ? (pool->direct ? 1 : 0) : -1; }

int kvx_pool_io_error(const kvx_pool* pool) {
  if (!pool || pool->fd < 0) return 0;
  return pool->io_errno.load();
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
  if (pool->fd >= 0) ::close(pool->fd);
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

int kvx_host_alloc(uint64_t bytes, void** out) {
  if (!out) return kvx::fail_arg("kvx_host_alloc: null out");
  KVX_CUDA_TRY(cudaHostAlloc(out, bytes ? bytes : 1, cudaHostAllocPortable), "kvx_host_alloc");
  return KVX_OK;
}

int kvx_host_free(void* ptr) {
  if (ptr) KVX_CUDA_TRY(cudaFreeHost(ptr), "kvx_host_free");
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
  if (pool->fd >= 0) {  // file pool: aligned bounce for O_DIRECT, then copy out
    if (int rc = kvx::check_io(pool, "kvx_read_page")) return rc;
    void* bounce = nullptr;
    if (posix_memalign(&bounce, 4096, pool->page_bytes) != 0) return kvx::fail_arg("kvx_read_page: out of memory");
    uint64_t done = 0;
    while (done < pool->page_bytes) {
      const ssize_t n = ::pread(pool->fd, static_cast<uint8_t*>(bounce) + done, pool->page_bytes - done,
                                static_cast<off_t>(page * pool->page_bytes + done));
      if (n < 0 && errno == EINTR) continue;
      if (n <= 0) {
        free(bounce);
        kvx::set_error(std::string("kvx_read_page: pread: ") + std::strerror(n < 0 ? errno : EIO));
        return KVX_ERR_IO;
      }
      done += static_cast<uint64_t>(n);
    }
    std::memcpy(host_out, bounce, pool->page_bytes);
    free(bounce);
    return KVX_OK;
  }
  KVX_CUDA_TRY(cudaMemcpy(host_out, pool->base + page * pool->page_bytes, pool->page_bytes, cudaMemcpyDefault),
               "kvx_read_page");
  return KVX_OK;
}

}  // extern "C"

extern "C" {

// Ordering events are recycled: the payload records two per moved layer
// (batch + transfer), and cudaEventCreate/Destroy cost microseconds each on
// the host path a migration runs on. A destroyed event goes back to its
// device's free list; re-recording it later is safe (a stream wait binds the
// record current when the wait is enqueued). Timing events are not pooled.
namespace kvx {
namespace {
std::mutex g_event_mu;
std::unordered_map<cudaEvent_t, int> g_event_device;  // pooled-kind events alive or free -> device
std::vector<cudaEvent_t> g_event_free[64];
}  // namespace
}  // namespace kvx

int kvx_event_create(void** out) {
  if (!out) return kvx::fail_arg("kvx_event_create: null out");
  int dev = 0;
  KVX_CUDA_TRY(cudaGetDevice(&dev), "kvx_event_create");
  {
    std::lock_guard<std::mutex> lock(kvx::g_event_mu);
    auto& fl = kvx::g_event_free[dev % 64];
    if (!fl.empty()) {
      *out = fl.back();
      fl.pop_back();
      return KVX_OK;
    }
  }
  cudaEvent_t e = nullptr;
  KVX_CUDA_TRY(cudaEventCreateWithFlags(&e, cudaEventDisableTiming), "kvx_event_create");
  {
    std::lock_guard<std::mutex> lock(kvx::g_event_mu);
    kvx::g_event_device[e] = dev;
  }
  *out = e;
  return KVX_OK;
}

int kvx_timer_create(void** out) {
  if (!out) return kvx::fail_arg("kvx_timer_create: null out");
  cudaEvent_t e = nullptr;
  KVX_CUDA_TRY(cudaEventCreate(&e), "kvx_timer_create");
  *out = e;
  return KVX_OK;
}

int kvx_timer_elapsed_ms(void* start, void* stop, float* ms) {
  if (!start || !stop || !ms) return kvx::fail_arg("kvx_timer_elapsed_ms: null argument");
  KVX_CUDA_TRY(cudaEventElapsedTime(ms, static_cast<cudaEvent_t>(start), static_cast<cudaEvent_t>(stop)),
               "kvx_timer_elapsed_ms");
  return KVX_OK;
}

int kvx_event_destroy(void* event) {
  if (!event) return KVX_OK;
  const auto e = static_cast<cudaEvent_t>(event);
  {
    std::lock_guard<std::mutex> lock(kvx::g_event_mu);
    const auto it = kvx::g_event_device.find(e);
    if (it != kvx::g_event_device.end()) {  // an ordering event: back to its device's free list
      kvx::g_event_free[it->second % 64].push_back(e);
      return KVX_OK;
    }
  }
  KVX_CUDA_TRY(cudaEventDestroy(e), "kvx_event_destroy");
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

namespace {
// Stream memory operations are driver-API entry points; they are resolved
// through the runtime (cudaGetDriverEntryPoint) so libkvx.so does not link
// libcuda directly and still loads on a machine without a GPU driver (the
// CPU test suite checks its exports there).
using WriteValue32 = CUresult (*)(CUstream, CUdeviceptr, cuuint32_t, unsigned int);
using WaitValue32 = CUresult (*)(CUstream, CUdeviceptr, cuuint32_t, unsigned int);

template <typename Fn>
int driver_fn(const char* name, Fn* out) {
  static std::mutex mu;
  std::lock_guard<std::mutex> lock(mu);
  void* fn = nullptr;
  cudaDriverEntryPointQueryResult q{};
  const cudaError_t e = cudaGetDriverEntryPoint(name, &fn, cudaEnableDefault, &q);
  if (e != cudaSuccess) return kvx::fail_cuda(e, name);
  if (q != cudaDriverEntryPointSuccess || !fn) {
    kvx::set_error(std::string(name) + ": driver entry point unavailable");
    return KVX_ERR_CUDA;
  }
  *out = reinterpret_cast<Fn>(fn);
  return KVX_OK;
}

int fail_cu(CUresult r, const char* what) {
  kvx::set_error(std::string(what) + ": CUDA driver error " + std::to_string(static_cast<int>(r)));
  return KVX_ERR_CUDA;
}
}  // namespace

extern "C" {

int kvx_signal_write(void* d_flag, uint32_t value, void* stream) {
  if (!d_flag || reinterpret_cast<uintptr_t>(d_flag) % 4) return kvx::fail_arg("kvx_signal_write: need a 4-B aligned flag");
  static WriteValue32 write_value = nullptr;
  if (!write_value)
    if (int rc = driver_fn("cuStreamWriteValue32", &write_value)) return rc;
  // Default flags: a memory barrier orders every prior write of the stream
  // (e.g. the K3 stores into a peer's pages) before the flag becomes visible.
  const CUresult r = write_value(static_cast<CUstream>(stream), reinterpret_cast<CUdeviceptr>(d_flag), value,
                                 CU_STREAM_WRITE_VALUE_DEFAULT);
  return r == CUDA_SUCCESS ? KVX_OK : fail_cu(r, "kvx_signal_write");
}

int kvx_signal_flush_supported(void* stream) {
  // Cached per device: 0 unknown, 1 no, 2 yes.
  static std::atomic<int> flush_cap[64] = {};
  int dev = 0;
  const cudaError_t e = cudaStreamGetDevice(static_cast<cudaStream_t>(stream), &dev);
  if (e != cudaSuccess) {
    kvx::fail_cuda(e, "kvx_signal_flush_supported: cudaStreamGetDevice");
    return -1;
  }
  std::atomic<int>& cap = flush_cap[(dev < 0 ? 0 : dev) % 64];
  int c = cap.load(std::memory_order_relaxed);
  if (c == 0) {
    int v = 0;
    const cudaError_t e2 = cudaDeviceGetAttribute(&v, cudaDevAttrCanFlushRemoteWrites, dev);
    if (e2 != cudaSuccess) {
      kvx::fail_cuda(e2, "kvx_signal_flush_supported: cudaDevAttrCanFlushRemoteWrites");
      return -1;
    }
    c = v ? 2 : 1;
    cap.store(c, std::memory_order_relaxed);
  }
  return c == 2 ? 1 : 0;
}

int kvx_signal_wait(const void* d_flag, uint32_t value, void* stream) {
  if (!d_flag || reinterpret_cast<uintptr_t>(d_flag) % 4) return kvx::fail_arg("kvx_signal_wait: need a 4-B aligned flag");
  static WaitValue32 wait_value = nullptr;
  if (!wait_value)
    if (int rc = driver_fn("cuStreamWaitValue32", &wait_value)) return rc;
  // The wait runs on the stream's device: FLUSH (outstanding remote writes,
  // e.g. the peer's K3 stores that preceded the flag, become visible to the
  // stream's later work) is requested when THAT device supports it. When it
  // does not, the writer's system-scope barrier (kvx_signal_write) is the
  // only ordering; kvx_signal_flush_supported() lets callers report such a
  // gate as unverified or use an event / host handoff instead.
  const int can_flush = kvx_signal_flush_supported(stream);
  if (can_flush < 0) return KVX_ERR_CUDA;
  const unsigned flags = CU_STREAM_WAIT_VALUE_GEQ | (can_flush ? static_cast<unsigned>(CU_STREAM_WAIT_VALUE_FLUSH) : 0u);
  const CUresult r = wait_value(static_cast<CUstream>(stream), reinterpret_cast<CUdeviceptr>(d_flag), value, flags);
  return r == CUDA_SUCCESS ? KVX_OK : fail_cu(r, "kvx_signal_wait");
}

}  // extern "C"
