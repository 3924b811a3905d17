// Host-only stand-in for libkvx (DIAGNOSTIC, never shipped): every kvx_* the
// store's payload calls, returning success without touching a device, so the
// host bookkeeping of KvStore + NodePayload can be profiled (gprof) on a
// machine with no GPU. Pools carry their sizes only; events are always
// complete. See tools/hostprof/store_path_host.cpp.
#include <cstdlib>
#include <cstring>

#include "kvx.h"

struct kvx_pool {
  uint64_t num_pages, page_bytes;
  int device;
};

extern "C" {
const char* kvx_last_error(void) { return ""; }
uint64_t kvx_page_bytes(const kvx_page_layout* l) {
  return 2ull * l->num_kv_heads * l->block_tokens * l->head_dim * (l->dtype == KVX_DTYPE_BF16 ? 2 : 4);
}
static int make(int dev, uint64_t n, uint64_t pb, kvx_pool** out) {
  *out = new kvx_pool{n, pb, dev};
  return KVX_OK;
}
int kvx_pool_create(int device, uint64_t n, uint64_t pb, kvx_pool** out) { return make(device, n, pb, out); }
int kvx_pool_create_host(uint64_t n, uint64_t pb, kvx_pool** out) { return make(-1, n, pb, out); }
int kvx_pool_create_file(const char*, uint64_t n, uint64_t pb, kvx_pool** out) { return make(-1, n, pb, out); }
int kvx_pool_file_direct(const kvx_pool*) { return -1; }
int kvx_pool_io_error(const kvx_pool*) { return 0; }
int kvx_pool_destroy(kvx_pool* p) {
  delete p;
  return KVX_OK;
}
void* kvx_pool_base(const kvx_pool*) { return nullptr; }
uint64_t kvx_pool_num_pages(const kvx_pool* p) { return p->num_pages; }
int kvx_enable_peer_access(int, int) { return KVX_OK; }
int kvx_stream_create(int, void** out) {
  *out = std::malloc(1);
  return KVX_OK;
}
int kvx_stream_destroy(void* s) {
  std::free(s);
  return KVX_OK;
}
int kvx_stream_synchronize(void*) { return KVX_OK; }
int kvx_malloc(int, uint64_t bytes, void** out) {
  *out = std::malloc(bytes ? bytes : 1);
  return KVX_OK;
}
int kvx_free(void* p) {
  std::free(p);
  return KVX_OK;
}
int kvx_host_alloc(uint64_t bytes, void** out) { return kvx_malloc(0, bytes, out); }
int kvx_host_free(void* p) { return kvx_free(p); }
int kvx_memcpy_async(void*, const void*, uint64_t, void*) { return KVX_OK; }
int kvx_read_page(const kvx_pool*, uint64_t, void*) { return KVX_OK; }
int kvx_event_create(void** out) {
  *out = std::malloc(1);
  return KVX_OK;
}
int kvx_event_destroy(void* e) {
  std::free(e);
  return KVX_OK;
}
int kvx_event_record(void*, void*) { return KVX_OK; }
int kvx_event_synchronize(void*) { return KVX_OK; }
int kvx_event_query(void*) { return KVX_OK; }
int kvx_stream_wait_event(void*, void*) { return KVX_OK; }
int kvx_copy_pages(const kvx_pool*, const uint32_t*, kvx_pool*, const uint32_t*, uint64_t, int, void*) { return KVX_OK; }
int kvx_copy_pages_capped(const kvx_pool*, const uint32_t*, kvx_pool*, const uint32_t*, uint64_t, int, uint32_t,
                          void*) {
  return KVX_OK;
}
int kvx_fill_pages(kvx_pool*, const uint32_t*, const kvx_block_tag*, uint64_t, uint64_t, const kvx_page_layout*, int,
                   void*) {
  return KVX_OK;
}
}
extern "C" int kvx_copy_pages_listed(const kvx_pool*, const uint32_t*, kvx_pool*, const uint32_t*, uint64_t, int,
                                     uint32_t, void*) {
  return KVX_OK;
}
