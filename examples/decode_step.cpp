// A C++ host driving the B200 payload path through the C ABI only
// (include/kvx.h: no CUDA headers, no PyTorch) — the shape of the reference's
// C++ callers (Engine / NodeManager) once the store's pages are real:
//   1. a DEVICE pool of Llama-3.1-8B KV pages and one session of 8K tokens,
//   2. migrate it layer by layer into a second (receiver) pool with K3,
//   3. decode over the received session: per layer, this step's token is
//      appended and attended in ONE launch (kvx_decode_attention_append),
//   4. check against the two-launch path (kvx_append_kv + attention) on a
//      copy of the pool: outputs and pages must match bit for bit.
// Build: make -C examples    Run: examples/decode_step
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <algorithm>
#include <random>
#include <vector>

#include "kvx.h"

#define CK(x)                                                                                  \
  do {                                                                                         \
    if (int rc_ = (x)) {                                                                       \
      std::fprintf(stderr, "%s:%d %s -> %d: %s\n", __FILE__, __LINE__, #x, rc_, kvx_last_error()); \
      std::exit(1);                                                                            \
    }                                                                                          \
  } while (0)

template <typename T>
T* dev_copy(const std::vector<T>& v, void* stream) {
  void* p = nullptr;
  CK(kvx_malloc(0, v.size() * sizeof(T), &p));
  CK(kvx_memcpy_async(p, v.data(), v.size() * sizeof(T), stream));
  return static_cast<T*>(p);
}

int main() {
  const int layers = 32, heads = 8, dim = 128, hq = 32, ctx = 8192, blocks = ctx / 16;
  const kvx_page_layout layout{heads, dim, 16, KVX_DTYPE_BF16};
  const uint64_t pb = kvx_page_bytes(&layout), n = static_cast<uint64_t>(layers) * blocks;
  void* st = nullptr;
  CK(kvx_stream_create(0, &st));
  kvx_pool *src = nullptr, *dst = nullptr, *dst2 = nullptr;
  CK(kvx_pool_create(0, 2 * n, pb, &src));
  CK(kvx_pool_create(0, 2 * n, pb, &dst));
  CK(kvx_pool_create(0, 2 * n, pb, &dst2));

  // the session's pages at a random placement in each pool
  std::mt19937 rng(1);
  std::vector<uint32_t> perm(2 * n);
  for (uint64_t i = 0; i < 2 * n; ++i) perm[i] = static_cast<uint32_t>(i);
  std::shuffle(perm.begin(), perm.end(), rng);
  std::vector<uint32_t> s_ids(perm.begin(), perm.begin() + n), d_ids(perm.begin() + n, perm.end());
  std::vector<kvx_block_tag> tags(n);
  for (uint64_t i = 0; i < n; ++i) tags[i] = kvx_block_tag{7, static_cast<uint32_t>(i / blocks), static_cast<uint32_t>(i % blocks)};
  uint32_t* ds = dev_copy(s_ids, st);
  uint32_t* dd = dev_copy(d_ids, st);
  kvx_block_tag* dt = dev_copy(tags, st);
  CK(kvx_fill_pages(src, ds, dt, n, 42, &layout, KVX_FILL_VALUES, st));

  // migrate layer by layer (the reference's per-layer NetArrive) into both receivers
  for (int l = 0; l < layers; ++l) {
    CK(kvx_copy_pages(src, ds + l * blocks, dst, dd + l * blocks, blocks, KVX_COPY_AUTO, st));
    CK(kvx_copy_pages(src, ds + l * blocks, dst2, dd + l * blocks, blocks, KVX_COPY_AUTO, st));
  }

  // one decode step over the received session, batch 1
  std::vector<uint16_t> q(hq * dim), kv(heads * dim);
  for (auto& x : q) x = static_cast<uint16_t>(0x3C00 | (rng() & 0x7F));
  for (auto& x : kv) x = static_cast<uint16_t>(0x3A00 | (rng() & 0xFF));
  std::vector<int32_t> lens{ctx}, slot{(ctx - 1) % 16};
  uint16_t* dq = dev_copy(q, st);
  uint16_t* dk = dev_copy(kv, st);
  int32_t* dl = dev_copy(lens, st);
  int32_t* dsl = dev_copy(slot, st);
  kvx_attn_params prm{hq, blocks, 0, 0.f, KVX_MERGE_AUTO, KVX_ATTN_EARLY_PREFETCH};
  const uint64_t ws_bytes = kvx_decode_attention_workspace(&layout, &prm, 1, ctx);
  void *ws = nullptr, *out_a = nullptr, *out_b = nullptr;
  CK(kvx_malloc(0, ws_bytes ? ws_bytes : 16, &ws));
  CK(kvx_malloc(0, static_cast<uint64_t>(layers) * hq * dim * 4, &out_a));
  CK(kvx_malloc(0, static_cast<uint64_t>(layers) * hq * dim * 4, &out_b));
  std::vector<uint8_t> zeros(ws_bytes ? ws_bytes : 16, 0);
  CK(kvx_memcpy_async(ws, zeros.data(), zeros.size(), st));
  for (int l = 0; l < layers; ++l) {
    float* oa = static_cast<float*>(out_a) + static_cast<uint64_t>(l) * hq * dim;
    float* ob = static_cast<float*>(out_b) + static_cast<uint64_t>(l) * hq * dim;
    CK(kvx_decode_attention_append(dst, &layout, &prm, dd + l * blocks, dl, dq, dk, dk, oa, 1, ctx, ws, ws_bytes, st));
    CK(kvx_append_kv(dst2, &layout, dd + l * blocks + (blocks - 1), dsl, dk, dk, 1, st));
    CK(kvx_decode_attention(dst2, &layout, &prm, dd + l * blocks, dl, dq, ob, 1, ctx, ws, ws_bytes, st));
  }
  std::vector<float> a(static_cast<size_t>(layers) * hq * dim), b(a.size());
  CK(kvx_memcpy_async(a.data(), out_a, a.size() * 4, st));
  CK(kvx_memcpy_async(b.data(), out_b, b.size() * 4, st));
  CK(kvx_stream_synchronize(st));
  std::vector<uint8_t> pa(pb), pbuf(pb);
  bool pages_ok = true;
  for (int l = 0; l < layers; ++l) {
    const uint32_t last = d_ids[static_cast<uint64_t>(l) * blocks + blocks - 1];
    CK(kvx_read_page(dst, last, pa.data()));
    CK(kvx_read_page(dst2, last, pbuf.data()));
    pages_ok = pages_ok && std::memcmp(pa.data(), pbuf.data(), pb) == 0;
  }
  const bool out_ok = std::memcmp(a.data(), b.data(), a.size() * 4) == 0;
  double mean = 0;
  for (float x : a) mean += x;
  std::printf("decode_step: %d layers x %d tokens migrated and decoded; fused == two-launch outputs: %s, "
              "appended pages: %s; mean output %.5f\n",
              layers, ctx, out_ok ? "bit-identical" : "DIFFER", pages_ok ? "identical" : "DIFFER", mean / a.size());
  for (void* p : {static_cast<void*>(ds), static_cast<void*>(dd), static_cast<void*>(dt), static_cast<void*>(dq),
                  static_cast<void*>(dk), static_cast<void*>(dl), static_cast<void*>(dsl), ws, out_a, out_b})
    kvx_free(p);
  kvx_pool_destroy(src);
  kvx_pool_destroy(dst);
  kvx_pool_destroy(dst2);
  kvx_stream_destroy(st);
  return out_ok && pages_ok ? 0 : 1;
}
