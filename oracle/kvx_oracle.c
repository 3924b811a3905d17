/* kvx_oracle.c — CPU restatement of the KV payload path. TEST INFRASTRUCTURE
 * (see kvx_oracle.h for scope and parity status). Plain C11 + OpenMP.
 *
 * Reference anchors for what each function restates:
 *   kvxo_fill_pages   a page is one BlockKey's per-layer slice:
 *                     kvstore.hpp:24-28 (BlockKey), kvstore.cpp:67 (its size)
 *   kvxo_pack         SwapOut/HostCopy source side, kvstore.cpp:230-269,
 *                     691-706; migration send side, kvstore.cpp:753-769
 *   kvxo_unpack       LoadH2D landing, kvstore.cpp:522-533, 599-611;
 *                     NetArrive landing, kvstore.cpp:914-923
 *   kvxo_copy_pages   one migrated layer, page to page (import_migration's
 *                     per-layer NetArrive, kvstore.cpp:753-769)
 *   kvxo_append_kv    the bytes of append_blocks' new token, kvstore.cpp:202-271
 *   kvxo_decode_attention  the decode step the reference models in
 *                     decode_step_time, costmodel.cpp:59-80 (parity unpinned)
 */
#include "kvx_oracle.h"

#include <math.h>
#include <stdlib.h>
#include <string.h>
#ifdef _OPENMP
#include <omp.h>
#endif

uint64_t kvxo_splitmix64(uint64_t x) {
  x += 0x9E3779B97F4A7C15ull;
  uint64_t z = x;
  z = (z ^ (z >> 30)) * 0xBF58476D1CE4E5B9ull;
  z = (z ^ (z >> 27)) * 0x94D049BB133111EBull;
  return z ^ (z >> 31);
}

static uint64_t block_base(uint64_t seed, const kvxo_tag* t) {
  uint64_t h = kvxo_splitmix64(seed);
  h = kvxo_splitmix64(h ^ t->session);
  h = kvxo_splitmix64(h ^ t->layer);
  return kvxo_splitmix64(h ^ t->block);
}

static float unit_value(uint64_t r) {
  const int32_t u = (int32_t)(r >> 40) - 8388608;
  volatile float x = (float)u * (1.0f / 8388608.0f); /* exact */
  return x * 1.7320508f;                              /* one IEEE multiply */
}

static uint16_t f32_to_bf16_rne(float f) {
  uint32_t bits;
  memcpy(&bits, &f, 4);
  return (uint16_t)((bits + 0x7FFFu + ((bits >> 16) & 1u)) >> 16);
}

static double bf16_to_f64(uint16_t h) {
  const uint32_t bits = (uint32_t)h << 16;
  float f;
  memcpy(&f, &bits, 4);
  return (double)f;
}

uint64_t kvxo_page_bytes(const kvxo_layout* l) {
  return 2ull * (uint64_t)l->num_kv_heads * (uint64_t)l->block_tokens * (uint64_t)l->head_dim *
         (l->dtype == 1 ? 2u : 4u);
}

int kvxo_threads(void) {
#ifdef _OPENMP
  return omp_get_max_threads();
#else
  return 1;
#endif
}

void kvxo_fill_pages(uint8_t* pool, uint64_t page_bytes, const uint32_t* ids, const kvxo_tag* tags, uint64_t n,
                     uint64_t seed, const kvxo_layout* layout, int mode) {
  const int dtype = layout ? layout->dtype : 1;
#pragma omp parallel for schedule(static)
  for (int64_t i = 0; i < (int64_t)n; ++i) {
    const uint64_t h = block_base(seed, &tags[i]);
    uint8_t* page = pool + (uint64_t)ids[i] * page_bytes;
    if (mode == 0) {
      for (uint64_t w = 0; w < page_bytes / 8; ++w) {
        const uint64_t x = kvxo_splitmix64(h + w);
        memcpy(page + 8 * w, &x, 8);
      }
    } else if (dtype == 0) {
      for (uint64_t e = 0; e < page_bytes / 4; ++e) {
        const float f = unit_value(kvxo_splitmix64(h + e));
        memcpy(page + 4 * e, &f, 4);
      }
    } else {
      for (uint64_t e = 0; e < page_bytes / 2; ++e) {
        const uint16_t b = f32_to_bf16_rne(unit_value(kvxo_splitmix64(h + e)));
        memcpy(page + 2 * e, &b, 2);
      }
    }
  }
}

void kvxo_pack(const uint8_t* pool, uint64_t page_bytes, const uint32_t* ids, uint64_t n, uint8_t* dst, int threads) {
#pragma omp parallel for schedule(static) num_threads(threads > 0 ? threads : kvxo_threads())
  for (int64_t i = 0; i < (int64_t)n; ++i) memcpy(dst + (uint64_t)i * page_bytes, pool + (uint64_t)ids[i] * page_bytes, page_bytes);
}

void kvxo_unpack(uint8_t* pool, uint64_t page_bytes, const uint32_t* ids, uint64_t n, const uint8_t* src,
                 int threads) {
#pragma omp parallel for schedule(static) num_threads(threads > 0 ? threads : kvxo_threads())
  for (int64_t i = 0; i < (int64_t)n; ++i) memcpy(pool + (uint64_t)ids[i] * page_bytes, src + (uint64_t)i * page_bytes, page_bytes);
}

void kvxo_copy_pages(const uint8_t* src_pool, const uint32_t* src_ids, uint8_t* dst_pool, const uint32_t* dst_ids,
                     uint64_t n, uint64_t page_bytes, int threads) {
#pragma omp parallel for schedule(static) num_threads(threads > 0 ? threads : kvxo_threads())
  for (int64_t i = 0; i < (int64_t)n; ++i)
    memcpy(dst_pool + (uint64_t)dst_ids[i] * page_bytes, src_pool + (uint64_t)src_ids[i] * page_bytes, page_bytes);
}

void kvxo_append_kv(uint8_t* pool, const kvxo_layout* l, const uint32_t* ids, const int32_t* slots, const void* k,
                    const void* v, uint64_t n) {
  const uint64_t pb = kvxo_page_bytes(l);
  const uint64_t row = (uint64_t)l->head_dim * (l->dtype == 1 ? 2u : 4u);
  const int H = l->num_kv_heads, T = l->block_tokens;
  for (uint64_t i = 0; i < n; ++i) {
    uint8_t* page = pool + (uint64_t)ids[i] * pb;
    for (int kv = 0; kv < 2; ++kv)
      for (int h = 0; h < H; ++h) {
        const uint8_t* src = (const uint8_t*)(kv ? v : k) + (i * H + h) * row;
        memcpy(page + ((uint64_t)(kv * H + h) * T + slots[i]) * row, src, row);
      }
  }
}

static double load_elt(const uint8_t* p, int dtype) {
  if (dtype == 1) {
    uint16_t h;
    memcpy(&h, p, 2);
    return bf16_to_f64(h);
  }
  float f;
  memcpy(&f, p, 4);
  return (double)f;
}

void kvxo_decode_attention(const uint8_t* pool, const kvxo_layout* l, int32_t num_q_heads, const uint32_t* tables,
                           int32_t max_blocks, const int32_t* ctx_lens, const void* q, double* out, int32_t batch,
                           float scale, int threads) {
  const int H = l->num_kv_heads, D = l->head_dim, T = l->block_tokens;
  const int g = num_q_heads / H;
  const uint64_t elt = l->dtype == 1 ? 2 : 4;
  const uint64_t pb = kvxo_page_bytes(l);
  const double sc = (double)scale;
#pragma omp parallel for collapse(2) schedule(dynamic) num_threads(threads > 0 ? threads : kvxo_threads())
  for (int b = 0; b < batch; ++b)
    for (int hq = 0; hq < num_q_heads; ++hq) {
      const int h = hq / g, ctx = ctx_lens[b];
      double qd[512];
      const uint8_t* qrow = (const uint8_t*)q + ((uint64_t)b * num_q_heads + hq) * D * elt;
      for (int d = 0; d < D; ++d) qd[d] = load_elt(qrow + d * elt, l->dtype);
      double* o = out + ((uint64_t)b * num_q_heads + hq) * D;
      double* logits = (double*)malloc(sizeof(double) * (size_t)(ctx > 0 ? ctx : 1));
      double mx = -INFINITY;
      for (int t = 0; t < ctx; ++t) {
        const uint8_t* page = pool + (uint64_t)tables[(uint64_t)b * max_blocks + t / T] * pb;
        const uint8_t* krow = page + ((uint64_t)h * T + (t % T)) * D * elt;
        double dot = 0.0;
        for (int d = 0; d < D; ++d) dot += qd[d] * load_elt(krow + d * elt, l->dtype);
        logits[t] = dot * sc;
        if (logits[t] > mx) mx = logits[t];
      }
      double denom = 0.0;
      for (int d = 0; d < D; ++d) o[d] = 0.0;
      for (int t = 0; t < ctx; ++t) {
        const double p = exp(logits[t] - mx);
        denom += p;
        const uint8_t* page = pool + (uint64_t)tables[(uint64_t)b * max_blocks + t / T] * pb;
        const uint8_t* vrow = page + ((uint64_t)(H + h) * T + (t % T)) * D * elt;
        for (int d = 0; d < D; ++d) o[d] += p * load_elt(vrow + d * elt, l->dtype);
      }
      for (int d = 0; d < D; ++d) o[d] = denom > 0.0 ? o[d] / denom : 0.0;
      free(logits);
    }
}
