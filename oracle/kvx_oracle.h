/* kvx_oracle.h — CPU restatement of the KV payload path. TEST INFRASTRUCTURE.
 *
 * Only tests/, __graft_entry__.smoke() and bench.py's CPU-baseline/reference
 * arm may load this; the product never links it (there is no CPU fallback).
 *
 * Parity status:
 *  - page fill / pack / unpack / page copy / append: bit-exact restatement.
 *    The reference moves no bytes; what a page IS comes from
 *    its accounting unit, layer_block_bytes = kv_bytes_per_layer(block_tokens)
 *    (/root/reference/proj/src/kvstore.cpp:67, costmodel.cpp:48-52), and which
 *    pages move where is pinned by the block-table state the reference itself
 *    computes (oracle/_ref, tests/test_state_parity.py). A page move is a
 *    permutation of bytes, so bit-exactness is well defined.
 *  - paged decode attention: PARITY UNPINNED by the reference (it only models
 *    the decode step, costmodel.cpp:59-80). Restated as textbook softmax
 *    attention in fp64 over the same bf16/fp32 inputs; GPU results are held
 *    to the tolerance stated in tests/test_kvx_gpu.py.
 */
#ifndef KVX_ORACLE_H_
#define KVX_ORACLE_H_

#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

typedef struct {
  int32_t num_kv_heads;
  int32_t head_dim;
  int32_t block_tokens;
  int32_t dtype; /* 0 = f32, 1 = bf16 (same codes as kvx.h) */
} kvxo_layout;

typedef struct {
  uint32_t session, layer, block;
} kvxo_tag;

uint64_t kvxo_splitmix64(uint64_t x);
uint64_t kvxo_page_bytes(const kvxo_layout* l);
int kvxo_threads(void);

/* mode 0: splitmix64 words; mode 1: dtype values on [-sqrt3, sqrt3). */
void kvxo_fill_pages(uint8_t* pool, uint64_t page_bytes, const uint32_t* ids, const kvxo_tag* tags, uint64_t n,
                     uint64_t seed, const kvxo_layout* layout, int mode);
void kvxo_pack(const uint8_t* pool, uint64_t page_bytes, const uint32_t* ids, uint64_t n, uint8_t* dst, int threads);
void kvxo_unpack(uint8_t* pool, uint64_t page_bytes, const uint32_t* ids, uint64_t n, const uint8_t* src,
                 int threads);
void kvxo_copy_pages(const uint8_t* src_pool, const uint32_t* src_ids, uint8_t* dst_pool, const uint32_t* dst_ids,
                     uint64_t n, uint64_t page_bytes, int threads);
void kvxo_append_kv(uint8_t* pool, const kvxo_layout* l, const uint32_t* ids, const int32_t* slots, const void* k,
                    const void* v, uint64_t n);
/* out[b][hq][d] in fp64. */
void kvxo_decode_attention(const uint8_t* pool, const kvxo_layout* l, int32_t num_q_heads, const uint32_t* tables,
                           int32_t max_blocks, const int32_t* ctx_lens, const void* q, double* out, int32_t batch,
                           float scale, int threads);

#ifdef __cplusplus
}
#endif

#endif /* KVX_ORACLE_H_ */
