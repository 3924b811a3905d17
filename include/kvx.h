/* kvx.h — C ABI of the B200 KV payload path (sm_100a kernels).
 *
 * The reference stores no KV bytes ("bytes are accounted,
 * not stored"); its per-(session, layer, block) accounting unit is
 * layer_block_bytes = kv_bytes_per_layer(block_tokens)
 * (/root/reference/proj/src/kvstore.cpp:67, costmodel.cpp:48-52). This ABI
 * gives each such block a physical PAGE of exactly that many bytes and moves
 * pages with hand-written kernels. Each entry point replaces a modelled
 * transfer of the reference:
 *
 *   kvx_pack        K1  DEVICE pages -> contiguous buffer (one layer's block
 *                       range): the D2H side of HostCopy/SwapOut
 *                       (kvstore.cpp:230-269, 691-706) and the send side of a
 *                       migration (import_migration, kvstore.cpp:753-769)
 *   kvx_unpack      K2  contiguous -> DEVICE pages: LoadH2D landing of
 *                       plan_layerwise_load/promote (kvstore.cpp:522-533,
 *                       599-611) and NetArrive landing (kvstore.cpp:914-923)
 *   kvx_copy_pages  K3  page -> page between any two pools (local HBM, a peer
 *                       GPU's pool over NVLink, mapped pinned host memory):
 *                       the fused pack+send+unpack of one migration layer
 *   kvx_fill_pages  K5  deterministic synthetic page contents (tests/bench)
 *   kvx_append_kv   K5  write one token's K/V into its page slot
 *                       (the bytes behind append_blocks, kvstore.cpp:202-271)
 *   kvx_decode_attention  K4  paged decode attention over block tables;
 *                       replaces the modelled decode step
 *                       (costmodel.cpp:59-80, engine.cpp:256-257)
 *
 * Conventions: plain pointers and sizes, no torch types; every call returns
 * KVX_OK (0) or a KVX_ERR_* code, message in kvx_last_error() (thread
 * local); kernels are launched asynchronously on the caller's stream
 * (`stream` is a cudaStream_t passed as void*, NULL = legacy default stream).
 * There is no CPU fallback: without a CUDA device every launching call fails
 * with KVX_ERR_CUDA.
 *
 * Page layout (for fill/append/attention; pack/unpack/copy treat pages as
 * opaque bytes): page = [2 (K, V)][num_kv_heads][block_tokens][head_dim]
 * elements of `dtype`, so one kv head's K (or V) for the page's tokens is one
 * contiguous block_tokens*head_dim run.
 */
#ifndef KVX_H_
#define KVX_H_

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define KVX_OK 0
#define KVX_ERR_CUDA 1        /* CUDA runtime/driver error or no device */
#define KVX_ERR_ARG 2         /* invalid argument                       */
#define KVX_ERR_UNSUPPORTED 3 /* shape/dtype/mode not implemented       */
#define KVX_ERR_IO 5          /* file-pool read/write failed (sticky)   */

#define KVX_DTYPE_F32 0
#define KVX_DTYPE_BF16 1

#define KVX_FILL_BITS 0   /* page = splitmix64 words                       */
#define KVX_FILL_VALUES 1 /* page = dtype values uniform on [-sqrt3,sqrt3) */

#define KVX_COPY_AUTO 0   /* TMA for local HBM<->HBM, SM for peer/host pools */
#define KVX_COPY_SM 1     /* SM kernel, 16-B vector loads/stores             */
#define KVX_COPY_TMA 2    /* SM kernel, cp.async.bulk (TMA) through smem     */
#define KVX_COPY_CE 3     /* copy engines (one memcpy per id run); host ids  */

typedef struct kvx_pool kvx_pool;

typedef struct {
  int32_t num_kv_heads;
  int32_t head_dim;
  int32_t block_tokens;
  int32_t dtype; /* KVX_DTYPE_* */
} kvx_page_layout;

typedef struct {
  uint32_t session;
  uint32_t layer;
  uint32_t block;
} kvx_block_tag; /* logical BlockKey a page holds (kvstore.hpp:24-28) */

typedef struct {
  int32_t num_q_heads; /* multiple of num_kv_heads (GQA group g = Hq / H) */
  int32_t max_blocks;  /* row stride of the block table                  */
  int32_t num_splits;  /* split-K over context; 0 = auto                  */
  float scale;         /* softmax scale; 0 = 1/sqrt(head_dim)             */
  int32_t split_merge; /* KVX_MERGE_*: how split-K partials are combined  */
  int32_t flags;       /* KVX_ATTN_* bits                                  */
} kvx_attn_params;

/* The caller guarantees that, in the stream, the kernel launched just before
 * this one writes neither the block tables, nor ctx_lens, nor any page other
 * than the one holding position ctx_lens[b] - 1 (true for a decode step,
 * which only appends its token): the block table and each warp's first
 * pages are then fetched before waiting on that kernel (programmatic
 * dependent launch), overlapping its tail. */
#define KVX_ATTN_EARLY_PREFETCH 1
/* Bits 8..11: clusters per (request, kv head) for an explicit split count
 * (num_splits = G x C): C-CTA clusters merge over DSMEM, then the G cluster
 * results merge in the workspace (needed). 0 / 1: one cluster (or the auto plan). */
#define KVX_ATTN_CLUSTERS(g) (((g) & 0xF) << 8)

/* Split-K merge strategies (both in-kernel, one launch). AUTO picks CLUSTER
 * when the splits of each (request, kv head) fit one thread-block cluster
 * (<= 16 CTAs) co-resident in a single wave, GLOBAL otherwise. */
enum {
  KVX_MERGE_AUTO = 0,
  KVX_MERGE_GLOBAL = 1,  /* partials in the workspace, last CTA merges (arrival counter) */
  KVX_MERGE_CLUSTER = 2  /* partials in shared memory, merged over DSMEM              */
};

const char* kvx_last_error(void);
int kvx_version(void);
/* Launches of this library's own kernels since load (all threads), and
 * calls into the cuBLAS library (kvx_model's projections) — counters a
 * host samples around a timed region. */
uint64_t kvx_launch_count(void);
uint64_t kvx_library_launch_count(void);
/* Bytes of one page for `layout` (2 * H * T * D * sizeof(dtype)). */
uint64_t kvx_page_bytes(const kvx_page_layout* layout);

/* ---- pools --------------------------------------------------------------- */
/* DEVICE pool in HBM of `device` (pages 256-B aligned). */
int kvx_pool_create(int device, uint64_t num_pages, uint64_t page_bytes, kvx_pool** out);
/* HOST pool: pinned, device-mapped host memory (HOST-tier payload). */
int kvx_pool_create_host(uint64_t num_pages, uint64_t page_bytes, kvx_pool** out);
/* DISK tier: a pool whose pages live in a file (created / grown to
 * num_pages * page_bytes; the file is kept on destroy). Pages move between a
 * file pool and a HOST pool with kvx_copy_pages(KVX_COPY_CE, host id arrays):
 * the reads/writes run in stream order (host callbacks on the stream), with
 * O_DIRECT when the filesystem supports it. kvx_pool_base() is NULL; I/O
 * errors are sticky and reported by every later call on the pool
 * (KVX_ERR_IO). The reference keeps DISK as byte accounting only
 * (kvstore.cpp:881-900 DiskWrite, :862-866 LoadDiskHost). */
int kvx_pool_create_file(const char* path, uint64_t num_pages, uint64_t page_bytes, kvx_pool** out);
/* 1 if the pool's file was opened with O_DIRECT, 0 if buffered, -1 if not a file pool. */
int kvx_pool_file_direct(const kvx_pool* pool);
/* The sticky errno of the first failed read/write on a file pool (0: none,
 * or not a file pool). File I/O runs as host callbacks in stream order, so a
 * failure does not fail the stream: callers that install pages after a sync
 * (NodePayload's DISK-lane applies) check this first. */
int kvx_pool_io_error(const kvx_pool* pool);
/* Wraps caller-owned device memory (not freed by kvx_pool_destroy). */
int kvx_pool_wrap(int device, void* base, uint64_t num_pages, uint64_t page_bytes, kvx_pool** out);
int kvx_pool_destroy(kvx_pool* pool);
void* kvx_pool_base(const kvx_pool* pool);
uint64_t kvx_pool_num_pages(const kvx_pool* pool);
uint64_t kvx_pool_page_bytes(const kvx_pool* pool);
int kvx_pool_device(const kvx_pool* pool); /* -1 for a host pool */
/* CUDA IPC: export a DEVICE pool (64-byte handle) / open a peer's pool in
 * this process so kernels here can store into it over NVLink. */
int kvx_pool_ipc_export(const kvx_pool* pool, void* handle64);
int kvx_pool_ipc_open(int device, const void* handle64, uint64_t num_pages, uint64_t page_bytes,
                      kvx_pool** out);
int kvx_enable_peer_access(int device, int peer);

/* ---- runtime helpers for C++/FFI hosts ------------------------------------
 * Thin wrappers so host code (libsymsim_b200's payload backend, cgo/JNI
 * callers) needs no CUDA headers or runtime of its own. */
int kvx_stream_create(int device, void** out);
int kvx_stream_destroy(void* stream);
int kvx_stream_synchronize(void* stream);
int kvx_malloc(int device, uint64_t bytes, void** out);
int kvx_free(void* ptr);
/* Pinned host memory (staging for async uploads). */
int kvx_host_alloc(uint64_t bytes, void** out);
int kvx_host_free(void* ptr);
/* cudaMemcpyAsync(kind = Default) on `stream`. */
int kvx_memcpy_async(void* dst, const void* src, uint64_t bytes, void* stream);
/* Synchronous copy of one page to host memory (verification / debugging). */
int kvx_read_page(const kvx_pool* pool, uint64_t page, void* host_out);
/* Events (timing disabled) for stream-ordered completion of page moves.
 * kvx_event_query returns KVX_OK when complete, KVX_NOT_READY otherwise. */
#define KVX_NOT_READY 4
int kvx_event_create(void** out);
int kvx_event_destroy(void* event);
int kvx_event_record(void* event, void* stream);
int kvx_event_synchronize(void* event);
int kvx_event_query(void* event);
int kvx_stream_wait_event(void* stream, void* event);
/* Device-side signals between GPUs (no host in the loop): `stream` writes
 * `value` to a 32-bit flag once all its prior work is complete and visible
 * (the flag may live in a peer GPU's memory opened through CUDA IPC), and a
 * stream waits until a flag is >= `value` before running its later work.
 * This is how a migration's per-layer arrival (the reference's NetArrive,
 * kvstore.cpp:914-923) gates the receiver's decode of that layer
 * (pipeline_gate, kvstore.cpp:46-59) across GPUs. */
int kvx_signal_write(void* d_flag, uint32_t value, void* stream);
int kvx_signal_wait(const void* d_flag, uint32_t value, void* stream);
/* 1 if the device of `stream` can flush remote writes at a wait
 * (cudaDevAttrCanFlushRemoteWrites), 0 if not, -1 on error. kvx_signal_wait
 * requests the flush on the stream's device when available; without it the
 * writer's system-scope barrier is the only ordering of the peer's data
 * before the flag, and callers should report a gate built on it as
 * unverified (or hand off through an event / the host). */
int kvx_signal_flush_supported(void* stream);

/* ---- page movement (K1-K3) ---------------------------------------------- */
/* dst[i * page_bytes ...] = page(ids[i]) for i < n. ids in device memory. */
int kvx_pack(const kvx_pool* src, const uint32_t* d_page_ids, uint64_t n, void* d_dst, int mode,
             void* stream);
/* page(ids[i]) = src[i * page_bytes ...]. */
int kvx_unpack(kvx_pool* dst, const uint32_t* d_page_ids, uint64_t n, const void* d_src, int mode,
               void* stream);
/* dst page(dst_ids[i]) = src page(src_ids[i]); pools may live on different
 * GPUs (peer access / IPC), or one may be a host pool. Both pools must have
 * the same page_bytes. ids are device pointers except for KVX_COPY_CE, which
 * takes host arrays. */
int kvx_copy_pages(const kvx_pool* src, const uint32_t* src_ids, kvx_pool* dst, const uint32_t* dst_ids,
                   uint64_t n, int mode, void* stream);
/* Background migration (the reference's NetArrive moves, kvstore.cpp:753-769,
 * run off the serving path): kvx_copy_pages with the SM movers' grid bounded
 * to max_ctas CTAs (0 = unbounded), so a migration running beside decode
 * occupies a fixed slice of the SMs and paces its HBM/NVLink traffic.
 * Ignored for KVX_COPY_CE. */
int kvx_copy_pages_capped(const kvx_pool* src, const uint32_t* src_ids, kvx_pool* dst, const uint32_t* dst_ids,
                          uint64_t n, int mode, uint32_t max_ctas, void* stream);
/* K3 with HOST id arrays (src_ids / dst_ids in host memory, range-checked
 * here): the ids travel in the launch parameters (up to 3,840 pages per
 * launch), so a move needs no device id array or upload — the CE lane's mover
 * for fragmented PCIe moves. (A launch copies its parameter block: per-layer
 * HBM moves in NodePayload keep the staged upload + kvx_copy_pages_capped,
 * measured cheaper on the host.)
 * mode: KVX_COPY_AUTO (TMA bulk mover for HBM<->HBM on one device, else the
 * SM vector mover), KVX_COPY_SM or KVX_COPY_TMA; max_ctas > 0 caps the grid.
 * At least one endpoint must be a device pool; not for file pools. Replaces
 * the same reference transfers as kvx_copy_pages. */
int kvx_copy_pages_listed(const kvx_pool* src, const uint32_t* src_ids, kvx_pool* dst, const uint32_t* dst_ids,
                          uint64_t n, int mode, uint32_t max_ctas, void* stream);


/* K3 over NCCL (the collective-library migration variant):
 * per chunk of pages_per_chunk pages — one migration layer — K1 packs the
 * chunk of `send` pages into a staging slot, one NCCL group sends it to
 * send_peer and receives recv_peer's chunk into the other slot, and K2
 * unpacks it into `recv` pages. Either side may be empty (n = 0), so a ring
 * rank both sends and receives in one call without deadlock. `comm` is an
 * ncclComm_t (kvx_nccl_comm_init_rank or the caller's own); d_staging holds
 * kvx_migrate_nccl_staging_bytes() bytes. NCCL is loaded at run time
 * (libnccl.so.2); without it the calls return KVX_ERR_UNSUPPORTED. All
 * asynchronous on `stream`. */
uint64_t kvx_migrate_nccl_staging_bytes(uint64_t page_bytes, uint64_t pages_per_chunk);
int kvx_migrate_nccl(const kvx_pool* send_pool, const uint32_t* d_send_ids, uint64_t n_send, int send_peer,
                     kvx_pool* recv_pool, const uint32_t* d_recv_ids, uint64_t n_recv, int recv_peer,
                     uint64_t pages_per_chunk, void* comm, void* d_staging, uint64_t staging_bytes, void* stream);
int kvx_nccl_get_unique_id(void* id128);
int kvx_nccl_comm_init_rank(void** comm, int nranks, const void* id128, int rank, int device);
int kvx_nccl_comm_destroy(void* comm);

/* ---- contents (K5) ------------------------------------------------------ */
int kvx_fill_pages(kvx_pool* pool, const uint32_t* d_page_ids, const kvx_block_tag* d_tags, uint64_t n,
                   uint64_t seed, const kvx_page_layout* layout, int fill_mode, void* stream);
/* Scrub (K5 check): counts into *d_mismatches (device u64, accumulated) the
 * pages whose bytes differ from the K5 content of their tag — a list of
 * (page, tag) pairs, or every block of a decode step's block tables
 * ([num_layers][batch][max_blocks], tag = (sessions[b], layer, block), blocks
 * past ctx_lens[b] skipped). Page ids outside the pool count as mismatches. */
int kvx_verify_pages(const kvx_pool* pool, const uint32_t* d_page_ids, const kvx_block_tag* d_tags, uint64_t n,
                     uint64_t seed, const kvx_page_layout* layout, int fill_mode, unsigned long long* d_mismatches,
                     void* stream);
int kvx_verify_block_tables(const kvx_pool* pool, const kvx_page_layout* layout, const uint32_t* d_tables,
                            const int32_t* d_ctx_lens, const int32_t* d_sessions, int32_t num_layers, int32_t batch,
                            int32_t max_blocks, uint64_t seed, int fill_mode, unsigned long long* d_mismatches,
                            void* stream);
/* For request i: page d_page_ids[i], token slot d_slots[i] (< block_tokens)
 * gets K = d_k[i][H][D], V = d_v[i][H][D] (layout dtype). */
int kvx_append_kv(kvx_pool* pool, const kvx_page_layout* layout, const uint32_t* d_page_ids,
                  const int32_t* d_slots, const void* d_k, const void* d_v, uint64_t n, void* stream);

/* ---- paged decode attention (K4) ----------------------------------------- */
/* out[b][hq][d] (fp32) = softmax(scale * q[b][hq] . K^T) V over the first
 * ctx_lens[b] tokens of request b, whose block table row is
 * d_block_tables[b * max_blocks ...]. q has the layout dtype. Workspace of
 * kvx_decode_attention_workspace() bytes (may be 0 -> NULL allowed): split-K
 * partials plus per-(request, kv head) arrival counters for the GLOBAL merge;
 * it must be zero-filled before its first use, and every launch leaves the
 * counters zeroed again (the last split of each group merges all splits
 * in-kernel). The CLUSTER merge does not touch it.
 * Preconditions: 0 <= ctx_lens[b] <= max_ctx <= max_blocks * block_tokens
 * for every request, every table entry < the pool's page count, and
 * 0 <= num_splits <= 256. Host-checkable ones return KVX_ERR_ARG; a device
 * table or ctx_lens entry that breaks them traps the kernel (the stream
 * fails with a CUDA error) rather than reading or writing out of bounds. */
uint64_t kvx_decode_attention_workspace(const kvx_page_layout* layout, const kvx_attn_params* params,
                                        int32_t batch, int32_t max_ctx);
int kvx_decode_attention(const kvx_pool* pool, const kvx_page_layout* layout, const kvx_attn_params* params,
                         const uint32_t* d_block_tables, const int32_t* d_ctx_lens, const void* d_q,
                         float* d_out, int32_t batch, int32_t max_ctx, void* d_workspace,
                         uint64_t workspace_bytes, void* stream);
/* One decode step of one layer, fused: first writes this step's token —
 * d_new_k[b][H][D] / d_new_v[b][H][D] (layout dtype), position
 * ctx_lens[b] - 1, into its slot of the page its block table names (the
 * bytes behind Engine::apply_step's append_blocks(1), engine.cpp:132-166,
 * kvstore.cpp:202-271) — then attends over ctx_lens[b] tokens as
 * kvx_decode_attention. On the bf16 / d128 / 16-token fast path the append
 * is done inside the attention launch by the CTA that streams the last page
 * (one launch per layer instead of two). */
int kvx_decode_attention_append(kvx_pool* pool, const kvx_page_layout* layout, const kvx_attn_params* params,
                                const uint32_t* d_block_tables, const int32_t* d_ctx_lens, const void* d_q,
                                const void* d_new_k, const void* d_new_v, float* d_out, int32_t batch,
                                int32_t max_ctx, void* d_workspace, uint64_t workspace_bytes, void* stream);

/* ---- the decode step around K4 (K6) --------------------------------------
 * The reference models a serving engine's quanta (prefill_time and
 * decode_step_time, costmodel.cpp:54-80; Engine::try_start,
 * engine.cpp:168-262). A kvx_model executes them on the GPU for a
 * Llama-shaped decoder with random bf16 weights: dense projections on cuBLAS
 * (library GEMMs), norms / RoPE / SiLU / sampling hand-written, and K4 with
 * this step's token appended (kvx_decode_attention_append) per layer over the
 * pages of a kvx_pool. The K/V written into a page is that slot's K5 content
 * (fill of its (session, layer, block) tag with fill_seed / fill_mode), so
 * pages stay oracle-checkable. One model may serve several callers (nodes)
 * but its activations are shared: calls must not overlap in time. */
typedef struct kvx_model kvx_model;
typedef struct {
  int32_t num_layers;   /* 32 (Llama-3.1-8B) */
  int32_t hidden;       /* 4096 */
  int32_t num_q_heads;  /* 32 */
  int32_t num_kv_heads; /* 8 */
  int32_t head_dim;     /* 128 (required) */
  int32_t intermediate; /* 14336 */
  int32_t vocab;        /* 128256 */
  float rms_eps;        /* 1e-5 */
  float rope_theta;     /* 500000 */
} kvx_model_config;

uint64_t kvx_model_weight_bytes(const kvx_model_config* cfg);
int kvx_model_create(int device, const kvx_model_config* cfg, uint64_t seed, kvx_model** out);
int kvx_model_destroy(kvx_model* model);
/* One decode step for `batch` requests (<= 256). d_tables: [num_layers][batch]
 * [max_blocks] page ids of each request's blocks per layer; d_ctx_lens[b]
 * tokens including this step's (written at position ctx - 1); d_sessions[b]
 * the session ids (K5 tags); d_tokens_in[b] the input token ids;
 * d_tokens_out[b] the greedy samples. layer_waits[layer_wait_offsets[l] ..
 * layer_wait_offsets[l+1]) are events (host array) the attention of layer l
 * waits for — loads still landing (NULL: none). Asynchronous on `stream`. */
int kvx_model_decode_step(kvx_model* model, kvx_pool* pool, const kvx_page_layout* layout, const uint32_t* d_tables,
                          const int32_t* d_ctx_lens, const int32_t* d_sessions, const int32_t* d_tokens_in,
                          int32_t batch, int32_t max_blocks, int32_t max_ctx, uint64_t fill_seed, int32_t fill_mode,
                          void* const* layer_waits, const int32_t* layer_wait_offsets, int32_t* d_tokens_out,
                          void* stream);
/* The dense work of prefilling `tokens` prompt tokens (all projections and
 * MLPs, 4,096-row passes, LM head of the last token). The prompt's K/V pages
 * are the store's Created fill; prefill attention is not executed. */
int kvx_model_prefill(kvx_model* model, int32_t tokens, void* stream);
/* One projection of the model's kind, Y[rows][out] (+= when accumulate)
 * X[rows][in] . W[out][in]^T (bf16 in/out, fp32 accumulation), on the model's
 * workspace: K7 (skinny_linear, tensor-core mma over streamed weights) for
 * rows <= 16 with in % 128 == 0 and out % 16 == 0, cuBLAS otherwise — the
 * decode step's projection path, exposed for tests and measurement. The
 * shape must be one of the model's (its split-K workspace is sized for them). */
int kvx_model_linear(kvx_model* model, const void* d_x, const void* d_w, void* d_y, int32_t rows, int32_t in,
                     int32_t out, int32_t accumulate, void* stream);
/* Timing helpers for hosts without CUDA headers: events with timing. */
int kvx_timer_create(void** out);
int kvx_timer_elapsed_ms(void* start, void* stop, float* ms);

#ifdef __cplusplus
}
#endif

#endif /* KVX_H_ */
