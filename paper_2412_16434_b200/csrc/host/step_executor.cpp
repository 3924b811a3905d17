// GpuStepExecutor: the engine's quanta executed on the B200
// (include/symsim/step_executor.hpp). No CUDA headers: everything goes
// through the kvx C ABI.

#include "symsim/step_executor.hpp"

#include <algorithm>
#include <chrono>
#include <cstring>
#include <stdexcept>
#include <string>

namespace symsim {

namespace {
void check(int rc, const char* what) {
  if (rc != KVX_OK) throw std::runtime_error(std::string("step executor: ") + what + ": " + kvx_last_error());
}
std::size_t up16(std::size_t n) { return (n + 15) & ~static_cast<std::size_t>(15); }
}  // namespace

kvx_model_config llama31_8b_config() {
  kvx_model_config c{};
  c.num_layers = 32;
  c.hidden = 4096;
  c.num_q_heads = 32;
  c.num_kv_heads = 8;
  c.head_dim = 128;
  c.intermediate = 14336;
  c.vocab = 128256;
  c.rms_eps = 1e-5f;
  c.rope_theta = 500000.f;
  return c;
}

ModelRuntime::ModelRuntime(int device, const kvx_model_config& cfg, std::uint64_t weight_seed)
    : device_(device), cfg_(cfg) {
  check(kvx_model_create(device, &cfg_, weight_seed, &model_), "model");
  check(kvx_stream_create(device, &stream_), "stream");
  check(kvx_timer_create(&t0_), "timer");
  check(kvx_timer_create(&t1_), "timer");
}

ModelRuntime::~ModelRuntime() {
  if (stream_) kvx_stream_synchronize(stream_);
  kvx_model_destroy(model_);
  kvx_event_destroy(t0_);
  kvx_event_destroy(t1_);
  kvx_free(dev_);
  kvx_host_free(host_);
  kvx_stream_destroy(stream_);
}

template <typename F>
std::int64_t ModelRuntime::timed(F&& launch) {
  check(kvx_event_record(t0_, stream_), "timer start");
  launch();
  check(kvx_event_record(t1_, stream_), "timer stop");
  check(kvx_event_synchronize(t1_), "step sync");
  float ms = 0.f;
  check(kvx_timer_elapsed_ms(t0_, t1_, &ms), "elapsed");
  return static_cast<std::int64_t>(static_cast<double>(ms) * 1e6 + 0.5);
}

void* ModelRuntime::device_scratch(std::size_t bytes) {
  if (bytes > dev_cap_) {
    check(kvx_stream_synchronize(stream_), "sync");
    kvx_free(dev_);
    dev_ = nullptr;
    dev_cap_ = std::max<std::size_t>(bytes * 2, std::size_t{1} << 20);
    check(kvx_malloc(device_, dev_cap_, &dev_), "device scratch");
  }
  return dev_;
}

void* ModelRuntime::host_scratch(std::size_t bytes) {
  if (bytes > host_cap_) {
    check(kvx_stream_synchronize(stream_), "sync");
    kvx_host_free(host_);
    host_ = nullptr;
    host_cap_ = std::max<std::size_t>(bytes * 2, std::size_t{1} << 20);
    check(kvx_host_alloc(host_cap_, &host_), "host scratch");
  }
  return host_;
}

GpuStepExecutor::GpuStepExecutor(ModelRuntime& runtime, NodePayload& payload) : rt_(runtime), payload_(payload) {
  const PayloadOptions& o = payload_.options();
  const kvx_model_config& c = rt_.config();
  if (!o.free_running)
    throw std::runtime_error("step executor: the node's payload must be free-running (pages of layers still "
                             "loading exist only for posted moves)");
  if (o.device != rt_.device()) throw std::runtime_error("step executor: payload and model on different devices");
  if (o.layout.num_kv_heads != c.num_kv_heads || o.layout.head_dim != c.head_dim || o.layout.dtype != KVX_DTYPE_BF16)
    throw std::runtime_error("step executor: page layout does not match the model");
}

GpuStepExecutor::~GpuStepExecutor() { kvx_free(d_mismatch_); }

std::uint64_t GpuStepExecutor::mismatched_pages() {
  if (!d_mismatch_) return 0;
  std::uint64_t n = 0;
  check(kvx_stream_synchronize(rt_.stream()), "sync");
  check(kvx_memcpy_async(&n, d_mismatch_, sizeof(n), rt_.stream()), "mismatch readback");
  check(kvx_stream_synchronize(rt_.stream()), "sync");
  return n;
}

Ns GpuStepExecutor::decode_step(const std::vector<Row>& rows) {
  const int B = static_cast<int>(rows.size());
  if (B == 0) return 0;
  const kvx_model_config& c = rt_.config();
  const std::uint32_t T = static_cast<std::uint32_t>(payload_.options().layout.block_tokens);
  const int L = c.num_layers;
  std::vector<std::pair<std::uint32_t, std::uint32_t>> reqs(rows.size());
  std::uint32_t max_blocks = 1;
  std::int64_t max_ctx = 1;
  for (std::size_t i = 0; i < rows.size(); ++i) {
    if (rows[i].ctx_tokens <= 0) throw std::logic_error("step executor: decoding a request with an empty cache");
    reqs[i] = {rows[i].session, static_cast<std::uint32_t>((rows[i].ctx_tokens + T - 1) / T)};
    max_blocks = std::max(max_blocks, reqs[i].second);
    max_ctx = std::max(max_ctx, rows[i].ctx_tokens);
    stats_.attended_tokens += rows[i].ctx_tokens;
  }
  // Table width and planning context in buckets (2^k and 1.5 x 2^k blocks):
  // steps of the same batch size then share one launch shape, which the
  // model replays as a CUDA graph. Padding entries are never read (each
  // request attends over its own ctx_lens[b] tokens).
  {
    std::uint32_t bucket = 16;
    while (bucket < max_blocks) bucket = (bucket & (bucket - 1)) == 0 ? bucket + bucket / 2 : (bucket / 3) * 4;
    max_blocks = bucket;
    max_ctx = static_cast<std::int64_t>(max_blocks) * T;
  }
  // Host staging: [tables L*B*max_blocks u32][ctx B][sessions B][tokens B].
  const std::size_t tab_bytes = up16(static_cast<std::size_t>(L) * B * max_blocks * 4);
  const std::size_t vec_bytes = up16(static_cast<std::size_t>(B) * 4);
  const std::size_t in_bytes = tab_bytes + 3 * vec_bytes;
  auto* host = static_cast<std::uint8_t*>(rt_.host_scratch(in_bytes + vec_bytes));
  auto* dev = static_cast<std::uint8_t*>(rt_.device_scratch(in_bytes + vec_bytes));
  auto* tables = reinterpret_cast<std::uint32_t*>(host);
  const auto t0 = std::chrono::steady_clock::now();
  std::memset(tables, 0, tab_bytes);
  waits_.clear();
  wait_off_.assign(1, 0);
  for (int l = 0; l < L; ++l) {
    const std::size_t before = waits_.size();
    if (!payload_.decode_rows(reqs, static_cast<std::uint16_t>(l), max_blocks,
                              tables + static_cast<std::size_t>(l) * B * max_blocks, waits_))
      throw std::logic_error("step executor: a decoding session has blocks with no DEVICE page (layer " +
                             std::to_string(l) + ")");
    stats_.gated_layers += waits_.size() > before;
    wait_off_.push_back(static_cast<std::int32_t>(waits_.size()));
  }
  stats_.host_table_ns +=
      std::chrono::duration_cast<std::chrono::nanoseconds>(std::chrono::steady_clock::now() - t0).count();
  auto* ctx = reinterpret_cast<std::int32_t*>(host + tab_bytes);
  auto* ses = reinterpret_cast<std::int32_t*>(host + tab_bytes + vec_bytes);
  auto* tok = reinterpret_cast<std::int32_t*>(host + tab_bytes + 2 * vec_bytes);
  auto* out = reinterpret_cast<std::int32_t*>(host + in_bytes);
  for (int b = 0; b < B; ++b) {
    ctx[b] = static_cast<std::int32_t>(rows[b].ctx_tokens);
    ses[b] = static_cast<std::int32_t>(rows[b].session);
    const auto it = last_token_.find(rows[b].session);
    tok[b] = it != last_token_.end() ? it->second
                                     : static_cast<std::int32_t>((rows[b].session * 2654435761u) % 128000u);
  }
  const PayloadOptions& o = payload_.options();
  kvx_pool* pool = payload_.pool(NodePayload::kDevicePool);
  const std::int64_t ns = rt_.timed([&] {
    // Inputs up, the step, the sampled tokens back: what a serving step moves.
    check(kvx_memcpy_async(dev, host, in_bytes, rt_.stream()), "inputs upload");
    check(kvx_model_decode_step(rt_.model(), pool, &o.layout, reinterpret_cast<const std::uint32_t*>(dev),
                                reinterpret_cast<const std::int32_t*>(dev + tab_bytes),
                                reinterpret_cast<const std::int32_t*>(dev + tab_bytes + vec_bytes),
                                reinterpret_cast<const std::int32_t*>(dev + tab_bytes + 2 * vec_bytes), B,
                                static_cast<std::int32_t>(max_blocks), static_cast<std::int32_t>(max_ctx), o.seed,
                                o.fill_mode, waits_.empty() ? nullptr : waits_.data(), wait_off_.data(),
                                reinterpret_cast<std::int32_t*>(dev + in_bytes), rt_.stream()),
          "decode step");
    check(kvx_memcpy_async(out, dev + in_bytes, static_cast<std::size_t>(B) * 4, rt_.stream()), "tokens readback");
  });
  for (int b = 0; b < B; ++b) last_token_[rows[b].session] = out[b];
  if (verify_every_ > 0 && stats_.steps % verify_every_ == 0) {
    if (!d_mismatch_) {
      check(kvx_malloc(rt_.device(), sizeof(std::uint64_t), &d_mismatch_), "mismatch counter");
      const std::uint64_t zero = 0;
      check(kvx_memcpy_async(d_mismatch_, &zero, sizeof(zero), rt_.stream()), "mismatch counter");
      check(kvx_stream_synchronize(rt_.stream()), "sync");
    }
    check(kvx_verify_block_tables(pool, &o.layout, reinterpret_cast<const std::uint32_t*>(dev),
                                  reinterpret_cast<const std::int32_t*>(dev + tab_bytes),
                                  reinterpret_cast<const std::int32_t*>(dev + tab_bytes + vec_bytes), L, B,
                                  static_cast<std::int32_t>(max_blocks), o.seed, o.fill_mode,
                                  static_cast<unsigned long long*>(d_mismatch_), rt_.stream()),
          "scrub");
    for (const auto& r : reqs) verified_pages_ += static_cast<std::uint64_t>(r.second) * L;
  }
  ++stats_.steps;
  stats_.rows += B;
  stats_.step_ns += ns;
  stats_.max_batch = std::max<std::int64_t>(stats_.max_batch, B);
  return ns;
}

Ns GpuStepExecutor::prefill(std::uint32_t session, std::int64_t tokens) {
  (void)session;
  if (tokens <= 0) return 0;
  const std::int64_t ns = rt_.timed([&] {
    check(kvx_model_prefill(rt_.model(), static_cast<std::int32_t>(tokens), rt_.stream()), "prefill");
  });
  ++stats_.prefills;
  stats_.prefill_ns += ns;
  return ns;
}

}  // namespace symsim
