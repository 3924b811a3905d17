#pragma once
// The B200 decode step behind the engine's quanta.
//
// GpuStepExecutor implements StepExecutor (engine.hpp) for one node: when
// the engine starts a quantum it
//   * builds the batch's block tables, layer by layer, from the node's
//     NodePayload (NodePayload::decode_rows: DEVICE pages installed or still
//     being loaded; the events of loads still writing a layer's pages gate
//     that layer's attention — the reference's pipeline_gate,
//     kvstore.cpp:46-59, made physical),
//   * uploads tables / context lengths / sessions / input tokens,
//   * runs the Llama-shaped decode step on the GPU (kvx_model_decode_step:
//     per layer the dense projections plus K4 with this step's token
//     appended into its page), reads back the sampled tokens,
// and returns the CUDA-event-measured duration of all of that, which the
// engine uses as the quantum's length instead of decode_step_time
// (costmodel.cpp:59-80). A prefill runs the dense work of its tokens
// (kvx_model_prefill) and is timed the same way.
//
// One ModelRuntime (weights, stream, staging) per device is shared by the
// executors of the nodes on it; the engine loop is single-threaded and every
// executed quantum synchronizes, so their calls never overlap.

#include <cstdint>
#include <memory>
#include <unordered_map>
#include <vector>

#include "kvx.h"
#include "symsim/engine.hpp"
#include "symsim/payload.hpp"

namespace symsim {

// Llama-3.1-8B (the KV shape of configs 2, 4 and 5).
kvx_model_config llama31_8b_config();

class ModelRuntime {
 public:
  ModelRuntime(int device, const kvx_model_config& cfg, std::uint64_t weight_seed);
  ~ModelRuntime();
  ModelRuntime(const ModelRuntime&) = delete;
  ModelRuntime& operator=(const ModelRuntime&) = delete;

  int device() const { return device_; }
  kvx_model* model() const { return model_; }
  const kvx_model_config& config() const { return cfg_; }
  void* stream() const { return stream_; }

  // Times `launch` (queued on stream()) with CUDA events; returns ns.
  template <typename F>
  std::int64_t timed(F&& launch);

  // Device / pinned scratch of at least `bytes` (grown on demand; callers
  // synchronize before reuse, which every timed call does).
  void* device_scratch(std::size_t bytes);
  void* host_scratch(std::size_t bytes);

 private:
  int device_;
  kvx_model_config cfg_;
  kvx_model* model_ = nullptr;
  void* stream_ = nullptr;
  void* t0_ = nullptr;
  void* t1_ = nullptr;
  void* dev_ = nullptr;
  std::size_t dev_cap_ = 0;
  void* host_ = nullptr;
  std::size_t host_cap_ = 0;
};

class GpuStepExecutor final : public StepExecutor {
 public:
  GpuStepExecutor(ModelRuntime& runtime, NodePayload& payload);
  ~GpuStepExecutor() override;
  // Every `every`-th decode step (0: never), after its timed region, scrub
  // every page it attended against the K5 content of its (session, layer,
  // block) tag (kvx_verify_block_tables): the bytes a migrated / reloaded /
  // appended cache holds when the engine consumes it.
  void verify_every(int every) { verify_every_ = every; }
  std::uint64_t verified_pages() const { return verified_pages_; }
  std::uint64_t mismatched_pages();  // synchronizes

  Ns decode_step(const std::vector<Row>& rows) override;
  Ns prefill(std::uint32_t session, std::int64_t tokens) override;

  struct Stats {
    std::int64_t steps = 0, prefills = 0;
    std::int64_t step_ns = 0, prefill_ns = 0;
    std::int64_t gated_layers = 0;      // layer attentions that waited on a load still landing
    std::int64_t attended_tokens = 0;   // sum over steps of the batch's context tokens
    std::int64_t rows = 0;              // sum over steps of the batch size (tokens emitted)
    std::int64_t max_batch = 0;
    std::int64_t host_table_ns = 0;     // host time building the block tables
  };
  const Stats& stats() const { return stats_; }

 private:
  ModelRuntime& rt_;
  NodePayload& payload_;
  std::unordered_map<std::uint32_t, std::int32_t> last_token_;  // per session: the previous step's sample
  std::vector<std::uint32_t> tables_;
  std::vector<void*> waits_;
  std::vector<std::int32_t> wait_off_;
  Stats stats_;
  int verify_every_ = 0;
  std::uint64_t verified_pages_ = 0;
  void* d_mismatch_ = nullptr;  // device u64
};

}  // namespace symsim
