// Engine: the consumer end of the KV hot path.
//
// Restates the reference engine's quantum semantics
// (/root/reference/proj/src/engine.cpp; SPEC.md engine section) so that,
// without an executor, the reference NodeManager/Simulation produce the
// same ledger and request records over this engine as over the reference
// one (tests/test_engine_parity.py). Anchors:
//   admission + loads + prompt reservation   engine.cpp:77-106
//   prefill boundary                         engine.cpp:108-130
//   decode-step boundary (append per token)  engine.cpp:132-166
//   quantum start (gate release, pausing)    engine.cpp:168-262
//   cooperative eviction for growth          engine.cpp:60-75
// With a StepExecutor attached, the quantum's prefill and decode step run on
// the node's GPU at quantum start and the quantum lasts their measured time.

#include "symsim/engine.hpp"

#include <algorithm>
#include <mutex>
#include <stdexcept>

namespace symsim {

namespace {
std::mutex g_exec_mu;
StepExecutorFactory g_exec_factory;
}  // namespace

void set_default_step_executor_factory(StepExecutorFactory factory) {
  std::lock_guard<std::mutex> lock(g_exec_mu);
  g_exec_factory = std::move(factory);
}

const char* policy_name(Policy p) {
  static const char* const kNames[] = {"recompute", "retain", "swap", "symphony"};
  const auto i = static_cast<unsigned>(p);
  return i < 4 ? kNames[i] : "?";
}

Policy policy_from(const std::string& name) {
  for (Policy p : {Policy::Recompute, Policy::Retain, Policy::Swap, Policy::Symphony})
    if (name == policy_name(p)) return p;
  throw std::runtime_error("unknown policy '" + name + "'");
}

Engine::Engine(const EngineConfig& cfg, const GpuProfile& gpu, KvStore& store)
    : cfg_(cfg), gpu_(gpu), store_(store) {
  if (cfg_.max_batch <= 0) throw std::runtime_error("engine: max_batch must be positive");
  StepExecutorFactory f;
  {
    std::lock_guard<std::mutex> lock(g_exec_mu);
    f = g_exec_factory;
  }
  if (f) exec_ = f(store_);
}

void Engine::enqueue(const RequestSpec& spec, Ns now) {
  if (spec.prefill_tokens <= 0 || spec.target_tokens <= 0)
    throw std::logic_error("engine: request with empty prefill or target");
  const bool live = std::any_of(slots_.begin(), slots_.end(), [&](const Slot& s) {
    return s.stage != Stage::Finished && s.spec.session == spec.session;
  });
  if (live) throw std::logic_error("engine: session already has a live request");
  Slot s;
  s.spec = spec;
  slots_.push_back(std::move(s));
  queue_.push_back(slots_.size() - 1);
  // The session's cache is pinned from arrival: nothing may purge it while
  // the request waits in the queue.
  store_.set_active(spec.session, true, now);
}

int Engine::active_count() const {
  const std::size_t n = decoding_.size() + waiting_.size() + paused_.size() + (prefill_slot_ != kNone ? 1 : 0);
  return static_cast<int>(n);
}

bool Engine::has_live_requests() const {
  return std::any_of(slots_.begin(), slots_.end(), [](const Slot& s) { return s.stage != Stage::Finished; });
}

// Modelled latency of a decode step over `batch` requests: the planning
// estimate even when quanta are executed (the plans a load or a gate makes
// ahead of time cannot wait for a measurement).
Ns Engine::batch_latency(int batch) const { return decode_step_time(std::max(1, batch), gpu_); }

// Frees DEVICE room for `need` bytes of cache growth: unpinned blocks of
// normal sessions first, then anything unpinned; a batch that still does
// not fit is a configuration error (engine.cpp:60-75, same message).
void Engine::make_room(std::int64_t need, Ns now, Outcome& out) {
  for (bool spare_high : {true, false}) {
    if (store_.device_free() >= need) return;
    store_.purge_from_device(need - store_.device_free(), now, spare_high, out.transfers);
  }
  if (store_.device_free() >= need) return;
  throw std::runtime_error(
      "engine: device tier cannot hold the running batch's cache growth "
      "(need " + std::to_string(need) + " bytes, free " + std::to_string(store_.device_free()) +
      ", t=" + std::to_string(now) + "ns, " + store_.device_usage_debug() +
      "); reduce max_batch or grow device capacity");
}

// Gets the queue head ready to prefill: a layer-wise load plan for a cache
// held here (once), then the prompt's DEVICE reservation. False leaves the
// head queued (head-of-line blocking on memory).
bool Engine::prepare_head(Ns now, Outcome& out) {
  Slot& s = slots_[queue_.front()];
  auto purge_for = [&](std::int64_t need) {
    if (store_.device_free() >= need) return;
    store_.purge_from_device(need - store_.device_free(), now, true, out.transfers);
    if (store_.device_free() < need) store_.purge_from_device(need - store_.device_free(), now, false, out.transfers);
  };
  if (s.spec.needs_load && !s.load_planned) {
    purge_for(store_.bytes_for_load(s.spec.session));
    const Ns per_layer = batch_latency(static_cast<int>(decoding_.size()) + 1) / gpu_.num_layers;
    auto plan = store_.plan_layerwise_load(s.spec.session, now, per_layer, TransferReason::Demand, out.transfers);
    if (!plan) return false;
    s.layer_ready = std::move(plan->layer_ready);
    s.load_planned = true;
  }
  if (!s.holds_prompt) {
    const std::int64_t need = store_.bytes_for_new_blocks(s.spec.session, s.spec.prefill_tokens);
    purge_for(need);
    if (store_.device_free() < need) return false;
    store_.reserve_device(need);
    s.held_bytes = need;
    s.holds_prompt = true;
  }
  return true;
}

// Prefill boundary: the prompt's blocks become real, and the request either
// decodes from the next quantum or waits for its cache to land.
void Engine::land_prefill(Ns at, Outcome& out) {
  Slot& s = slots_[prefill_slot_];
  store_.unreserve_device(s.held_bytes);
  s.held_bytes = 0;
  store_.append_blocks(s.spec.session, s.spec.prefill_tokens, at, out.transfers);
  s.decode_entry = at;
  s.gate = at;
  if (!s.layer_ready.empty()) {
    const GateResult g = pipeline_gate(s.layer_ready, at, batch_latency(static_cast<int>(decoding_.size()) + 1));
    s.gate = g.gate_start;
    s.load_stall = g.stall;
  }
  const bool ready = s.gate <= at;
  s.stage = ready ? Stage::Decoding : Stage::WaitingCache;
  (ready ? decoding_ : waiting_).push_back(prefill_slot_);
  prefill_slot_ = kNone;
  prefill_end_ = -1;
}

// Decode-step boundary: every emitter's token lands in the cache (the final
// one included), finished requests leave the batch.
void Engine::land_step(Ns at, Outcome& out) {
  for (std::size_t i : emitters_) {
    Slot& s = slots_[i];
    if (s.stage != Stage::Decoding) throw std::logic_error("engine: emitter not decoding");
    ++s.emitted;
    ++s.steps;
    if (s.first_token < 0) s.first_token = at;
    const std::int64_t grow = store_.bytes_for_new_blocks(s.spec.session, 1);
    if (grow > 0) make_room(grow, at, out);
    store_.append_blocks(s.spec.session, 1, at, out.transfers);
    if (s.emitted != s.spec.target_tokens) continue;
    s.stage = Stage::Finished;
    s.finish = at;
    store_.set_active(s.spec.session, false, at);
    FinishedRequest f;
    f.spec = s.spec;
    f.admit = s.admit;
    f.decode_entry = s.decode_entry;
    f.first_token = s.first_token;
    f.finish = s.finish;
    f.load_stall = s.load_stall;
    f.participations = s.steps;
    out.finished.push_back(std::move(f));
  }
  decoding_.erase(std::remove_if(decoding_.begin(), decoding_.end(),
                                 [this](std::size_t i) { return slots_[i].stage != Stage::Decoding; }),
                  decoding_.end());
  step_end_ = -1;
  emitters_.clear();
}

// Cache-waiters whose gate passes by the time this quantum's decode step
// starts join the batch, in waiting order.
void Engine::release_gated(Ns t_decode) {
  std::vector<std::size_t> keep;
  for (std::size_t i : waiting_) {
    if (slots_[i].gate <= t_decode) {
      slots_[i].stage = Stage::Decoding;
      decoding_.push_back(i);
    } else {
      keep.push_back(i);
    }
  }
  waiting_.swap(keep);
}

// Priority pausing (engine.cpp:212-246): with a latency budget and a
// high-priority request decoding, resume paused requests oldest-first while
// the step fits, then pause the newest normal requests until it fits.
// Without either, everything paused resumes.
void Engine::balance_priority() {
  const Ns budget = ns_from_ms(cfg_.pause_latency_budget_ms);
  const bool high = std::any_of(decoding_.begin(), decoding_.end(),
                                [this](std::size_t i) { return slots_[i].spec.high_priority; });
  if (budget <= 0 || !high) {
    for (std::size_t i : paused_) {
      slots_[i].stage = Stage::Decoding;
      decoding_.push_back(i);
    }
    paused_.clear();
    return;
  }
  while (!paused_.empty() && decode_step_time(static_cast<int>(decoding_.size()) + 1, gpu_) <= budget) {
    slots_[paused_.front()].stage = Stage::Decoding;
    decoding_.push_back(paused_.front());
    paused_.erase(paused_.begin());
  }
  while (decoding_.size() > 1 && decode_step_time(static_cast<int>(decoding_.size()), gpu_) > budget) {
    // Newest normal request by decode entry; ties go to the later slot.
    std::size_t pick = kNone;
    for (std::size_t k = 0; k < decoding_.size(); ++k) {
      const Slot& c = slots_[decoding_[k]];
      if (c.spec.high_priority) continue;
      if (pick == kNone) {
        pick = k;
        continue;
      }
      const Slot& p = slots_[decoding_[pick]];
      if (c.decode_entry > p.decode_entry || (c.decode_entry == p.decode_entry && decoding_[k] > decoding_[pick]))
        pick = k;
    }
    if (pick == kNone) break;  // all high-priority: run over budget
    slots_[decoding_[pick]].stage = Stage::Paused;
    paused_.push_back(decoding_[pick]);
    decoding_.erase(decoding_.begin() + static_cast<std::ptrdiff_t>(pick));
  }
}

// Starts a quantum at `now` if one is runnable: admit the queue head (strict
// FCFS, memory permitting), release gated waiters, apply priority pausing,
// then fix the prefill and the decode batch and their durations — modelled,
// or executed on the GPU right now and measured.
void Engine::open_quantum(Ns now, Outcome& out) {
  if (prefill_end_ >= 0 || step_end_ >= 0) {
    out.next_wake = prefill_end_ >= 0 ? prefill_end_ : step_end_;
    return;
  }
  std::size_t admitted = kNone;
  bool may_admit = !queue_.empty() && active_count() < cfg_.max_batch;
  if (may_admit && cfg_.prefill_mode == PrefillMode::DecodeFirst && !(decoding_.empty() && waiting_.empty()))
    may_admit = false;
  if (may_admit && prepare_head(now, out)) {
    admitted = queue_.front();
    queue_.pop_front();
    slots_[admitted].stage = Stage::Prefilling;
    slots_[admitted].admit = now;
  }
  Ns prefill_ns = 0;
  if (admitted != kNone) {
    const Slot& s = slots_[admitted];
    if (exec_) {
      prefill_ns = std::max<Ns>(1, exec_->prefill(s.spec.session, s.spec.prefill_tokens));
      executed_prefill_ns_ += prefill_ns;
    } else {
      prefill_ns = prefill_time(s.spec.prefill_tokens, gpu_);
    }
  }
  const Ns t_decode = now + prefill_ns;
  release_gated(t_decode);
  balance_priority();

  if (admitted == kNone && decoding_.empty()) {
    if (!waiting_.empty()) {
      Ns wake = slots_[waiting_.front()].gate;
      for (std::size_t i : waiting_) wake = std::min(wake, slots_[i].gate);
      out.next_wake = wake;
    }
    return;
  }
  prefill_slot_ = admitted;
  emitters_ = decoding_;
  Ns step_ns = 0;
  if (!emitters_.empty()) {
    if (exec_) {
      std::vector<StepExecutor::Row> rows;
      rows.reserve(emitters_.size());
      for (std::size_t i : emitters_)
        rows.push_back({slots_[i].spec.session, store_.cached_tokens(slots_[i].spec.session)});
      step_ns = std::max<Ns>(1, exec_->decode_step(rows));
      executed_decode_ns_ += step_ns;
      ++executed_steps_;
    } else {
      step_ns = decode_step_time(static_cast<int>(emitters_.size()), gpu_);
    }
  }
  prefill_end_ = admitted != kNone ? t_decode : -1;
  step_end_ = t_decode + step_ns;
  prefill_busy_ += prefill_ns;
  out.next_wake = prefill_end_ >= 0 ? prefill_end_ : step_end_;
}

Engine::Outcome Engine::advance(Ns now) {
  Outcome out;
  if (prefill_end_ >= 0) {
    if (now < prefill_end_) {
      out.next_wake = prefill_end_;
      return out;
    }
    if (now > prefill_end_) throw std::logic_error("engine: missed prefill boundary");
    land_prefill(now, out);
  }
  if (step_end_ >= 0) {
    if (now < step_end_) {
      out.next_wake = step_end_;
      return out;
    }
    if (now > step_end_) throw std::logic_error("engine: missed quantum end");
    land_step(now, out);
  }
  open_quantum(now, out);
  return out;
}

std::string Engine::diagnostics() const {
  std::string d = "queued=" + std::to_string(queue_.size()) + " decoding=" + std::to_string(decoding_.size()) +
                  " waiting=" + std::to_string(waiting_.size()) + " paused=" + std::to_string(paused_.size());
  if (!queue_.empty()) {
    const Slot& h = slots_[queue_.front()];
    d += " head_session=" + std::to_string(h.spec.session) + " head_turn=" + std::to_string(h.spec.turn);
  }
  for (std::size_t i : waiting_)
    d += " gate[" + std::to_string(slots_[i].spec.session) + "]=" + std::to_string(slots_[i].gate);
  return d;
}

}  // namespace symsim
