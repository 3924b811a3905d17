// Sizing and link timing for the B200 KV store.
//
// Behaviour follows /root/reference/proj/src/costmodel.cpp (validate messages
// :10-31, kv_bytes :43-46, kv_bytes_per_layer :48-52, prefill_time :54-57,
// decode_step_time :59-80, transfer_time :82-95). Floating-point expressions
// keep the reference's evaluation order so every llround() lands on the same
// integer nanosecond: state parity with the oracle is bit-exact, and the
// event order the lockstep runtime derives from these times is identical.

#include "symsim/costmodel.hpp"

#include <stdexcept>

namespace symsim {

namespace {

void require(bool ok, const char* what) {
  if (!ok) throw std::runtime_error(what);
}

// Linear interpolation over a strictly increasing (batch, ms) curve, clamped.
double curve_lookup(const std::vector<std::pair<int, double>>& curve, int batch) {
  const double b = batch;
  if (b <= curve.front().first) return curve.front().second;
  if (b >= curve.back().first) return curve.back().second;
  std::size_t hi = 1;
  while (curve[hi].first < b) ++hi;
  const double b0 = curve[hi - 1].first, t0 = curve[hi - 1].second;
  const double b1 = curve[hi].first, t1 = curve[hi].second;
  return t0 + (t1 - t0) * (b - b0) / (b1 - b0);
}

double link_bandwidth(Link link, const LinkProfile& links) {
  switch (link) {
    case Link::PcieH2D:
    case Link::PcieD2H:
      return links.pcie_bandwidth;
    case Link::DiskRead:
    case Link::DiskWrite:
      return links.disk_bandwidth;
    case Link::Network:
      return links.network_bandwidth;
  }
  throw std::logic_error("transfer_time: bad link");
}

}  // namespace

void GpuProfile::validate() const {
  require(prefill_throughput > 0, "gpu: prefill_throughput must be positive");
  require(decode_base_ms > 0, "gpu: decode_base_ms must be positive");
  require(decode_half_batch > 0, "gpu: decode_half_batch must be positive");
  require(hbm_capacity > 0, "gpu: hbm_capacity must be positive");
  require(kv_bytes_per_token > 0, "gpu: kv_bytes_per_token must be positive");
  require(num_layers > 0, "gpu: num_layers must be positive");
  int prev_batch = 0;
  bool first = true;
  for (const auto& [batch, ms] : decode_curve_ms) {
    require(batch > 0 && ms > 0, "gpu: decode_curve_ms entries must be positive");
    require(first || batch > prev_batch, "gpu: decode_curve_ms batch sizes must be strictly increasing");
    prev_batch = batch;
    first = false;
  }
}

void LinkProfile::validate() const {
  require(pcie_bandwidth > 0, "link: pcie_bandwidth must be positive");
  require(disk_bandwidth > 0, "link: disk_bandwidth must be positive");
  require(network_bandwidth > 0, "link: network_bandwidth must be positive");
  require(per_transfer_latency >= 0, "link: per_transfer_latency must be nonnegative");
}

const char* link_name(Link link) {
  static const char* const kNames[] = {"pcie_h2d", "pcie_d2h", "disk_read", "disk_write", "network"};
  const auto i = static_cast<unsigned>(link);
  return i < 5 ? kNames[i] : "?";
}

std::int64_t kv_bytes(std::int64_t tokens, const GpuProfile& gpu) {
  require(tokens >= 0, "kv_bytes: negative token count");
  return tokens * gpu.kv_bytes_per_token;
}

std::int64_t kv_bytes_per_layer(std::int64_t tokens, const GpuProfile& gpu) {
  const std::int64_t layers = gpu.num_layers;
  return (kv_bytes(tokens, gpu) + layers - 1) / layers;
}

Ns prefill_time(std::int64_t tokens, const GpuProfile& gpu) {
  require(tokens > 0, "prefill_time: token count must be positive");
  return ns_from_sec(static_cast<double>(tokens) / gpu.prefill_throughput);
}

Ns decode_step_time(int batch_size, const GpuProfile& gpu) {
  require(batch_size > 0, "decode_step_time: batch size must be positive");
  const double ms = gpu.decode_curve_ms.empty()
                        ? gpu.decode_base_ms * (1.0 + batch_size / gpu.decode_half_batch)
                        : curve_lookup(gpu.decode_curve_ms, batch_size);
  return ns_from_ms(ms);
}

Ns transfer_time(std::int64_t bytes, Link link, const LinkProfile& links) {
  require(bytes >= 0, "transfer_time: negative byte count");
  if (bytes == 0) return 0;
  const double bw = link_bandwidth(link, links);
  return links.per_transfer_latency + ns_from_sec(static_cast<double>(bytes) / bw);
}

}  // namespace symsim
