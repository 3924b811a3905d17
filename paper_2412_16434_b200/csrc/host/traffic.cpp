// Serving-traffic generators and latency aggregates (include/symsim/traffic.hpp).

#include "symsim/traffic.hpp"

#include <algorithm>
#include <cmath>
#include <numeric>
#include <random>

namespace symsim::traffic {

std::vector<int> zipf_turns(std::size_t sessions, double s, double scale, int min_turns, std::uint64_t seed) {
  std::vector<std::size_t> rank_of(sessions);
  std::iota(rank_of.begin(), rank_of.end(), std::size_t{0});
  std::mt19937_64 rng(seed);
  std::shuffle(rank_of.begin(), rank_of.end(), rng);  // rank_of[r] = session at rank r + 1
  std::vector<int> turns(sessions, min_turns);
  for (std::size_t r = 0; r < sessions; ++r) {
    const double want = scale / std::pow(static_cast<double>(r + 1), s);
    turns[rank_of[r]] = std::max(min_turns, static_cast<int>(std::lround(want)));
  }
  return turns;
}

std::vector<Ns> poisson_gaps(std::size_t n, double mean_s, std::uint64_t seed) {
  std::mt19937_64 rng(seed);
  std::exponential_distribution<double> gap(1.0 / mean_s);
  std::vector<Ns> out(n);
  for (auto& g : out) g = ns_from_sec(gap(rng));
  return out;
}

double percentile(std::vector<double> v, double q) {
  if (v.empty()) return 0.0;
  std::sort(v.begin(), v.end());
  q = std::clamp(q, 0.0, 1.0);
  const double pos = q * static_cast<double>(v.size() - 1);
  const std::size_t lo = static_cast<std::size_t>(pos);
  const std::size_t hi = std::min(lo + 1, v.size() - 1);
  return v[lo] + (v[hi] - v[lo]) * (pos - static_cast<double>(lo));
}

LatencyStats latency_stats(const std::vector<double>& v) {
  LatencyStats s;
  s.n = v.size();
  if (v.empty()) return s;
  s.p50 = percentile(v, 0.5);
  s.p90 = percentile(v, 0.9);
  s.p99 = percentile(v, 0.99);
  s.mean = std::accumulate(v.begin(), v.end(), 0.0) / static_cast<double>(v.size());
  return s;
}

double rps_within_slo(const std::vector<LoadPoint>& sweep, double slo) {
  double best = 0.0;
  for (const LoadPoint& p : sweep)
    if (p.p50 <= slo) best = std::max(best, p.rps);
  return best;
}

}  // namespace symsim::traffic
