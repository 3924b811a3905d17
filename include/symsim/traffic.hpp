#pragma once
// Serving-traffic generators and latency aggregates for configs 4 and 5
// (SURVEY.md §8d, §8f row 3). The reference has neither: its workload
// module (proj/src/workload.cpp) synthesizes a ShareGPT-like corpus and
// closed-loop arrivals with typing-speed think times, and its report keeps
// means and steady requests/s only (report.cpp:65-76). The serving metric of
// BASELINE.json ("requests/s at equal p50 latency") needs:
//   * Poisson turn arrivals: exponential think times between a turn's
//     completion and the user's next prompt (config 4);
//   * skewed session popularity: Zipf(s) over a seeded ranking of sessions,
//     mapped to turns per session (config 5, s = 1.2);
//   * p50 (and p90 / p99) of TTFT, TPOT and normalized latency;
//   * requests/s at a common p50 service level across load sweeps.
// Pure functions over plain types, so the reference's Trace / RunReport
// (out of scope here) are only touched by the callers.

#include <cstddef>
#include <cstdint>
#include <vector>

#include "symsim/time.hpp"

namespace symsim::traffic {

// Turns per session under Zipf(s) popularity: sessions are ranked by a
// seeded shuffle (mt19937_64(seed)); the session at rank r (1-based) gets
// max(min_turns, round(scale / r^s)) turns. out[i] is session i's count.
std::vector<int> zipf_turns(std::size_t sessions, double s, double scale, int min_turns, std::uint64_t seed);

// n exponential gaps with mean `mean_s` seconds (a Poisson process), in ns,
// drawn from mt19937_64(seed).
std::vector<Ns> poisson_gaps(std::size_t n, double mean_s, std::uint64_t seed);

// q-quantile (q in [0, 1]) with linear interpolation between order
// statistics (numpy's default); 0 for an empty input.
double percentile(std::vector<double> values, double q);

struct LatencyStats {
  std::size_t n = 0;
  double p50 = 0, p90 = 0, p99 = 0, mean = 0;
};
LatencyStats latency_stats(const std::vector<double>& values);

// One point of a load sweep: offered users, measured steady requests/s and
// the p50 latency the SLO is judged on.
struct LoadPoint {
  int users = 0;
  double rps = 0;
  double p50 = 0;
};
// Requests/s a policy sustains within a p50 SLO: the highest rps among the
// sweep points whose p50 <= slo (0 when none meets it).
double rps_within_slo(const std::vector<LoadPoint>& sweep, double slo);

}  // namespace symsim::traffic
