#pragma once
// Minimal slice of the reference workload vocabulary that the KV store needs.
// The full trace/workload module (proj/include/symsim/workload.hpp) is out of
// scope for the B200 hot path ("workload: OUT OF SCOPE"); only
// the session priority class crosses into the store
// (reference: proj/include/symsim/workload.hpp:20).
//
// When this header is compiled together with the reference's own callers
// (tests/cpp/build_ref_harness.sh), the include path resolves
// "symsim/workload.hpp" to the reference header instead, which declares the
// same enum with the same enumerators.

namespace symsim {

enum class PriorityClass { Normal, High };

}  // namespace symsim
