// fw_stub.cpp — TEST BUILD ONLY.  In a real integration gw::fw_solve stays
// in the reference's proj/src/solvers.cpp (FW is outside the B200 path);
// this test library cannot link that file next to gw_b200.cpp, so FW
// reports that it is not part of the drop-in.
#include <stdexcept>

#include "gw/solvers.hpp"

namespace gw {
SolveReport fw_solve(const DistanceMatrix&, const DistanceMatrix&, const ProbabilityVector&,
                     const ProbabilityVector&, const SolverConfig&, const SolveOptions&) {
  throw std::runtime_error(
      "fw_solve is kept from the reference's solvers.cpp in an integration; not in the drop-in");
}
}  // namespace gw
