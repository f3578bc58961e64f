// Experiment knobs.  The product build ignores the environment: every knob returns its measured
// default, so kernel choices, split counts (summation orders) and grids never depend on environment
// variables, and the kernels carry no timing-experiment branches.  `make EXPERIMENTS=1` defines
// PBD_EXPERIMENTS, which reads the PBD_* / PBDK_* overrides the A/B scripts under scripts/ use and
// compiles the PBDK_CONV_DEBUG timing modes into the convolution kernels.
#pragma once

#include <cstdlib>

namespace pbd {

#ifdef PBD_EXPERIMENTS
constexpr bool kExperiments = true;
#else
constexpr bool kExperiments = false;
#endif

inline const char* knob_env(const char* name) { return kExperiments ? std::getenv(name) : nullptr; }

// Programmatic dependent launch for the executors' convolutions (on; PBD_PDL=0 for A/B runs).
inline bool pdl_enabled() {
  const char* e = knob_env("PBD_PDL");
  return e == nullptr || e[0] != '0';
}

}  // namespace pbd
