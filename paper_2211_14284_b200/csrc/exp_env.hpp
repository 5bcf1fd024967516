#pragma once
#include <cstdlib>

namespace rm {

// Experiment / instrumentation switches read from the environment (ring sizes, grid, profiling
// counters, alternative kernels): compiled in only with -DRM_EXPERIMENTS, so the product build reads
// none of them.  The documented runtime knobs (rm.h, rm_setup) are RM_SETUP_THREADS, RM_NBOX1 and
// RM_PATCH_STREAM.
inline const char* exp_env(const char* name) {
#ifdef RM_EXPERIMENTS
  return std::getenv(name);
#else
  (void)name;
  return nullptr;
#endif
}

}  // namespace rm
