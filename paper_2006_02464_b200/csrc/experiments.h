// Profiling overrides read from the environment (plan shapes, kernel flags), compiled in
// only with -DCW_EXPERIMENTS (experiment builds: CW_BUILD_TAG=x CW_NVCC_DEFS=-DCW_EXPERIMENTS,
// used by tools/). The product library never reads the environment on its plan or action
// paths: every plan is a pure function of the arch tables and the batch size.
#pragma once
#include <cstdlib>

namespace cw {
inline const char* exp_env(const char* name) {
#ifdef CW_EXPERIMENTS
  return std::getenv(name);
#else
  (void)name;
  return nullptr;
#endif
}
}  // namespace cw
