// Error plumbing shared by the extern "C" entry points.
#pragma once
#include <string>
#include "runtime.h"

struct cw_runtime {
  cw::Runtime rt;
  bool owned = true;  // false: owned by a cw_engine
};

namespace cw {
void set_error(const std::string& msg);
// "" -> 0, else record the message and return -1.
inline int check(const std::string& err) {
  if (err.empty()) return 0;
  set_error(err);
  return -1;
}
inline int fail(const std::string& err) {
  set_error(err);
  return -1;
}
}  // namespace cw
