// Drop-in C++ surface of the B200 dispatch path: shared glue.
//
// The headers in include/embdispatch/ declare the reference's `embdispatch`
// API (/root/reference/proj/include/embdispatch/*.hpp) for the hot path and
// implement it over the C ABI of libedx.so (include/edx.h).  Status codes come
// back as the reference's exception types with the reference's messages, so
// callers written against the reference compile and behave unchanged.
// Link with -ledx (paper_2512_21615_b200/libedx.so).
#pragma once

#include <stdexcept>
#include <string>
#include <vector>

#include "edx.h"

namespace embdispatch {
namespace edxc {

inline void check(int rc) {
  if (rc == EDX_OK) return;
  const std::string msg = edx_last_error();
  switch (rc) {
    case EDX_INVALID_ARGUMENT: throw std::invalid_argument(msg);
    case EDX_LOGIC_ERROR: throw std::logic_error(msg);
    default: throw std::runtime_error(msg);
  }
}

}  // namespace edxc
}  // namespace embdispatch
