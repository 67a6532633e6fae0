// common.h — host-side error plumbing shared by the C-ABI translation units.
#pragma once
#include <cuda_runtime.h>

#include <stdexcept>
#include <string>

#include "../../include/sutradhara_b200.h"

namespace sb {

// Error carrying a C-ABI status code (include/sutradhara_b200.h).
struct Error : std::runtime_error {
  int code;
  Error(int c, const std::string& m) : std::runtime_error(m), code(c) {}
};

void set_last_error(const std::string& msg);

#define SB_CUDA(x)                                                                        \
  do {                                                                                    \
    cudaError_t e_ = (x);                                                                 \
    if (e_ != cudaSuccess)                                                                \
      throw ::sb::Error(SB_ERR_CUDA, std::string(#x) + ": " + cudaGetErrorString(e_));    \
  } while (0)

#define SB_CHECK_LAUNCH() SB_CUDA(cudaGetLastError())

// Wraps a C-ABI body: converts exceptions into status codes + last error.
template <class F>
int guard(F&& f) {
  // errors recorded by earlier runtime calls of other components are not ours
  // to report (a sticky device fault still resurfaces on our own calls)
  (void)cudaGetLastError();
  try {
    return f();
  } catch (const Error& e) {
    set_last_error(e.what());
    return e.code;
  } catch (const std::exception& e) {
    set_last_error(e.what());
    return SB_ERR_INVALID;
  }
}

}  // namespace sb
