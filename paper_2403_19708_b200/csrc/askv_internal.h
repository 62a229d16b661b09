// Internal helpers shared by the C-ABI translation units.
#pragma once

#include <cuda_runtime.h>

#include <cstdarg>
#include <cstdio>
#include <string>

#include "../../include/askv.h"

namespace askv {

void set_error(const char* fmt, ...);
void clear_error();

inline int cuda_status(cudaError_t e, const char* what) {
  if (e == cudaSuccess) return ASKV_OK;
  set_error("%s: %s", what, cudaGetErrorString(e));
  return ASKV_ECUDA;
}

inline int launch_status(const char* what) { return cuda_status(cudaGetLastError(), what); }

#define ASKV_REQUIRE(cond, ...)          \
  do {                                   \
    if (!(cond)) {                       \
      ::askv::set_error(__VA_ARGS__);    \
      return ASKV_EINVAL;                \
    }                                    \
  } while (0)

}  // namespace askv
