// strait_capi.cuh — error reporting shared by the C-ABI entry points.
#pragma once

#include <cuda_runtime.h>
#include <stdint.h>

#include "../../include/strait.h"

namespace strait {

// Record a thread-local message (strait_last_error) and return `code`.
int set_error(int code, const char* fmt, ...);
// After a launch: map a pending CUDA error to STRAIT_ECUDA and count the launch.
int check_launch(const char* what);

}  // namespace strait
