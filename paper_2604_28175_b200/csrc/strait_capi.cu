// strait_capi.cu — library-wide C-ABI plumbing: version, thread-local error
// message, and the launch counter used as evidence that the device path ran.
#include <cuda_runtime.h>

#include <atomic>
#include <cmath>
#include <cstdarg>
#include <cstdio>

#include "strait_capi.cuh"
#include "../../include/strait_node.h"
#include "../../include/strait_replay.h"

namespace {
thread_local char g_err[1024] = "";
std::atomic<int64_t> g_launches{0};
}  // namespace

namespace strait {

int set_error(int code, const char* fmt, ...) {
  va_list ap;
  va_start(ap, fmt);
  vsnprintf(g_err, sizeof g_err, fmt, ap);
  va_end(ap);
  return code;
}

int check_launch(const char* what) {
  cudaError_t e = cudaGetLastError();
  if (e != cudaSuccess) return set_error(STRAIT_ECUDA, "%s: %s", what, cudaGetErrorString(e));
  g_launches.fetch_add(1, std::memory_order_relaxed);
  return STRAIT_OK;
}

}  // namespace strait

extern "C" int strait_abi_version(void) { return STRAIT_ABI_VERSION; }
extern "C" int64_t strait_struct_size(int32_t id) {
  switch (id) {
    case 0: return sizeof(StraitSweepArgs);
    case 1: return sizeof(StraitSweepExpandArgs);
    case 2: return sizeof(StraitRefitArgs);
    case 3: return sizeof(StraitReplayModels);
    case 4: return sizeof(StraitReplayConfig);
    case 5: return sizeof(StraitReplayArgs);
    case 6: return sizeof(StraitTraceRec);
    case 7: return sizeof(StraitMetricsArgs);
    case 8: return sizeof(StraitStreamSpec);
    case 9: return sizeof(StraitGroundTruth);
    case 10: return sizeof(StraitGpuHdr);
    case 11: return sizeof(StraitNodeEntry);
    case 12: return sizeof(StraitProposeArgs);
    case 13: return sizeof(StraitProposeOut);
  }
  return -1;
}
extern "C" const char* strait_last_error(void) { return g_err; }
extern "C" int64_t strait_kernel_launches(void) { return g_launches.load(); }
