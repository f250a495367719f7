// capi_util.h -- status helpers shared by capi.cu and comm.cu.
#pragma once
#include <cuda_runtime.h>

#include "internal.h"

namespace hack {
hack_status_t fail(hack_status_t st, const char* fmt, ...);
hack_status_t cuda_status(cudaError_t e, const char* where);
hack_status_t check_device();
hack_status_t make_kernel_cfg(const hack_config_t* c, KernelCfg* kc);
hack_status_t make_cache_view(const KernelCfg& kc, const hack_kv_cache_t* c, CacheView* cv);
}  // namespace hack
