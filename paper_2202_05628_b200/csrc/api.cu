// Library identity, status strings and CUDA error plumbing for the C ABI.
#include <stdio.h>
#include <string.h>

#include "common.cuh"

namespace artemis {

static thread_local char g_last_error[256] = "";

void set_cuda_error(cudaError_t e) {
    snprintf(g_last_error, sizeof(g_last_error), "%s: %s", cudaGetErrorName(e),
             cudaGetErrorString(e));
}

int check_launch() {
    cudaError_t e = cudaGetLastError();
    if (e == cudaSuccess) return ARTEMIS_OK;
    set_cuda_error(e);
    return e == cudaErrorMemoryAllocation ? ARTEMIS_ERR_OOM : ARTEMIS_ERR_CUDA;
}

}  // namespace artemis

extern "C" const char *artemis_version(void) { return "libartemis 0.1.0 sm_100a"; }

extern "C" const char *artemis_status_string(int status) {
    switch (status) {
        case ARTEMIS_OK: return "ok";
        case ARTEMIS_ERR_ARG: return "invalid argument";
        case ARTEMIS_ERR_RANGE: return "grid coordinates outside [0, 2^21)";
        case ARTEMIS_ERR_EMPTY: return "empty leaf set";
        case ARTEMIS_ERR_DUPLICATE: return "duplicate Morton code";
        case ARTEMIS_ERR_OOM: return "out of device memory";
        case ARTEMIS_ERR_CUDA: return "CUDA error";
        case ARTEMIS_ERR_WORKSPACE: return "workspace too small";
        case ARTEMIS_ERR_NODEVICE: return "no sm_100 CUDA device";
        case ARTEMIS_ASSET_TRUNCATED_HEADER: return "file ends inside header";
        case ARTEMIS_ASSET_BAD_MAGIC: return "magic mismatch (expected NVO1)";
        case ARTEMIS_ASSET_BAD_VERSION: return "unsupported container version";
        case ARTEMIS_ASSET_ZERO_COUNT: return "declared voxel count is zero";
        case ARTEMIS_ASSET_TRUNCATED_LEAVES: return "file ends inside leaf table";
        case ARTEMIS_ASSET_TRUNCATED_FLUT: return "file ends inside FLUT block";
        case ARTEMIS_ASSET_RIG_OFFSET: return "rig offset does not follow the FLUT block";
        case ARTEMIS_ASSET_TRUNCATED_RIG: return "file ends inside rig block";
        case ARTEMIS_ASSET_TRAILING: return "trailing bytes after the asset";
        default: return "unknown status";
    }
}

extern "C" const char *artemis_last_cuda_error(void) { return artemis::g_last_error; }

extern "C" int artemis_device_ok(void) {
    int n = 0;
    if (cudaGetDeviceCount(&n) != cudaSuccess || n < 1) {
        cudaGetLastError();
        return 0;
    }
    int dev = 0, major = 0;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&major, cudaDevAttrComputeCapabilityMajor, dev);
    return major == 10 ? 1 : 0;
}

// Synchronous device -> host copy of `bytes` (parity helpers read the
// frame pipeline's internal buffers through this).
extern "C" int artemis_copy_to_host(void *dst, const void *src, size_t bytes,
                                    artemis_stream stream) {
    if (!bytes) return ARTEMIS_OK;
    if (!dst || !src) return ARTEMIS_ERR_ARG;
    cudaError_t e = cudaMemcpyAsync(dst, src, bytes, cudaMemcpyDeviceToHost,
                                    reinterpret_cast<cudaStream_t>(stream));
    if (e == cudaSuccess) e = cudaStreamSynchronize(reinterpret_cast<cudaStream_t>(stream));
    if (e != cudaSuccess) {
        artemis::set_cuda_error(e);
        return ARTEMIS_ERR_CUDA;
    }
    return ARTEMIS_OK;
}
