// dh status plumbing: thread-local last-error message behind dh_last_error().
#include <string>

#include "common.cuh"
#include "dh_capi.h"

namespace dh {

namespace {
thread_local std::string g_last_error;
}

int set_error(int code, const char* msg) {
    g_last_error = msg ? msg : "";
    return code;
}

int set_cuda_error(cudaError_t e, const char* what, const char* file, int line) {
    g_last_error = std::string(cudaGetErrorString(e)) + " at " + what + " (" + file + ":" +
                   std::to_string(line) + ")";
    return DH_ERR_CUDA;
}

}  // namespace dh

extern "C" const char* dh_last_error(void) { return dh::g_last_error.c_str(); }

extern "C" int dh_version(void) { return 1; }
