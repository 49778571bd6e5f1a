// Library-level entry points: version, thread-local error text, device info.
#include <cstdarg>
#include <cstdio>
#include <cstring>

#include "common.cuh"

namespace nao {

static thread_local char g_err[1024] = {0};

void set_error(const char* fmt, ...) {
    va_list ap;
    va_start(ap, fmt);
    vsnprintf(g_err, sizeof g_err, fmt, ap);
    va_end(ap);
}

}  // namespace nao

extern "C" {

int nao_version(void) { return 1; }

int nao_last_error(char* buf, size_t buf_len) {
    size_t n = strlen(nao::g_err);
    if (buf && buf_len) {
        size_t c = n < buf_len - 1 ? n : buf_len - 1;
        memcpy(buf, nao::g_err, c);
        buf[c] = 0;
    }
    return (int)n;
}

int nao_device_info(int* sm_count, int* cc_major, int* cc_minor) {
    int dev = 0;
    NAO_CHECK_CUDA(cudaGetDevice(&dev));
    NAO_CHECK_CUDA(cudaDeviceGetAttribute(sm_count, cudaDevAttrMultiProcessorCount, dev));
    NAO_CHECK_CUDA(cudaDeviceGetAttribute(cc_major, cudaDevAttrComputeCapabilityMajor, dev));
    NAO_CHECK_CUDA(cudaDeviceGetAttribute(cc_minor, cudaDevAttrComputeCapabilityMinor, dev));
    return NAO_OK;
}

}  // extern "C"
