// Error plumbing and device queries of libsfw_b200.so.
#include <cuda_runtime.h>

#include <cstring>
#include <string>

#include "sfw_common.cuh"

namespace sfw {

static thread_local std::string g_last;

void set_error(int code, const std::string& msg) {
    (void)code;
    g_last = msg;
}

int fail(int code, const std::string& msg, char* errbuf, int errlen) {
    set_error(code, msg);
    if (errbuf && errlen > 0) {
        std::strncpy(errbuf, msg.c_str(), (size_t)errlen - 1);
        errbuf[errlen - 1] = 0;
    }
    return code;
}

}  // namespace sfw

extern "C" const char* sfw_last_error(void) { return sfw::g_last.c_str(); }

extern "C" int sfw_device_info(int* n_sm, char* name, int name_len) {
    int n = 0;
    if (cudaGetDeviceCount(&n) != cudaSuccess || n == 0) {
        cudaGetLastError();
        return -1;
    }
    int dev = 0;
    cudaGetDevice(&dev);
    cudaDeviceProp prop;
    if (cudaGetDeviceProperties(&prop, dev) != cudaSuccess) return -1;
    if (n_sm) *n_sm = prop.multiProcessorCount;
    if (name && name_len > 0) {
        std::strncpy(name, prop.name, (size_t)name_len - 1);
        name[name_len - 1] = 0;
    }
    return prop.major * 10 + prop.minor;
}
