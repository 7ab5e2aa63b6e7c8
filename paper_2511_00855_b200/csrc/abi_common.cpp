// abi_common.cpp — error state and device queries of the C-ABI.
#include <cuda_runtime.h>

#include <string>

#include "fg_internal.hpp"

namespace fgb {
namespace {
thread_local std::string t_code;
thread_local std::string t_what;
}  // namespace

void set_last_error(const std::string& code, const std::string& what) {
    t_code = code;
    t_what = what;
}
void clear_last_error() {
    t_code.clear();
    t_what.clear();
}

void HostTimer::mark(const char* what) {
    if (!on) return;
    if (mode() == 1) cudaDeviceSynchronize();
    const auto now = std::chrono::steady_clock::now();
    std::fprintf(stderr, "[host timing] %-14s %-26s %8.3f ms\n", scope, what,
                 std::chrono::duration<double, std::milli>(now - t).count());
    t = now;
}
}  // namespace fgb

extern "C" {

int fg_abi_version(void) { return FG_ABI_VERSION; }
const char* fg_last_error_code(void) { return fgb::t_code.c_str(); }
const char* fg_last_error_message(void) { return fgb::t_what.c_str(); }

int fg_device_count(int* count) {
    return fgb::guarded([&] {
        int n = 0;
        const cudaError_t e = cudaGetDeviceCount(&n);
        if (e != cudaSuccess) {
            cudaGetLastError();
            n = 0;
        }
        *count = n;
    });
}

}  // extern "C"
