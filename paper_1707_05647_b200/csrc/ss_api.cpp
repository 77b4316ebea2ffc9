// ss_api.cpp -- diagnostics of the C ABI: thread-local last error, version,
// kernel-launch counter (observability for bench.py's gpu_launches).
#include <atomic>
#include <cstdarg>
#include <cstdio>

#include "../../include/starscreen_b200.h"

namespace ss {
namespace {
thread_local char g_last_error[1024] = "";
std::atomic<uint64_t> g_launches{0};
}  // namespace

void set_error(const char* fmt, ...) {
    va_list ap;
    va_start(ap, fmt);
    vsnprintf(g_last_error, sizeof(g_last_error), fmt, ap);
    va_end(ap);
}

void note_launch(uint64_t n) { g_launches.fetch_add(n, std::memory_order_relaxed); }
}  // namespace ss

extern "C" {
const char* ss_last_error(void) { return ss::g_last_error; }
int ss_version(void) { return 1; }
uint64_t ss_launch_count(void) { return ss::g_launches.load(std::memory_order_relaxed); }
}
