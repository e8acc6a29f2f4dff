// abi.cu — error state, version, launch counter and grid sizes of the C ABI.

#include "common.cuh"

namespace nacc {

static thread_local std::string g_last_error;
static std::atomic<uint64_t> g_launches{0};

void set_error(const std::string &msg) { g_last_error = msg; }
void clear_error() { g_last_error.clear(); }
void count_launch(int n) { g_launches.fetch_add((uint64_t)n, std::memory_order_relaxed); }

}  // namespace nacc

extern "C" {

const char *nacc_last_error(void) { return nacc::g_last_error.c_str(); }
int nacc_abi_version(void) { return NACC_ABI_VERSION; }
uint64_t nacc_launch_count(void) { return nacc::g_launches.load(std::memory_order_relaxed); }

}  // extern "C"
