// Error state and launch accounting for the C-ABI (p2r_last_error etc.).
#include <atomic>
#include <cstdio>
#include <string>

#include "p2r_internal.h"

namespace p2r {

namespace {
thread_local std::string g_last_error;
std::atomic<uint64_t> g_launches{0};
}  // namespace

p2r_status set_error(p2r_status code, const char* msg) {
  g_last_error = msg ? msg : "";
  return code;
}

p2r_status set_cuda_error(cudaError_t e, const char* where) {
  g_last_error = std::string(where) + ": " + cudaGetErrorString(e);
  return P2R_ECUDA;
}

void count_launch() { g_launches.fetch_add(1, std::memory_order_relaxed); }
void count_launches(uint64_t n) { g_launches.fetch_add(n, std::memory_order_relaxed); }

}  // namespace p2r

extern "C" const char* p2r_last_error(void) { return p2r::g_last_error.c_str(); }
extern "C" const char* p2r_version(void) { return "p2r-b200 0.1 sm_100a"; }
extern "C" uint64_t p2r_launch_count(void) { return p2r::g_launches.load(); }
