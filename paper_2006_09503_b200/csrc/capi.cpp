// Library-level C-ABI: error reporting and version.
#include <string>

#include "capi_internal.h"
#include "p2bw.h"

namespace p2bw {
namespace {
thread_local std::string g_last_error;
}
void set_last_error(const std::string& msg) { g_last_error = msg; }
}  // namespace p2bw

extern "C" const char* p2bw_last_error(void) { return p2bw::g_last_error.c_str(); }

extern "C" const char* p2bw_version(void) { return "p2bw 0.1 (sm_100a)"; }
