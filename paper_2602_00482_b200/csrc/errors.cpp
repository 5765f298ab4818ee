// Thread-local last-error slot behind tt_last_error().
#include <string>

#include "capi_internal.h"

namespace ttb {
thread_local std::string g_last_error;
void set_last_error(const std::string& msg) { g_last_error = msg; }
}  // namespace ttb

extern "C" const char* tt_last_error(void) { return ttb::g_last_error.c_str(); }
