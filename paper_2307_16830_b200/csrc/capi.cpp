// Error reporting for the C-ABI (gridopf.h).
#include <string>

#include "internal.h"

namespace gn {
static thread_local std::string g_last_error;
void set_error(const std::string &msg) { g_last_error = msg; }
}  // namespace gn

extern "C" const char *gn_last_error(void) { return gn::g_last_error.c_str(); }
extern "C" int gn_version(void) { return 1; }
