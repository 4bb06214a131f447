// capi.cu -- error reporting and version of the C ABI (include/bsparse.h).
#include <stdarg.h>
#include <stdio.h>

#include "capi_util.cuh"

namespace as {
static thread_local char g_err[512] = "";
void set_error(const char* fmt, ...) {
  va_list ap;
  va_start(ap, fmt);
  vsnprintf(g_err, sizeof(g_err), fmt, ap);
  va_end(ap);
}
}  // namespace as

extern "C" {
const char* as_last_error(void) { return as::g_err; }
int as_abi_version(void) { return 1; }
}
