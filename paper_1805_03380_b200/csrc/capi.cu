// capi.cu -- error reporting and version of the C ABI (include/bsparse.h).
#include <stdarg.h>
#include <stdio.h>

#include "capi_util.cuh"

namespace as {
int g_engine = 0;  // as_set_engine
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
int as_set_engine(int engine) {
  if (engine < 0 || engine > 2) {
    as::set_error("engine must be 0, 1 or 2, got %d", engine);
    return AS_ERR_ARG;
  }
  as::g_engine = engine;
  return AS_OK;
}
}
