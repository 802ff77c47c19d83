// Error reporting + ABI version for the bastion C ABI.
#include <stdarg.h>

#include "common.cuh"

namespace bst {
static thread_local char g_err[1024] = "";

void set_error(const char* fmt, ...) {
  va_list ap;
  va_start(ap, fmt);
  vsnprintf(g_err, sizeof(g_err), fmt, ap);
  va_end(ap);
}
}  // namespace bst

extern "C" int bst_abi_version(void) { return 1; }
extern "C" const char* bst_last_error(void) { return bst::g_err; }
