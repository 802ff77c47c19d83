#include <stdlib.h>
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

namespace bst {
static thread_local bst_prefetch_t g_pf = {};
bst_prefetch_t take_prefetch() {
  bst_prefetch_t p = g_pf;
  g_pf = bst_prefetch_t{};
  return p;
}
}  // namespace bst

extern "C" int bst_set_prefetch(const bst_prefetch_t* pf) {
  bst::g_pf = pf ? *pf : bst_prefetch_t{};
  return BST_OK;
}

namespace bst {
int pdl_enabled() {
  static int v = -1;
  if (v < 0) {
    const char* e = getenv("BST_PDL");
    v = e ? atoi(e) : 1;
  }
  return v;
}
}  // namespace bst
