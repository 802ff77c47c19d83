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

namespace bst {
// launch sequence numbers for boundary tracing (host side; 0 = untraced)
static int g_bnd_seq = 0;
int bnd_next_seq() {
#ifdef BST_TRACE
  return (++g_bnd_seq) % 4096;
#else
  return 0;
#endif
}
void bnd_reset_seq() { g_bnd_seq = 0; }
}  // namespace bst

extern "C" int bst_debug_bnd_reset(void) {  // restart the boundary-trace launch numbering
  bst::bnd_reset_seq();
  return BST_OK;
}
