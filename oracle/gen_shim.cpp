// gen_shim.cpp -- TEST INFRASTRUCTURE (see sssp_oracle.c header).
//
// liboracle.so carries its own copy of the reference-compatible graph generators
// (paper_2602_10080_b200/csrc/host/generators.cpp, a restatement of the reference's
// graph.py:306-420 pinned by the reference-produced csr_sha256 values), so that the
// bench's CPU reference arm and the test checkers never map the product library.
// This file supplies the error hook the generator source reports through.
#include <cstdarg>
#include <cstdio>

static thread_local char g_oracle_err[512];

namespace mlmq {
void set_last_error(const char* fmt, ...) {
  va_list ap;
  va_start(ap, fmt);
  vsnprintf(g_oracle_err, sizeof(g_oracle_err), fmt, ap);
  va_end(ap);
}
}  // namespace mlmq

extern "C" const char* oracle_last_error(void) { return g_oracle_err; }
