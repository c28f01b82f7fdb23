// C-ABI error plumbing shared by every entry point of libppmoe.
#include <stdarg.h>
#include <stdlib.h>

#include "common.cuh"

namespace pp {

static thread_local std::string t_last_error;

void set_error(const std::string& msg) { t_last_error = msg; }

int fail(int code, const char* fmt, ...) {
  char buf[1024];
  va_list ap;
  va_start(ap, fmt);
  vsnprintf(buf, sizeof(buf), fmt, ap);
  va_end(ap);
  t_last_error = buf;
  return code;
}

// Off by default: measured no gain on the CUDA-graph step (cfg2, 1 B200: 9.77 M tokens/s with,
// 9.84-9.89 M without), and an early-launched dependent grid can take the SMs a gated GEMM
// leaves to the side-stream Trans/Agg kernels it waits on (deadlock in the EP parity runs).
bool pdl_enabled() {
  static const bool on = [] {
    const char* v = getenv("PPMOE_PDL");
    return v != nullptr && atoi(v) != 0;
  }();
  return on;
}

}  // namespace pp

extern "C" const char* pp_last_error(void) { return pp::t_last_error.c_str(); }

extern "C" int pp_version(void) { return 1; }
