// Construction host driver (placeholder while the JIT kernels land).
#include "common.h"
#include "_jit_source.inc"
using namespace imp;
extern "C" int imp_build(const imp_build_desc* d, imp_imdp** out,
                         imp_build_stats* stats) {
  return guarded([&] { fail(IMP_E_ARG, "imp_build: not implemented yet"); });
}
