// stencil_build.cuh -- K5: level-set stencil construction on the GPU (placeholder,
// filled in by the K5 milestone).
#pragma once
#include "ctx.h"

namespace pmghost {

template <int D, int N>
void run_stencil_build(Ctx&, const pmg_lsf_t*, int, const pmg_stencil_cfg_t*) {
  throw PmgError(PMG_ERR_INVALID_ARG, "build_stencils: GPU stencil build not available yet");
}

}  // namespace pmghost
