// Device producer of O (AceWavefunction.grad_theta_batch); see producer.cu.
#pragma once
#include <cuda_runtime.h>

#include <cstdint>

#include "engine.h"

namespace wssr {

size_t grad_theta_smem(const wssr_ace_spec& s, int tile);
int grad_theta_tile(const wssr_ace_spec& s);
// out [W x ldo]; *node_flag (device int) set when a walker sits on a node
cudaError_t grad_theta(Context& ctx, const wssr_ace_spec& s, const double* positions, int64_t W,
                       double* out, int64_t ldo, int* node_flag);

}  // namespace wssr
