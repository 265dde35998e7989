// Per-cell block scaling launchers (blockscale.cu).
#pragma once
#include "common.cuh"
namespace mg {
// dinv: block-diagonal BSR (N blocks); ahat: scalar CSR cell-major
void block_scale(const Csr &a, Csr &dinv, Csr &ahat, bool equilibrate);
void block_apply(const Csr &dinv, const double *x, double *z);
}  // namespace mg
