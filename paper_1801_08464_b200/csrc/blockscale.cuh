// Per-cell block scaling launchers (blockscale.cu).
#pragma once
#include "common.cuh"
namespace mg {
// dinv: block-diagonal BSR (N blocks); ahat: scalar CSR cell-major
void block_scale(const Csr &a, Csr &dinv, Csr &ahat, bool equilibrate);
void block_apply(const Csr &dinv, const double *x, double *z);
// the same with the input read through a device-resident pointer slot (CUDA-graph
// replays of the MGR apply take a new input without a copy: see mgr_apply)
void block_apply_indirect(const Csr &dinv, const double *const *xslot, double *z);
void set_device_ptr(const double **slot, const double *value);
// symmetric infinity-norm equilibration (linsolve.py:107-122): row = row abs max
// (0 -> 1), colscale = 1 / col abs max of diag(1/row)|A| (0 -> 1), out = the
// scaled matrix with exact zeros dropped
void equilibrate(const Csr &a, Csr &out, double *row_dev, double *colscale_dev);
// max_i sum_j |a_ij|  (the a_norm GmresSolver passes to gmres, linsolve.py:98)
double abs_row_sum_max(const Csr &a);
}  // namespace mg
