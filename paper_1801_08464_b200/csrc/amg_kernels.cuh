// AMG setup launchers (amg_setup.cu).
#pragma once
#include "common.cuh"
namespace mg {
void row_diag(const Csr &a, double *d);
// flips rows with negative diagonal (dropping exact zeros like diags @ csr);
// returns false (and leaves out/sgn empty) when no row has a negative diagonal.
// Throws MG_ERR_AMG_SETUP on a zero diagonal.
bool sign_normalise(const Csr &a, Csr &out, DBuf<double> &sgn);
// strength mask aligned with a's entries; returns the number of strong entries
int64_t strength(const Csr &a, double theta, DBuf<int8_t> &s);
// PMIS C/F splitting (0 undecided, 1 F, 2 C); returns the number of rounds
int pmis(const Csr &a, const int8_t *s, uint64_t seed, int level, DBuf<int8_t> &state);
// coarse index of each C point (-1 for F); returns nc
int coarse_map(const int8_t *state, int n, DBuf<int> &cmap);
Csr ext_interp(const Csr &a, const int8_t *s, const int8_t *state, const int *cmap, int nc, int max_elmts);
void l1_inverse(const Csr &a, double *dinv);
void to_dense(const Csr &a, double *d);
}  // namespace mg
