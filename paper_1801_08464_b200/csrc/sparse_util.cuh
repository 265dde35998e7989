// Sparse-sparse host launchers (spgemm.cu).
#pragma once
#include "common.cuh"

namespace mg {
// C = A B, scipy csr_matmat semantics (exact zeros dropped, sorted columns)
// C = A B with scipy csr_matmat sums; sorted = false leaves each row's columns in
// hash-slot order (only for an intermediate consumed as the right factor of another
// product, whose sums do not depend on that order)
// b_unique: B's rows hold distinct columns (a product formed here), enabling the
// conflict-free one-B-row windows for long B rows
Csr spgemm(const Csr &a, const Csr &b, bool sorted = true, bool b_unique = false);
// variable-major scalar CSR (u = var * N + cell) -> cell-major b x b block CSR
Csr csr_varmajor_to_bsr(const Csr &a, int b);
// A^T with ascending columns per row
Csr transpose(const Csr &a);
// rows_dev: nr source rows (sorted); cmap_dev: column map (source col -> new col or -1)
Csr extract(const Csr &a, const int *rows_dev, int nr, const int *cmap_dev, int nc);
Csr copy_csr(const Csr &a);
// p[i] = i
void iota_i32(int *p, int64_t n);
void scale_i64(int64_t *a, int64_t s, int n);
}  // namespace mg
