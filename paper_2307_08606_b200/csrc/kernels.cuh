// sm_100a kernels of the ASADMM iteration loop.
//
// Data layout in HBM:
//   * A_q        complex64, column-major, leading dimension ld_q =
//                roundup(rows_q, 64) (zero-padded rows), so every pixel's
//                column is a 512-B aligned contiguous run.  Never moved:
//                elimination compacts the index list J_q instead and every
//                matvec streams only the active columns A(:, J_q).
//   * G_q        complex128 inverse of the rows x rows capacitance
//                beta I + mu A_J A_J^H (dual form) or of the N_q x N_q
//                Gram mu A_J^H A_J + beta I (primal form), column-major.
//   * solver state (x_full, x_hat, rhs, data, s, x_G, sigma, gap) complex128;
//     screening ring of |x_k - x_{k-1}|, W x N doubles per sensor.
// Arithmetic: A is promoted to fp64 in registers; all products and sums are
// fp64 (the fp64 oracle sees the very same complex64 operator values).
#pragma once
#include <cuda_runtime.h>
#include <stdint.h>


// The kernels live in topical headers, included in dependency order.
#include "kernels_async.cuh"
#include "kernels_matvec.cuh"
#include "kernels_dense.cuh"
#include "kernels_batched.cuh"
#if RADMM_EXPERIMENTAL
#include "kernels_fused.cuh"  // parked single-pass sweeps (not shipped)
#endif
#include "kernels_ozaki.cuh"
