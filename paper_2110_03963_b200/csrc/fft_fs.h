// fft_fs.h -- host interface of the fused-stage FFT passes (kernels_fft_fs.cu), used by the
// four-step / three-level circulant mixer in kernels_fft.cu (Sec. 3).
//
// The fused-stage passes compute the same row / column passes as the shared-memory Stockham
// engine of kernels_fft.cu, with fewer trips through shared memory: a transform's first stage
// reads its inputs straight from global memory into registers, its last stage writes its outputs
// straight from registers to global memory, and where one transform follows another inside a pass
// (row: forward -> spectrum -> inverse; column: inverse -> phase / <Q> -> forward) the last stage
// of the first and the first stage of the second run on the same registers (the second transform
// runs its radices in reverse order, so the element sets match).  DESIGN.md §7.2.
#pragma once

#include <cuda_runtime.h>
#include <stdint.h>

#include <vector>

namespace qva {

struct FsRowArgs {
    double2 *buf;               // rows of length n, row r at buf + r * n
    int row_off;                // global index of local row 0
    int row_mod;                // > 0: twiddle row index = row % row_mod (three-level inner rows)
    int spec;                   // 0: constant (e0 at bin 0 of global row 0, ec elsewhere); 1: real lambda
    const double *lam_perm;     // spec 1: transposed order, position row * n + k
    double beta, scale;         // spec 1: e = exp(-i beta lambda) * scale
    double2 ec, e0_over_ec;     // spec 0
    const double2 *tw;          // stage tables (fs_stage_tables order)
    const double2 *big_lo, *big_hi;  // final twiddle w_M^{-K x} = conj(hi[r >> s] lo[r & (2^s - 1)])
    int big_shift;
};

struct FsColArgs {
    const double2 *in;          // column block source (matrix base added per blockIdx.y)
    double2 *out;
    int M2;                     // row stride of the matrix (columns)
    int col_off, M2g;           // global index of local column 0 / global row stride (natural index)
    uint64_t mat_stride;        // blockIdx.y selects the matrix at this stride (three-level inner passes)
    int mat_off;                // global index of matrix 0 (outer twiddle K)
    int init;                   // 1: v = amp0 (no load; forward-only passes)
    int ops;                    // bit 1: <Q> partials, bit 2: phase, bit 64: outer twiddle (kernels_fft.cu OP_*)
    const double *q;            // qualities at local index x1 * M2 + column
    double amp0, gamma;
    double *partials;           // <Q> partial pairs, slot blockIdx.x
    const double2 *tw;          // stage tables
    const double2 *big_lo, *big_hi;  // forward store twiddle w_M^{C k1}
    int big_shift;
    const double2 *otw_lo, *otw_hi;  // outer twiddle w_N^{-x K}
    int otw_shift;
};

// A compiled fused-stage codelet of length n with its forward radix order (0-terminated).
bool fs_row_available(int n);
bool fs_col_available(int n);
// Stage twiddle tables of the length-n codelet: forward stages then inverse (pre-conjugated)
// stages, entry (t - 1) * m + k of a stage (m, R) = exp(-/+ 2 pi i t k / (m R)).
bool fs_stage_tables(int n, bool col, std::vector<double2> &tab);  // of the selected row / column codelet
// rows: n_rows rows (a multiple of fs_row_block(n)); one pass forward -> spectrum -> inverse ->
// final twiddle, in place
int fs_row_block(int n);
cudaError_t fs_row_launch(int n, const FsRowArgs &a, uint64_t n_rows, cudaStream_t s);
// columns: n = column length, cols = columns per matrix (multiple of fs_col_width(n)), nmat matrices;
// inv / fwd select the transforms (inverse -> ops -> forward)
cudaError_t fs_col_launch(int n, const FsColArgs &a, int cols, int nmat, bool inv, bool fwd, cudaStream_t s);
int fs_col_width(int n);  // columns per CTA of the length-n column codelet (0: none)

}  // namespace qva
