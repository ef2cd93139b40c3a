// dist.cu -- data-plane kernels of the multi-GPU single-matrix CUP
// (paper_1112_5717_b200/dist.py, config 5: 1D block-cyclic column tiles).
//
// The collectives move rows x columns pieces of the ranks' local matrices.
// Each kernel is one pass over HBM (coalesced: consecutive threads take
// consecutive columns of a row):
//   * pack:   a strided piece into a contiguous wire buffer; for p <= 2^16 the
//             wire carries 16-bit words x - 2^15 (half the NVLink volume);
//   * unpack: a received wire piece into its global columns of a gathered
//             block (column map minus an offset), undoing the 16-bit offset;
//   * select: a gathered block's columns owned by this rank back into the
//             local matrix (column map);
//   * shift:  the U-row move of factor.cpp:62-70 applied per row block on this
//             rank's columns (row i0 + j -> row r + j where the global column is
//             beyond r + j, the vacated entries zeroed), one thread per column
//             walking j upward so overlapping source/target rows stay exact.
#include <algorithm>

#include "kernels.cuh"
#include "runtime.h"

namespace rl {
namespace {

constexpr int TX = 256;

__global__ void pack_kernel_d(const u32* __restrict__ src, i64 lds, i64 rows, i64 cols, int wire16,
                              void* __restrict__ dst) {
    const i64 c = (i64)blockIdx.x * TX + threadIdx.x;
    if (c >= cols) return;
    for (i64 r = blockIdx.y; r < rows; r += gridDim.y) {
        const u32 v = __ldcs(src + r * lds + c);
        if (wire16) static_cast<int16_t*>(dst)[r * cols + c] = (int16_t)((i32)v - 32768);
        else static_cast<u32*>(dst)[r * cols + c] = v;
    }
}

__global__ void unpack_kernel_d(const void* __restrict__ src, i64 rows, i64 cols, int wire16,
                                u32* __restrict__ dst, i64 ldd, const i64* __restrict__ colmap, i64 off) {
    const i64 c = (i64)blockIdx.x * TX + threadIdx.x;
    if (c >= cols) return;
    const i64 dc = colmap ? colmap[c] - off : c;
    for (i64 r = blockIdx.y; r < rows; r += gridDim.y) {
        const u32 v = wire16 ? (u32)((i32) static_cast<const int16_t*>(src)[r * cols + c] + 32768)
                             : static_cast<const u32*>(src)[r * cols + c];
        dst[r * ldd + dc] = v;
    }
}

__global__ void select_kernel_d(const u32* __restrict__ src, i64 lds, i64 rows, const i64* __restrict__ colmap,
                                i64 off, i64 cols, u32* __restrict__ dst, i64 ldd) {
    const i64 c = (i64)blockIdx.x * TX + threadIdx.x;
    if (c >= cols) return;
    const i64 sc = colmap[c] - off;
    for (i64 r = blockIdx.y; r < rows; r += gridDim.y) dst[r * ldd + c] = src[r * lds + sc];
}

__global__ void shift_kernel_d(u32* __restrict__ x, i64 ldx, i64 cols, i64 r, i64 i0, i64 rt,
                               const i64* __restrict__ gpos) {
    const i64 l = (i64)blockIdx.x * TX + threadIdx.x;
    if (l >= cols) return;
    const i64 J = min(rt, max((i64)0, gpos[l] - r));  // rows j with r + j < gpos[l]
    for (i64 j = 0; j < J; ++j) {
        x[(r + j) * ldx + l] = x[(i0 + j) * ldx + l];
        x[(i0 + j) * ldx + l] = 0;
    }
}

dim3 grid_for(i64 rows, i64 cols) {
    const unsigned gx = (unsigned)((cols + TX - 1) / TX);
    const unsigned gy = (unsigned)std::min<i64>(std::max<i64>(rows, 1), std::max<i64>(1, 4096 / std::max(1u, gx)));
    return dim3(gx, gy);
}

}  // namespace

void dist_pack(const u32* src, i64 lds, i64 rows, i64 cols, int wire16, void* dst, cudaStream_t s) {
    if (rows <= 0 || cols <= 0) return;
    pack_kernel_d<<<grid_for(rows, cols), TX, 0, s>>>(src, lds, rows, cols, wire16, dst);
    RL_CUDA_CHECK(cudaGetLastError());
}
void dist_unpack(const void* src, i64 rows, i64 cols, int wire16, u32* dst, i64 ldd, const i64* colmap, i64 off,
                 cudaStream_t s) {
    if (rows <= 0 || cols <= 0) return;
    unpack_kernel_d<<<grid_for(rows, cols), TX, 0, s>>>(src, rows, cols, wire16, dst, ldd, colmap, off);
    RL_CUDA_CHECK(cudaGetLastError());
}
void dist_select(const u32* src, i64 lds, i64 rows, const i64* colmap, i64 off, i64 cols, u32* dst, i64 ldd,
                 cudaStream_t s) {
    if (rows <= 0 || cols <= 0) return;
    select_kernel_d<<<grid_for(rows, cols), TX, 0, s>>>(src, lds, rows, colmap, off, cols, dst, ldd);
    RL_CUDA_CHECK(cudaGetLastError());
}
void dist_shift_u_rows(u32* x, i64 ldx, i64 cols, i64 r, i64 i0, i64 rt, const i64* gpos, cudaStream_t s) {
    if (cols <= 0 || rt <= 0 || i0 == r) return;
    shift_kernel_d<<<(unsigned)((cols + TX - 1) / TX), TX, 0, s>>>(x, ldx, cols, r, i0, rt, gpos);
    RL_CUDA_CHECK(cudaGetLastError());
}

}  // namespace rl
