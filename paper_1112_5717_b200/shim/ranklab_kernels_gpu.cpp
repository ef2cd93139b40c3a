// ranklab_kernels_gpu.cpp -- the library's declared substitution seam on the
// B200 path: ranklab::mm (proj/include/ranklab/kernels.hpp:26-27, "a faster
// kernel can replace the implementation behind this exact contract",
// kernels.hpp:13-19) and ranklab::trsm (kernels.hpp:37-38), through the C ABI
// (rl_mm_u32 / rl_trsm_u32, include/ranklab_gpu.h).
//
// Link this translation unit in place of the reference's definitions: build
// kernels.cpp with -Dmm=mm_reference_cpu -Dtrsm=trsm_reference_cpu.
// Every caller in the other translation units -- trtri/trulm/trlum (tri.cpp),
// in_place_mm / solve (solvers.cpp), the echelon forms (echelon.cpp), selfcheck,
// the CLI -- then multiplies and solves on the GPU.  (trmm lives in kernels.cpp
// itself and keeps its calls to the renamed CPU mm; it is out of scope,
// SURVEY.md 2.)
//
// Contract kept: dimension checks and messages of kernels.cpp:8-40, C must not
// overlap A or B (OverlapError), T must not overlap B, Unit never reads the
// diagonal, NonUnit throws SingularDiagonal(index) before touching B, the
// OpCounter charged exactly as the reference at the given threshold, any stride,
// degenerate views are no-ops.  Allocation budget (kernels.hpp:16-17): device
// workspaces of the calling thread's context, no ranklab::Mat.
#include <algorithm>
#include <cstdint>
#include <string>

#include "ranklab/kernels.hpp"
#include "ranklab_gpu.h"
#include "rl_errors.hpp"

namespace ranklab {

namespace {

// ConstMatView exposes no pointer; its window (allocation, stride, origin) is
// read through pointers-to-member formed in a derived class (matrix.hpp:32-67).
struct Peek : ConstMatView {
    static const Elem* base(const ConstMatView& v) {
        if (v.empty()) return nullptr;
        const Elem* ConstMatView::*alloc = &Peek::alloc_;
        std::size_t ConstMatView::*stride = &Peek::stride_;
        std::size_t ConstMatView::*r0 = &Peek::r0_;
        std::size_t ConstMatView::*c0 = &Peek::c0_;
        return v.*alloc + (v.*r0) * (v.*stride) + v.*c0;
    }
    static std::int64_t stride(const ConstMatView& v) {
        std::size_t ConstMatView::*s = &Peek::stride_;
        const std::size_t st = v.*s;
        return static_cast<std::int64_t>(st ? st : 1);
    }
};
const std::uint32_t* base_of(const ConstMatView& a) { return Peek::base(a); }
std::int64_t stride_of(const ConstMatView& a) {
    return a.empty() ? std::max<std::int64_t>(1, (std::int64_t)a.cols()) : Peek::stride(a);
}

void charge(OpCounter& ctr, const std::uint64_t ops[4]) {
    ctr.n_mul += ops[0];
    ctr.n_addsub += ops[1];
    ctr.n_divinv += ops[2];
    ctr.n_ztest += ops[3];
}

}  // namespace

void mm(ConstMatView a, ConstMatView b, MatView c, Elem alpha, Elem beta, OpCounter& ctr) {
    const std::size_t m = c.rows(), n = c.cols(), l = a.cols();
    if (a.rows() != m || b.rows() != l || b.cols() != n)  // kernels.cpp:32-37
        throw DimensionMismatch("mm " + std::to_string(a.rows()) + "x" + std::to_string(a.cols()) +
                                " * " + std::to_string(b.rows()) + "x" + std::to_string(b.cols()) +
                                " -> " + std::to_string(m) + "x" + std::to_string(n));
    if (a.overlaps(c)) throw OverlapError("mm: C overlaps A");  // kernels.cpp:38-39
    if (b.overlaps(c)) throw OverlapError("mm: C overlaps B");
    std::uint64_t ops[4] = {0, 0, 0, 0};
    const int st = rl_mm_u32(base_of(a), stride_of(a), base_of(b), stride_of(b),
                             const_cast<std::uint32_t*>(base_of(c)), stride_of(c), (std::int64_t)m, (std::int64_t)l,
                             (std::int64_t)n, alpha, beta, c.field().modulus(), ops);
    if (st != RL_OK) gpu_shim::rethrow(st, "rl_mm_u32", c.field().modulus());
    charge(ctr, ops);
}

void trsm(Side side, UpLo uplo, Diag diag, ConstMatView t, MatView b, OpCounter& ctr, std::size_t threshold) {
    if (t.rows() != t.cols())  // kernels.cpp:10-13
        throw DimensionMismatch("triangular operand is " + std::to_string(t.rows()) + "x" +
                                std::to_string(t.cols()));
    const std::size_t need = side == Side::Left ? b.rows() : b.cols();
    if (t.rows() != need)  // kernels.cpp:16-20
        throw DimensionMismatch("triangular side " + std::to_string(t.rows()) + " vs operand dimension " +
                                std::to_string(need));
    if (t.overlaps(b)) throw OverlapError("trsm: T overlaps B");
    if (threshold == 0) threshold = 1;
    std::uint64_t ops[4] = {0, 0, 0, 0};
    const int st = rl_trsm_u32(side == Side::Right ? 1 : 0, uplo == UpLo::Lower ? 1 : 0,
                               diag == Diag::Unit ? 1 : 0, base_of(t), stride_of(t),
                               const_cast<std::uint32_t*>(base_of(b)), stride_of(b), (std::int64_t)b.rows(),
                               (std::int64_t)b.cols(), b.field().modulus(), (std::int64_t)threshold, ops);
    if (st != RL_OK) gpu_shim::rethrow(st, "rl_trsm_u32", b.field().modulus());
    charge(ctr, ops);
}

}  // namespace ranklab
