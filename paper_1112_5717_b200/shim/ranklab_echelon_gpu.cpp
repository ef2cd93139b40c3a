// ranklab_echelon_gpu.cpp -- the drop-in for the reductions after cup:
//   ranklab::col_ech_trans / red_col_ech_trans   proj/include/ranklab/echelon.hpp:28-29
//   ranklab::invert_in_place                     proj/include/ranklab/solvers.hpp:22
// on the B200 path through the C ABI (include/ranklab_gpu.h).
//
// Link in place of the reference definitions: build echelon.cpp with
// -Dcol_ech_trans=col_ech_trans_reference_cpu
// -Dred_col_ech_trans=red_col_ech_trans_reference_cpu and solvers.cpp with
// -Dinvert_in_place=invert_in_place_reference_cpu.  Same
// contract: in place on the caller's MatView, OpCounter charged exactly as the
// reference, SingularMatrix from invert_in_place with the body left as
// red_col_ech_trans produced it, no ranklab::Mat allocated.
#include <algorithm>
#include <cstdint>
#include <string>
#include <vector>

#include "ranklab/echelon.hpp"
#include "ranklab/errors.hpp"
#include "ranklab/solvers.hpp"
#include "ranklab_gpu.h"
#include "rl_errors.hpp"

namespace ranklab {

namespace {

std::int64_t stride_of(MatView a) {
    return a.rows() > 1 ? static_cast<std::int64_t>(&a(1, 0) - &a(0, 0))
                        : static_cast<std::int64_t>(a.cols());
}

void charge(OpCounter& ctr, const std::uint64_t ops[4]) {
    ctr.n_mul += ops[0];
    ctr.n_addsub += ops[1];
    ctr.n_divinv += ops[2];
    ctr.n_ztest += ops[3];
}

template <class T>
T echelon(MatView a, OpCounter& ctr, int reduced) {
    const std::size_t m = a.rows(), n = a.cols();
    T out;
    out.col_perm = Perm(n);
    if (m == 0 || n == 0) return out;
    std::int64_t rank = 0;
    std::vector<std::uint32_t> rrp(std::min(m, n)), sigma(n);
    std::uint64_t ops[4] = {0, 0, 0, 0};
    const int st = rl_col_ech_trans_u32(&a(0, 0), static_cast<std::int64_t>(m),
                                        static_cast<std::int64_t>(n), stride_of(a),
                                        a.field().modulus(), reduced, &rank, rrp.data(),
                                        sigma.data(), ops);
    if (st != RL_OK) gpu_shim::rethrow(st, "rl_col_ech_trans_u32", a.field().modulus());
    charge(ctr, ops);
    out.rank = static_cast<std::size_t>(rank);
    rrp.resize(out.rank);
    out.row_profile = std::move(rrp);
    out.col_perm = Perm(std::move(sigma));
    return out;
}

}  // namespace

EchelonTransform col_ech_trans(MatView a, OpCounter& ctr) {
    return echelon<EchelonTransform>(a, ctr, 0);
}

ReducedEchelonTransform red_col_ech_trans(MatView a, OpCounter& ctr) {
    return echelon<ReducedEchelonTransform>(a, ctr, 1);
}

void invert_in_place(MatView a, OpCounter& ctr) {
    const std::size_t n = a.rows();
    if (a.cols() != n) throw DimensionMismatch("inverse of non-square matrix");
    if (n == 0) return;
    std::uint64_t ops[4] = {0, 0, 0, 0};
    const int st = rl_invert_u32(&a(0, 0), static_cast<std::int64_t>(n), stride_of(a),
                                 a.field().modulus(), ops);
    charge(ctr, ops);
    if (st != RL_OK) gpu_shim::rethrow(st, "rl_invert_u32", a.field().modulus());
}

}  // namespace ranklab
