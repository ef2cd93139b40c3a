// ranklab_cup_gpu.cpp -- the drop-in: ranklab::cup (proj/include/ranklab/factor.hpp:34)
// and its mirror ranklab::ple (factor.hpp:37)
// implemented on the B200 path through the C ABI (include/ranklab_gpu.h).
//
// Link this translation unit in place of the reference's definition of cup (build
// factor.cpp with -Dcup=cup_reference_cpu -Dple=ple_reference_cpu): every caller --
// rank_and_profile, determinant, solve, col_ech_trans, in_place_mm, selfcheck, the
// CLI, the acceptance suite -- then runs its CUP on the GPU, unchanged.
// Contract kept: in place on the caller's MatView (any stride), any shape incl.
// empty (factor.cpp:32), rank deficiency is an output, OpCounter charged exactly as
// the reference would, errors rethrown as ranklab::Error.
#include <algorithm>
#include <cstdint>
#include <string>
#include <vector>

#include "ranklab/factor.hpp"
#include "ranklab_gpu.h"
#include "rl_errors.hpp"

namespace ranklab {

PackedCup cup(MatView a, OpCounter& ctr) {
    const std::size_t m = a.rows(), n = a.cols();
    PackedCup out;
    out.col_perm = Perm(n);
    if (m == 0 || n == 0) return out;
    std::uint32_t* base = &a(0, 0);
    const std::int64_t lda = m > 1 ? static_cast<std::int64_t>(&a(1, 0) - &a(0, 0))
                                   : static_cast<std::int64_t>(n);
    std::int64_t rank = 0;
    std::vector<std::uint32_t> rrp(std::min(m, n)), sigma(n);
    std::uint64_t ops[4] = {0, 0, 0, 0};
    const int st = rl_cup_u32(base, static_cast<std::int64_t>(m), static_cast<std::int64_t>(n),
                              lda, a.field().modulus(), &rank, rrp.data(), sigma.data(), ops);
    if (st != RL_OK) gpu_shim::rethrow(st, "rl_cup_u32", a.field().modulus());
    ctr.n_mul += ops[0];
    ctr.n_addsub += ops[1];
    ctr.n_divinv += ops[2];
    ctr.n_ztest += ops[3];
    out.rank = static_cast<std::size_t>(rank);
    rrp.resize(out.rank);
    out.row_profile = std::move(rrp);
    out.col_perm = Perm(std::move(sigma));
    return out;
}

// ranklab::ple (factor.hpp:37), cup's column-split mirror, through rl_ple_u32
// (computed as cup(A^T)^T on the device).  Same contract; factor.cpp is then
// built with -Dple=ple_reference_cpu as well.
PackedPle ple(MatView a, OpCounter& ctr) {
    const std::size_t m = a.rows(), n = a.cols();
    PackedPle out;
    out.row_perm = Perm(m);
    if (m == 0 || n == 0) return out;
    std::uint32_t* base = &a(0, 0);
    const std::int64_t lda = m > 1 ? static_cast<std::int64_t>(&a(1, 0) - &a(0, 0))
                                   : static_cast<std::int64_t>(n);
    std::int64_t rank = 0;
    std::vector<std::uint32_t> prof(std::min(m, n)), perm(m);
    std::uint64_t ops[4] = {0, 0, 0, 0};
    const int st = rl_ple_u32(base, static_cast<std::int64_t>(m), static_cast<std::int64_t>(n),
                              lda, a.field().modulus(), &rank, prof.data(), perm.data(), ops);
    if (st != RL_OK) gpu_shim::rethrow(st, "rl_ple_u32", a.field().modulus());
    ctr.n_mul += ops[0];
    ctr.n_addsub += ops[1];
    ctr.n_divinv += ops[2];
    ctr.n_ztest += ops[3];
    out.rank = static_cast<std::size_t>(rank);
    prof.resize(out.rank);
    out.col_profile = std::move(prof);
    out.row_perm = Perm(std::move(perm));
    return out;
}

}  // namespace ranklab
