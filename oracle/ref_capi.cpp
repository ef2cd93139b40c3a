// oracle/ref_capi.cpp -- C entry points over the UNMODIFIED reference library.
//
// TEST INFRASTRUCTURE ONLY (parity checker and the bench's reference arm).
// Compiled by oracle/Makefile together with /root/reference/proj/src/*.cpp
// into oracle/_ref/libranklab_ref.so; nothing from the reference is copied
// into this repository.  Every function forwards to the reference's own
// public API on a MatView over the caller's buffer:
//   ranklab::cup / ple         proj/include/ranklab/factor.hpp:34-37
//   ranklab::mm / trsm         proj/include/ranklab/kernels.hpp:26-38
//   ranklab::rank_and_profile  proj/include/ranklab/solvers.hpp:13
//   ranklab::determinant       proj/include/ranklab/solvers.hpp:16
//   ranklab::invert_in_place   proj/include/ranklab/solvers.hpp:22
//   ranklab::col_ech_trans / red_col_ech_trans  proj/include/ranklab/echelon.hpp:28-29
//   ranklab::random_matrix / random_rank_matrix / random_nonsingular_matrix /
//   random_triangular_matrix / SplitMix64 / naive_gauss
//                              proj/include/ranklab/reference.hpp
#include <cstdint>
#include <cstring>
#include <exception>

#include "ranklab/echelon.hpp"
#include "ranklab/factor.hpp"
#include "ranklab/kernels.hpp"
#include "ranklab/reference.hpp"
#include "ranklab/solvers.hpp"

using namespace ranklab;

namespace {

enum : int {
    REF_OK = 0,
    REF_EDIM = 1,
    REF_EOVERLAP = 2,
    REF_ESINGULAR = 3,
    REF_EFIELD = 4,
    REF_EOTHER = 9,
};

template <class F>
int guard(F&& f) {
    try {
        f();
        return REF_OK;
    } catch (const DimensionMismatch&) {
        return REF_EDIM;
    } catch (const OverlapError&) {
        return REF_EOVERLAP;
    } catch (const SingularMatrix&) {
        return REF_ESINGULAR;
    } catch (const SingularDiagonal&) {
        return REF_ESINGULAR;
    } catch (const NotPrime&) {
        return REF_EFIELD;
    } catch (const ModulusOutOfRange&) {
        return REF_EFIELD;
    } catch (...) {
        return REF_EOTHER;
    }
}

void put_ops(const OpCounter& c, std::uint64_t* ops) {
    if (!ops) return;
    ops[0] = c.n_mul;
    ops[1] = c.n_addsub;
    ops[2] = c.n_divinv;
    ops[3] = c.n_ztest;
}

MatView view_of(const PrimeField& f, std::uint32_t* a, std::int64_t m, std::int64_t n,
                std::int64_t ld) {
    return MatView(f, a, static_cast<std::size_t>(ld), 0, 0, static_cast<std::size_t>(m),
                   static_cast<std::size_t>(n));
}

} // namespace

extern "C" {

int ref_cup_u32(std::uint32_t* a, std::int64_t m, std::int64_t n, std::int64_t lda,
                std::uint32_t p, std::int64_t* rank, std::uint32_t* rrp,
                std::uint32_t* sigma, std::uint64_t* ops) {
    return guard([&] {
        PrimeField f(p);
        OpCounter c;
        PackedCup pc = cup(view_of(f, a, m, n, lda), c);
        *rank = static_cast<std::int64_t>(pc.rank);
        for (std::size_t j = 0; j < pc.rank; ++j) rrp[j] = pc.row_profile[j];
        for (std::size_t j = 0; j < pc.col_perm.order(); ++j) sigma[j] = pc.col_perm[j];
        put_ops(c, ops);
    });
}

// ranklab::ple (factor.hpp:37): rank, col_profile (cap min(m,n)), row_perm (order m).
int ref_ple_u32(std::uint32_t* a, std::int64_t m, std::int64_t n, std::int64_t lda,
                std::uint32_t p, std::int64_t* rank, std::uint32_t* prof,
                std::uint32_t* perm, std::uint64_t* ops) {
    return guard([&] {
        PrimeField f(p);
        OpCounter c;
        PackedPle pp = ple(view_of(f, a, m, n, lda), c);
        *rank = static_cast<std::int64_t>(pp.rank);
        for (std::size_t j = 0; j < pp.rank; ++j) prof[j] = pp.col_profile[j];
        for (std::size_t j = 0; j < pp.row_perm.order(); ++j) perm[j] = pp.row_perm[j];
        put_ops(c, ops);
    });
}

int ref_mm_u32(const std::uint32_t* a, std::int64_t lda, const std::uint32_t* b,
               std::int64_t ldb, std::uint32_t* c, std::int64_t ldc, std::int64_t m,
               std::int64_t l, std::int64_t n, std::uint32_t alpha, std::uint32_t beta,
               std::uint32_t p, std::uint64_t* ops) {
    return guard([&] {
        PrimeField f(p);
        OpCounter ctr;
        ConstMatView av(f, a, lda, 0, 0, m, l);
        ConstMatView bv(f, b, ldb, 0, 0, l, n);
        mm(av, bv, view_of(f, c, m, n, ldc), alpha, beta, ctr);
        put_ops(ctr, ops);
    });
}

// side: 0 Left 1 Right; uplo: 0 Upper 1 Lower; diag: 0 NonUnit 1 Unit.
int ref_trsm_u32(int side, int uplo, int diag, const std::uint32_t* t, std::int64_t ldt,
                 std::int64_t k, std::uint32_t* b, std::int64_t ldb, std::int64_t m,
                 std::int64_t n, std::uint32_t p, std::int64_t threshold,
                 std::uint64_t* ops) {
    return guard([&] {
        PrimeField f(p);
        OpCounter ctr;
        ConstMatView tv(f, t, ldt, 0, 0, k, k);
        trsm(side ? Side::Right : Side::Left, uplo ? UpLo::Lower : UpLo::Upper,
             diag ? Diag::Unit : Diag::NonUnit, tv, view_of(f, b, m, n, ldb), ctr,
             static_cast<std::size_t>(threshold));
        put_ops(ctr, ops);
    });
}

int ref_rank_and_profile_u32(std::uint32_t* a, std::int64_t m, std::int64_t n,
                             std::int64_t lda, std::uint32_t p, std::int64_t* rank,
                             std::uint32_t* rrp) {
    return guard([&] {
        PrimeField f(p);
        OpCounter c;
        auto rp = rank_and_profile(view_of(f, a, m, n, lda), c);
        *rank = static_cast<std::int64_t>(rp.first);
        for (std::size_t j = 0; j < rp.first; ++j) rrp[j] = rp.second[j];
    });
}

int ref_determinant_u32(std::uint32_t* a, std::int64_t n, std::int64_t lda,
                        std::uint32_t p, std::uint32_t* det) {
    return guard([&] {
        PrimeField f(p);
        OpCounter c;
        *det = determinant(view_of(f, a, n, n, lda), c);
    });
}

int ref_col_ech_trans_u32(std::uint32_t* a, std::int64_t m, std::int64_t n,
                          std::int64_t lda, std::uint32_t p, int reduced,
                          std::int64_t* rank, std::uint32_t* rrp, std::uint32_t* sigma,
                          std::uint64_t* ops) {
    return guard([&] {
        PrimeField f(p);
        OpCounter c;
        MatView v = view_of(f, a, m, n, lda);
        std::size_t r;
        if (reduced) {
            ReducedEchelonTransform t = red_col_ech_trans(v, c);
            r = t.rank;
            for (std::size_t j = 0; j < r; ++j) rrp[j] = t.row_profile[j];
            for (std::size_t j = 0; j < t.col_perm.order(); ++j) sigma[j] = t.col_perm[j];
        } else {
            EchelonTransform t = col_ech_trans(v, c);
            r = t.rank;
            for (std::size_t j = 0; j < r; ++j) rrp[j] = t.row_profile[j];
            for (std::size_t j = 0; j < t.col_perm.order(); ++j) sigma[j] = t.col_perm[j];
        }
        *rank = static_cast<std::int64_t>(r);
        put_ops(c, ops);
    });
}

int ref_invert_u32(std::uint32_t* a, std::int64_t n, std::int64_t lda, std::uint32_t p,
                   std::uint64_t* ops) {
    OpCounter c;
    const int st = guard([&] {
        PrimeField f(p);
        invert_in_place(view_of(f, a, n, n, lda), c);
    });
    put_ops(c, ops);
    return st;
}

int ref_random_matrix_u32(std::int64_t m, std::int64_t n, std::uint64_t seed,
                          std::uint32_t p, std::uint32_t* out) {
    return guard([&] {
        PrimeField f(p);
        Mat a = random_matrix(m, n, seed, f);
        for (std::int64_t i = 0; i < m; ++i)
            for (std::int64_t j = 0; j < n; ++j) out[i * n + j] = a(i, j);
    });
}

int ref_random_rank_matrix_u32(std::int64_t m, std::int64_t n, std::int64_t r,
                               std::uint64_t seed, std::uint32_t p, int generic,
                               std::uint32_t* out) {
    return guard([&] {
        PrimeField f(p);
        Mat a = random_rank_matrix(m, n, r, seed, f,
                                   generic ? RankPlacement::Generic : RankPlacement::Spread);
        for (std::int64_t i = 0; i < m; ++i)
            for (std::int64_t j = 0; j < n; ++j) out[i * n + j] = a(i, j);
    });
}

// reference.cpp:255-287 generators (the CLI bench inputs).
int ref_random_nonsingular_u32(std::int64_t n, std::uint64_t seed, std::uint32_t p,
                               std::uint32_t* out) {
    return guard([&] {
        PrimeField f(p);
        Mat a = random_nonsingular_matrix(n, seed, f);
        for (std::int64_t i = 0; i < n; ++i)
            for (std::int64_t j = 0; j < n; ++j) out[i * n + j] = a(i, j);
    });
}

int ref_random_triangular_u32(std::int64_t n, std::uint64_t seed, std::uint32_t p,
                              std::uint32_t* out) {
    return guard([&] {
        PrimeField f(p);
        Mat a = random_triangular_matrix(n, UpLo::Upper, seed, f);
        for (std::int64_t i = 0; i < n; ++i)
            for (std::int64_t j = 0; j < n; ++j) out[i * n + j] = a(i, j);
    });
}

int ref_naive_gauss_u32(const std::uint32_t* a, std::int64_t m, std::int64_t n,
                        std::uint32_t p, std::int64_t* rank, std::uint32_t* rrp) {
    return guard([&] {
        PrimeField f(p);
        ConstMatView v(f, a, n, 0, 0, m, n);
        NaiveGaussResult g = naive_gauss(v);
        *rank = static_cast<std::int64_t>(g.rank);
        for (std::size_t j = 0; j < g.rank; ++j) rrp[j] = g.row_profile[j];
    });
}

int ref_splitmix64(std::uint64_t seed, std::int64_t count, std::uint64_t* out) {
    return guard([&] {
        SplitMix64 rng(seed);
        for (std::int64_t i = 0; i < count; ++i) out[i] = rng.next();
    });
}

} // extern "C"
