// shim_check.cpp -- TEST HARNESS for the C++ drop-in shims (tests/test_shims.py,
// tests/test_gpu_shims.py).  Linked like acceptance_gpu: the reference objects
// with cup/ple/echelon/invert/mm/trsm renamed to *_reference_cpu, plus the
// GPU shims.  Modes:
//   errors  -- every RL_* status surfaces as the reference's exception subclass
//              (errors.hpp:9-66); needs no GPU (the checks run before any
//              device work), except the last line which reports the base Error
//              a missing device raises;
//   parity  -- mm (all alpha/beta kinds) and the 8 trsm variants at several
//              thresholds on random strided views: bodies and OpCounter charges
//              equal the reference's (mm_reference_cpu / trsm_reference_cpu).
#include <cstdio>
#include <cstring>
#include <string>

#include "ranklab/echelon.hpp"
#include "ranklab/errors.hpp"
#include "ranklab/factor.hpp"
#include "ranklab/kernels.hpp"
#include "ranklab/reference.hpp"
#include "ranklab/solvers.hpp"

namespace ranklab {
void mm_reference_cpu(ConstMatView a, ConstMatView b, MatView c, Elem alpha, Elem beta, OpCounter& ctr);
void trsm_reference_cpu(Side side, UpLo uplo, Diag diag, ConstMatView t, MatView b, OpCounter& ctr,
                        std::size_t threshold);
}  // namespace ranklab

using namespace ranklab;

static int fails = 0;
#define EXPECT(cond, what)                                   \
    do {                                                     \
        if (!(cond)) {                                       \
            std::printf("FAIL %s\n", what);                  \
            ++fails;                                         \
        }                                                    \
    } while (0)

template <class E, class F>
static void expect_throw(const char* what, F&& f) {
    try {
        f();
        std::printf("FAIL %s: no exception\n", what);
        ++fails;
    } catch (const E& e) {
        std::printf("ok %s: %s\n", what, e.what());
    } catch (const std::exception& e) {
        std::printf("FAIL %s: wrong exception %s\n", what, e.what());
        ++fails;
    }
}

static bool same_ops(const OpCounter& a, const OpCounter& b) {
    return a.n_mul == b.n_mul && a.n_addsub == b.n_addsub && a.n_divinv == b.n_divinv && a.n_ztest == b.n_ztest;
}

static int errors_mode() {
    PrimeField f(7);
    OpCounter c;
    Mat a(f, 3, 4), b(f, 5, 2), cm(f, 3, 2);
    expect_throw<DimensionMismatch>("mm dims", [&] { mm(a.view(), b.view(), cm.view(), 1, 0, c); });
    Mat s(f, 6, 6);
    expect_throw<OverlapError>("mm C overlaps A",
                               [&] { mm(s.view(0, 3, 0, 3), s.view(0, 3, 3, 6), s.view(1, 4, 1, 4), 1, 1, c); });
    expect_throw<OverlapError>("mm C overlaps B",
                               [&] { mm(s.view(0, 3, 0, 3), s.view(3, 6, 3, 6), s.view(3, 6, 2, 5), 1, 1, c); });
    Mat t(f, 3, 3), bb(f, 3, 4);
    expect_throw<DimensionMismatch>("trsm non-square", [&] {
        trsm(Side::Left, UpLo::Upper, Diag::Unit, a.view(0, 3, 0, 2), bb.view(), c);
    });
    expect_throw<DimensionMismatch>("trsm side", [&] {
        trsm(Side::Right, UpLo::Upper, Diag::Unit, t.view(), bb.view(), c);
    });
    expect_throw<OverlapError>("trsm T overlaps B", [&] {
        trsm(Side::Left, UpLo::Lower, Diag::Unit, s.view(0, 3, 0, 3), s.view(1, 4, 1, 4), c);
    });
    // NonUnit with zeros on the diagonal: the reference names the index its
    // traversal meets first (ascending for Left/Lower)
    for (int i = 0; i < 3; ++i) t(i, i) = 1;
    t(1, 1) = 0;
    t(2, 2) = 0;
    expect_throw<SingularDiagonal>("trsm singular diagonal", [&] {
        trsm(Side::Left, UpLo::Lower, Diag::NonUnit, t.view(), bb.view(), c);
    });
    try {
        trsm(Side::Left, UpLo::Lower, Diag::NonUnit, t.view(), bb.view(), c);
    } catch (const SingularDiagonal& e) {
        std::string ours = e.what();
        try {
            trsm_reference_cpu(Side::Left, UpLo::Lower, Diag::NonUnit, t.view(), bb.view(), c, 1);
        } catch (const SingularDiagonal& r) {
            EXPECT(ours == r.what(), "SingularDiagonal index equals the reference's");
        }
    }
    // the index is local to the base block the traversal stops in, for every
    // variant and threshold
    for (int side = 0; side < 2; ++side)
        for (int uplo = 0; uplo < 2; ++uplo)
            for (std::size_t th : {1, 2, 3, 5, 16}) {
                Mat T(f, 11, 11), B(f, 11, 3);
                for (int i = 0; i < 11; ++i) T(i, i) = 1;
                T(4, 4) = 0;
                T(9, 9) = 0;
                const Side sd = side ? Side::Right : Side::Left;
                const UpLo ul = uplo ? UpLo::Lower : UpLo::Upper;
                Mat Bv = sd == Side::Left ? Mat(f, 11, 3) : Mat(f, 3, 11);
                std::string ours, ref;
                try { trsm(sd, ul, Diag::NonUnit, T.view(), Bv.view(), c, th); } catch (const SingularDiagonal& e) { ours = e.what(); }
                try { trsm_reference_cpu(sd, ul, Diag::NonUnit, T.view(), Bv.view(), c, th); } catch (const SingularDiagonal& e) { ref = e.what(); }
                EXPECT(!ours.empty() && ours == ref, ("SingularDiagonal " + std::to_string(side) + std::to_string(uplo) +
                                                       " th=" + std::to_string(th) + ": " + ours + " vs " + ref).c_str());
            }
    expect_throw<DimensionMismatch>("invert non-square", [&] { invert_in_place(a.view(), c); });
    std::printf("errors: %d failures\n", fails);
    return fails;
}

static int parity_mode() {
    SplitMix64 rng(77);
    const std::uint32_t primes[] = {2, 3, 7, 65521, 8388593, 2147483647u};
    for (int t = 0; t < 120; ++t) {
        PrimeField f(primes[rng.below(6)]);
        const std::size_t m = 1 + rng.below(70), l = rng.below(70), n = 1 + rng.below(70);
        Mat A = random_matrix(m + 2, l + 3, rng.next(), f), B = random_matrix(l + 1, n + 2, rng.next(), f);
        Mat C1 = random_matrix(m + 1, n + 1, rng.next(), f);
        Mat C2 = C1;
        const Elem vals[] = {0, f.one(), f.modulus() - 1, static_cast<Elem>(rng.below(f.modulus()))};
        const Elem alpha = vals[rng.below(4)], beta = vals[rng.below(4)];
        OpCounter c1, c2;
        mm(A.view(1, m + 1, 2, l + 2), B.view(1, l + 1, 1, n + 1), C1.view(0, m, 1, n + 1), alpha, beta, c1);
        mm_reference_cpu(A.view(1, m + 1, 2, l + 2), B.view(1, l + 1, 1, n + 1), C2.view(0, m, 1, n + 1), alpha,
                         beta, c2);
        EXPECT(C1 == C2 && same_ops(c1, c2), ("mm case " + std::to_string(t)).c_str());
    }
    for (int t = 0; t < 160; ++t) {
        PrimeField f(primes[rng.below(6)]);
        const Side side = rng.below(2) ? Side::Left : Side::Right;
        const UpLo uplo = rng.below(2) ? UpLo::Upper : UpLo::Lower;
        const Diag diag = rng.below(2) ? Diag::Unit : Diag::NonUnit;
        const std::size_t k = 1 + rng.below(60), o = 1 + rng.below(50);
        const std::size_t th = 1 + rng.below(40);
        Mat T = random_matrix(k + 1, k + 1, rng.next(), f);
        for (std::size_t i = 0; i < k + 1; ++i)
            if (T(i, i) == 0) T(i, i) = f.one();
        const std::size_t bm = side == Side::Left ? k : o, bn = side == Side::Left ? o : k;
        Mat B1 = random_matrix(bm + 1, bn + 2, rng.next(), f);
        Mat B2 = B1;
        OpCounter c1, c2;
        trsm(side, uplo, diag, T.view(1, k + 1, 1, k + 1), B1.view(1, bm + 1, 2, bn + 2), c1, th);
        trsm_reference_cpu(side, uplo, diag, T.view(1, k + 1, 1, k + 1), B2.view(1, bm + 1, 2, bn + 2), c2, th);
        EXPECT(B1 == B2 && same_ops(c1, c2), ("trsm case " + std::to_string(t)).c_str());
    }
    std::printf("parity: %d failures\n", fails);
    return fails;
}

int main(int argc, char** argv) {
    const std::string mode = argc > 1 ? argv[1] : "errors";
    return mode == "parity" ? parity_mode() : errors_mode();
}
