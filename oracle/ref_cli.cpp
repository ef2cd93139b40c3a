// ref_cli.cpp -- TEST INFRASTRUCTURE.  The reference's command-line behaviour
// (proj/tools/main.cpp: factor, echelon, solve, inverse, bench) rebuilt on the
// reference library compiled from its own sources, with a small argv parser in
// place of CLI11 (absent from /root/reference).  tests/test_cli.py compares the
// package CLI (python -m paper_1112_5717_b200) with this program byte for byte.
// Only the subcommand bodies' observable contract is reproduced: output bytes,
// exit codes, error lines.
#include <chrono>
#include <cstdlib>
#include <fstream>
#include <iostream>
#include <map>
#include <set>
#include <sstream>
#include <string>

#include "ranklab/bench.hpp"
#include "ranklab/echelon.hpp"
#include "ranklab/errors.hpp"
#include "ranklab/factor.hpp"
#include "ranklab/io.hpp"
#include "ranklab/kernels.hpp"
#include "ranklab/reference.hpp"
#include "ranklab/solvers.hpp"

using namespace ranklab;

namespace {

void header(std::ostream& o, const std::string& algo, std::size_t rank,
            const std::vector<std::uint32_t>& prof, const Perm& perm) {
    o << "algo " << algo << "\nrank " << rank << "\nprofile";
    for (auto v : prof) o << ' ' << v;
    o << "\nperm";
    for (std::size_t i = 0; i < perm.order(); ++i) o << ' ' << perm[i];
    o << '\n';
}

struct Args {
    std::map<std::string, std::string> v;
    std::set<std::string> flags;
    std::string get(const std::string& k, const std::string& d = "") const {
        auto it = v.find(k);
        return it == v.end() ? d : it->second;
    }
};

int run(const std::string& sub, const Args& a) {
    std::ofstream file;
    std::ostream* out = &std::cout;
    auto open_out = [&] {
        const std::string path = a.get("--out");
        if (path.empty()) return;
        file.open(path, std::ios::binary);
        if (!file) throw Error("cannot open " + path + " for writing");
        out = &file;
    };
    if (sub == "factor") {
        Mat m = read_matrix_file(a.get("--in"));
        open_out();
        OpCounter c;
        const std::string algo = a.get("--algo", "cup");
        const bool expand = a.flags.count("--expand");
        if (algo == "cup") {
            PackedCup pc = cup(m.view(), c);
            header(*out, algo, pc.rank, pc.row_profile, pc.col_perm);
            if (expand) {
                CupFactors fx = expand_cup(m.view(), pc);
                *out << "C\n";
                write_matrix(*out, fx.c.view());
                *out << "U\n";
                write_matrix(*out, fx.u.view());
            } else {
                *out << "body\n";
                write_matrix(*out, m.view());
            }
        } else if (algo == "ple") {
            PackedPle pp = ple(m.view(), c);
            header(*out, algo, pp.rank, pp.col_profile, pp.row_perm);
            if (expand) {
                PleFactors fx = expand_ple(m.view(), pp);
                *out << "L\n";
                write_matrix(*out, fx.l.view());
                *out << "E\n";
                write_matrix(*out, fx.e.view());
            } else {
                *out << "body\n";
                write_matrix(*out, m.view());
            }
        } else {
            throw Error("unknown --algo '" + algo + "' (expected cup or ple)");
        }
        out->flush();
        if (a.flags.count("--count-ops"))
            std::cout << "ops mul=" << c.n_mul << " addsub=" << c.n_addsub << " divinv="
                      << c.n_divinv << " ztest=" << c.n_ztest << " arith=" << c.arith_total()
                      << " total=" << c.full_total() << '\n';
        return 0;
    }
    if (sub == "echelon") {
        Mat m = read_matrix_file(a.get("--in"));
        open_out();
        OpCounter c;
        if (a.flags.count("--reduced")) {
            ReducedEchelonTransform t = red_col_ech_trans(m.view(), c);
            header(*out, "redcolech", t.rank, t.row_profile, t.col_perm);
            *out << "R\n";
            write_matrix(*out, reduced_form(m.view(), t).view());
        } else {
            EchelonTransform t = col_ech_trans(m.view(), c);
            header(*out, "colech", t.rank, t.row_profile, t.col_perm);
            *out << "E\n";
            write_matrix(*out, echelon_form(m.view(), t).view());
        }
        return 0;
    }
    if (sub == "solve") {
        Mat m = read_matrix_file(a.get("--in"));
        Mat b = read_matrix_file(a.get("--rhs"));
        if (m.field() != b.field()) throw Error("matrix and right-hand side use different moduli");
        OpCounter c;
        SolveResult res = solve(m.view(), b.view(), c);
        if (!res.consistent) {
            std::cout << "INCONSISTENT row " << res.witness_row << '\n';
            return 3;
        }
        open_out();
        write_matrix(*out, res.x->view());
        return 0;
    }
    if (sub == "inverse") {
        Mat m = read_matrix_file(a.get("--in"));
        OpCounter c;
        try {
            invert_in_place(m.view(), c);
        } catch (const SingularMatrix&) {
            std::cerr << "SINGULAR\n";
            return 1;
        }
        open_out();
        write_matrix(*out, m.view());
        return 0;
    }
    if (sub == "bench") {
        const std::string algo = a.get("--algo");
        std::size_t n = std::stoull(a.get("--n")), m = std::stoull(a.get("--m", "0")),
                    r = std::stoull(a.get("--r", "0"));
        PrimeField f(std::stoull(a.get("--field", "65521")));
        const std::uint64_t seed = std::stoull(a.get("--seed", "1"));
        const std::size_t trials = std::stoull(a.get("--trials", "1"));
        const std::size_t thr = std::stoull(a.get("--threshold", "1"));
        const bool json = a.flags.count("--json");
        const RankPlacement place =
            a.get("--placement", "generic") == "spread" ? RankPlacement::Spread : RankPlacement::Generic;
        if (m == 0) m = n;
        if (r == 0 || r > std::min(m, n)) r = std::min(m, n);
        for (std::size_t t = 0; t < trials; ++t) {
            BenchReport rep;
            rep.algo = algo;
            rep.m = m;
            rep.n = n;
            rep.r = r;
            rep.p = f.modulus();
            rep.seed = seed + t;
            const std::uint64_t s = rep.seed;
            OpCounter c;
            if (algo == "cup" || algo == "ple") {
                Mat x = (m == n && r == n) ? random_nonsingular_matrix(n, s, f)
                                           : random_rank_matrix(m, n, r, s, f, place);
                rep.r = algo == "cup" ? cup(x.view(), c).rank : ple(x.view(), c).rank;
            } else if (algo == "mm") {
                Mat x = random_matrix(n, n, s, f), y = random_matrix(n, n, s + 0x9E37, f);
                Mat z(f, n, n);
                mm(x.view(), y.view(), z.view(), f.one(), 0, c);
                rep.m = rep.r = n;
            } else if (algo == "trsm") {
                Mat tt = random_triangular_matrix(n, UpLo::Upper, s, f);
                Mat y = random_matrix(n, n, s + 0x9E37, f);
                trsm(Side::Right, UpLo::Upper, Diag::NonUnit, tt.view(), y.view(), c, thr);
                rep.m = rep.r = n;
            } else if (algo == "colech" || algo == "redcolech") {
                Mat x = random_nonsingular_matrix(n, s, f);
                if (algo == "colech") col_ech_trans(x.view(), c);
                else red_col_ech_trans(x.view(), c);
                rep.m = rep.r = n;
            } else {
                throw Error("unknown --algo '" + algo + "'");
            }
            rep.ops = c;
            rep.predicted = predicted_arith(algo, rep.m, n, rep.r);
            rep.ratio = rep.predicted > 0 ? double(c.arith_total()) / rep.predicted : 0;
            std::cout << (json ? format_report_json(rep) : format_report_kv(rep)) << '\n';
        }
        return 0;
    }
    std::cerr << "unknown subcommand\n";
    return 1;
}

}  // namespace

int main(int argc, char** argv) {
    if (argc < 2) return 1;
    Args a;
    static const std::set<std::string> flag_names = {"--expand", "--count-ops", "--reduced", "--json"};
    for (int i = 2; i < argc; ++i) {
        std::string k = argv[i];
        if (flag_names.count(k)) {
            a.flags.insert(k);
        } else if (i + 1 < argc) {
            a.v[k] = argv[++i];
        } else {
            return 1;
        }
    }
    try {
        return run(argv[1], a);
    } catch (const std::exception& e) {
        std::cerr << "error: " << e.what() << '\n';
        return 1;
    }
}
