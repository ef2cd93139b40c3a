// rl_errors.hpp -- maps the C ABI's RL_* status codes back onto the reference's
// exception hierarchy (proj/include/ranklab/errors.hpp:9-66) for the C++ shims.
#pragma once
#include <cstdint>
#include <cstdlib>
#include <cstring>
#include <string>

#include "ranklab/errors.hpp"
#include "ranklab_gpu.h"

namespace ranklab {
namespace gpu_shim {

// Throws the ranklab::Error subclass the reference would have thrown for the
// failure `st` of the C-ABI call `who` (p = the field's modulus).
[[noreturn]] inline void rethrow(int st, const char* who, std::uint64_t p) {
    const std::string detail = rl_last_error();
    const std::string msg = std::string(who) + ": " + detail;
    switch (st) {
    case RL_EDIM:
        throw DimensionMismatch(msg);
    case RL_EOVERLAP:
        throw OverlapError(detail.empty() ? msg : detail);
    case RL_ESINGULAR: {
        // trsm reports the index the reference's traversal meets first
        const char* at = std::strstr(detail.c_str(), "singular diagonal at ");
        if (at) throw SingularDiagonal(std::strtoull(at + 21, nullptr, 10));
        throw SingularMatrix();
    }
    case RL_EFIELD:
        if (p < 2 || p >= (1ull << 31)) throw ModulusOutOfRange(p);
        throw NotPrime(p);
    default:  // RL_ECUDA / RL_ENCCL / RL_EINVAL / RL_ENOMEM: no reference counterpart
        throw Error(msg);
    }
}

}  // namespace gpu_shim
}  // namespace ranklab
