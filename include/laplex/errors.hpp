// laplex/errors.hpp -- drop-in exception taxonomy of the B200 LAPLEX path.
//
// Same type names and hierarchy as the reference (proj/include/laplex/
// errors.hpp:8-50): every type derives from laplex::Error (a
// std::runtime_error).  throw_for_code() maps the C-ABI's integer codes
// (include/laplex_c.h) back onto them.
#pragma once

#include <stdexcept>
#include <string>

#include "laplex_c.h"

namespace laplex {

struct Error : std::runtime_error {
    using std::runtime_error::runtime_error;
};

#define LAPLEX_DROPIN_ERROR(Name) \
    struct Name : Error {         \
        using Error::Error;       \
    }
LAPLEX_DROPIN_ERROR(EmptyInput);
LAPLEX_DROPIN_ERROR(NonFinite);
LAPLEX_DROPIN_ERROR(DimensionMismatch);
LAPLEX_DROPIN_ERROR(PhasePresent);
LAPLEX_DROPIN_ERROR(PhaseAbsent);
LAPLEX_DROPIN_ERROR(AsymmetricCotangent);
LAPLEX_DROPIN_ERROR(SizeCapExceeded);
LAPLEX_DROPIN_ERROR(NonPowerOfTwo);
LAPLEX_DROPIN_ERROR(NumericalBreakdown);
LAPLEX_DROPIN_ERROR(DivergenceDetected);
LAPLEX_DROPIN_ERROR(IoError);
LAPLEX_DROPIN_ERROR(InvalidSize);
LAPLEX_DROPIN_ERROR(InvalidFlag);
#undef LAPLEX_DROPIN_ERROR

/// Rethrow a C-ABI status as the matching reference exception type.
inline void throw_for_code(int code) {
    if (code == LAPLEX_OK) return;
    const std::string msg = laplex_last_error();
    switch (code) {
        case LAPLEX_E_EMPTY_INPUT: throw EmptyInput(msg);
        case LAPLEX_E_NON_FINITE: throw NonFinite(msg);
        case LAPLEX_E_DIMENSION_MISMATCH: throw DimensionMismatch(msg);
        case LAPLEX_E_PHASE_PRESENT: throw PhasePresent(msg);
        case LAPLEX_E_PHASE_ABSENT: throw PhaseAbsent(msg);
        case LAPLEX_E_ASYMMETRIC_COTANGENT: throw AsymmetricCotangent(msg);
        case LAPLEX_E_INVALID_SIZE: throw InvalidSize(msg);
        default: throw Error("laplex (B200): " + msg);
    }
}

}  // namespace laplex
