// laplex/laplex.hpp -- umbrella include of the B200 drop-in (hot path:
// errors, common, scan, operator, gradients; reference laplex.hpp:3-10).
// The reference's application headers (limits.hpp, baselines.hpp,
// density.hpp) are callers of this API and are not part of the drop-in; they
// compile unchanged against these headers.
#pragma once

#include "laplex/common.hpp"
#include "laplex/errors.hpp"
#include "laplex/gradients.hpp"
#include "laplex/operator.hpp"
#include "laplex/scan.hpp"
