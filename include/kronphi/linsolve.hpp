// Forwarding header: code written against the reference's
// "kronphi/linsolve.hpp" compiles unchanged against the B200 drop-in
// (LUFactors, lu_factor, lu_solve, solve on the device blocked LU).
#pragma once
#include "kronphi_b200/kronphi.hpp"
