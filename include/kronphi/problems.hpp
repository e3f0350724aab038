// Forwarding header: code written against the reference's
// "kronphi/problems.hpp" compiles unchanged against the B200 drop-in.
#pragma once
#include "kronphi_b200/kronphi.hpp"
