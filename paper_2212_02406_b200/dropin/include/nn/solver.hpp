#pragma once
// Drop-in header name of /root/reference/proj/include/nn/solver.hpp; the B200
// declarations live in nnb_dropin.hpp.
#include "nn/nnb_dropin.hpp"
