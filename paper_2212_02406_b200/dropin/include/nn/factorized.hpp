#pragma once
// Drop-in header name of /root/reference/proj/include/nn/factorized.hpp; the B200
// declarations live in nnb_dropin.hpp.
#include "nn/nnb_dropin.hpp"
