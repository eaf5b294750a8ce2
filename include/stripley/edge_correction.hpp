// Drop-in include path: the reference's <stripley/edge_correction.hpp>
// (/root/reference/proj/core/include/stripley/edge_correction.hpp) served by the
// B200 library's C++ API, so reference programs compile unchanged.
#pragma once
#include "../stripley_gpu.hpp"
