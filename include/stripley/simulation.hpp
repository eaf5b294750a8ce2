// Drop-in include path: the reference's <stripley/simulation.hpp>
// (/root/reference/proj/core/include/stripley/simulation.hpp) served by the
// B200 library's C++ API, so reference programs compile unchanged.
#pragma once
#include "../stripley_gpu.hpp"
