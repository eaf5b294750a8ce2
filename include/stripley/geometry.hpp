// Drop-in include path: the reference's <stripley/geometry.hpp>
// (/root/reference/proj/core/include/stripley/geometry.hpp) served by the
// B200 library's C++ API, so reference programs compile unchanged.
#pragma once
#include "../stripley_gpu.hpp"
