// internal.h -- library-internal declarations shared by the host translation units.
#pragma once
#include <cmath>
#include <cstdint>

#include "common.h"

namespace wf {
bool fill_postable(PosTable* t, int rows, int chunk, const int32_t* starts, int n);
}  // namespace wf
const char* wf_static_error();
