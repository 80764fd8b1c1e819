// internal.h -- library-internal declarations shared by the host translation units.
#pragma once
#include <cmath>
#include <cstdint>

#include "../../include/wf.h"
#include "common.h"

namespace wf {
bool fill_postable(PosTable* t, int rows, int chunk, const int32_t* starts, int n);
}  // namespace wf
const char* wf_static_error();
// record the error of a context-less call (wf_last_error(NULL) returns it)
wf_status wf_set_static_error(wf_status s, const char* msg);
void wf_clear_ctxless_error();
