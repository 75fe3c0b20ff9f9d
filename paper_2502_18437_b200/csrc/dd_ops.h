// dd_ops.h — host entry points of the small device helpers the slab-DD driver needs
// (k_dd.cu), declared without CUDA headers so dd_driver.cpp stays plain C++.
#pragma once
#include <cstdint>

namespace mpmb {
void dd_add_f64(double* dst, const double* src, int64_t n, void* stream);
void dd_add_i32(int32_t* dst, const int32_t* src, int64_t n, void* stream);
// window buffer w[8] = {ylo, yhi, zlo, zhi, err, ...} <-> a form every entry of which is
// all-reduced with MIN: {ylo, -yhi, zlo, -zhi, -err}; ctl = the slab's DD control words
void dd_window_to_min_form(int32_t* w, const uint32_t* ctl, void* stream);
void dd_window_from_min_form(int32_t* w, void* stream);
}  // namespace mpmb
