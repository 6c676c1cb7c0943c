// rule.cuh — the KADABRA stopping rule evaluated on the device.
//
// kadabra.hpp:59-67 (f/g kernels) + 148-151 (kadabra_check) at the maximum
// per-vertex count. With uniform deltas (kadabra.hpp:30-36) f and g are
// monotone in b under IEEE round-to-nearest, so the all-vertex test of
// kadabra_converged (kadabra.hpp:133-144) equals the test at max_v data[v].
// Explicit _rn intrinsics keep the reference's operation order and forbid
// FMA contraction (the reference is an x86-64 SSE2 build).
#pragma once

#include <cstdint>

namespace adsb {

struct RuleParams {
    uint64_t omega;
    double omega_d;
    double log_inv;
    double eps;
};

// kadabra.hpp:59-67 + 148-151 at the maximum count, IEEE _rn ops only.
__device__ __forceinline__ bool rule_passes(uint64_t max_count, uint64_t tau, const RuleParams& r) {
    if (tau >= r.omega) return true;
    const double tau_d = __ull2double_rn(tau);
    const double b = __ddiv_rn(__ull2double_rn(max_count), tau_d);
    const double two_b_w_l = __ddiv_rn(__dmul_rn(__dmul_rn(2.0, b), r.omega_d), r.log_inv);
    const double scale = __ddiv_rn(r.log_inv, tau_d);
    const double w_t = __ddiv_rn(r.omega_d, tau_d);
    const double tf = __dsub_rn(1.0 / 3.0, w_t);
    const double f = __dmul_rn(scale, __dadd_rn(tf, __dsqrt_rn(__dadd_rn(__dmul_rn(tf, tf), two_b_w_l))));
    if (f > r.eps) return false;
    const double tg = __dadd_rn(1.0 / 3.0, w_t);
    const double g = __dmul_rn(scale, __dadd_rn(tg, __dsqrt_rn(__dadd_rn(__dmul_rn(tg, tg), two_b_w_l))));
    return !(g > r.eps);
}


}  // namespace adsb
