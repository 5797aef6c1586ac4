// Profiler -> tuner closed loop: the adaptive channel controller (SURVEY.md §8(f)
// f3; §5.3 "Profiler-to-tuner composability", Listing 1
// L311-351).  The paper couples an eBPF profiler program (writes latency into a
// map) and a tuner program (reads it to pick channels).  Here the "map" is the
// comm's Adaptive state, fed by device-timed telemetry (comm.cu), and the rule
// is DESIGN.md R15 (the paper shows the behaviour, not the logic):
//     ref = ref[c] if known else ref[c-1]
//     if ref known and m > factor * ref:  c = c_min            (back off)
//     else:                               ref[c] = m; c = min(c + 1, cap)
// A window without samples leaves c unchanged.
#include <cmath>
#include <cstring>

#include "polar.h"
#include "polar_internal.h"

namespace polar {

void adaptive_reset(Adaptive& a, const polar_adaptive_params& p) {
    a.prm = p;
    a.c = p.c_min;
    a.contended = false;
    a.windows = 0;
    a.samples = 0;
    a.last_mean = 0.0;
    for (double& r : a.ref) r = 0.0;
    a.win_sum = 0.0;
    a.win_cnt = 0;
    a.calls = 0;
    a.cap = POLAR_MAXCH;
}

polar_status adaptive_validate(const polar_adaptive_params& p) {
    if (p.period < 1 || p.c_min < 1 || p.c_min > POLAR_MAXCH) return POLAR_EINVAL;
    if (!(p.contention_factor > 1.0) || !(p.latency_scale > 0.0)) return POLAR_EINVAL;
    return POLAR_OK;
}

// Close one window with mean latency m (<= 0 or NaN: no samples) under cap.
void adaptive_close_window(Adaptive& a, double m, uint32_t cap) {
    if (cap < 1) cap = 1;
    if (cap > POLAR_MAXCH) cap = POLAR_MAXCH;
    if (a.c > cap) a.c = cap;
    if (!(m > 0.0)) return;   // the tuner received no samples: remains where it is
    a.windows++;
    a.last_mean = m;
    double ref = a.ref[a.c];
    if (!(ref > 0.0) && a.c > 1) ref = a.ref[a.c - 1];
    if (ref > 0.0 && m > a.prm.contention_factor * ref) {
        a.contended = true;
        a.c = a.prm.c_min < cap ? a.prm.c_min : cap;
        return;
    }
    a.contended = false;
    a.ref[a.c] = m;
    if (a.c < cap) a.c++;
}

}  // namespace polar

extern "C" polar_status polar_adaptive_simulate(const polar_adaptive_params* params, uint32_t cap, const double* lat,
                                                uint32_t nwindows, uint32_t* channels_out) {
    if (!params || (nwindows && (!lat || !channels_out))) return POLAR_EINVAL;
    polar_status st = polar::adaptive_validate(*params);
    if (st != POLAR_OK) return st;
    polar::Adaptive a;
    polar::adaptive_reset(a, *params);
    if (cap < 1) cap = 1;
    if (cap > POLAR_MAXCH) cap = POLAR_MAXCH;
    if (a.c > cap) a.c = cap;
    for (uint32_t w = 0; w < nwindows; ++w) {
        const double m = lat[(size_t)w * (POLAR_MAXCH + 1) + a.c];
        polar::adaptive_close_window(a, std::isnan(m) ? 0.0 : m * params->latency_scale, cap);
        channels_out[w] = a.c;
    }
    return POLAR_OK;
}
