// Decision-cost micro-benchmark and zero-loss swap stress (BASELINE.json config 5).
//
// Method follows SPEC.md bench module L477-481 / L503 (>= 1e4 warm-up calls
// excluded, monotonic clock, full sample buffer, p50/p99) and reload module
// L444-446 (4 invokers + 1 reloader, 1000 swaps, per-thread generation
// monotonicity, reject-preserves-old).  Paper context: native 20/30 ns
// P50/P99, swap 1.07 us, 0 lost calls over 400,000.
#include <algorithm>
#include <atomic>
#include <chrono>
#include <cstring>
#include <thread>
#include <vector>

#include "polar.h"
#include "polar_internal.h"

namespace {

using clk = std::chrono::steady_clock;

inline uint64_t now_ns() {
    return (uint64_t)std::chrono::duration_cast<std::chrono::nanoseconds>(clk::now().time_since_epoch()).count();
}

double pct(std::vector<uint64_t>& v, double q) {
    if (v.empty()) return 0.0;
    size_t k = (size_t)(q * (double)(v.size() - 1) + 0.5);
    std::nth_element(v.begin(), v.begin() + k, v.end());
    return (double)v[k];
}

}  // namespace

extern "C" {

polar_status polar_bench_decide(const polar_ctx* ctxs, uint32_t nctx, uint64_t nwarm, uint64_t ncalls,
                                uint64_t* samples_ns, polar_bench_stats* out) {
    if (!ctxs || nctx == 0 || !out || ncalls == 0) return POLAR_EINVAL;
    polar_decision d;
    volatile uint32_t sink = 0;
    for (uint64_t i = 0; i < nwarm; ++i) {
        if (polar_decide(&ctxs[i % nctx], &d) != POLAR_OK) return POLAR_EINVAL;
        sink += d.nchannels;
    }
    std::vector<uint64_t> s(ncalls);
    // timer overhead: empty timing pairs
    std::vector<uint64_t> e(std::min<uint64_t>(ncalls, 100000));
    for (auto& x : e) {
        uint64_t t0 = now_ns();
        uint64_t t1 = now_ns();
        x = t1 - t0;
    }
    for (uint64_t i = 0; i < ncalls; ++i) {
        const polar_ctx* c = &ctxs[i % nctx];
        uint64_t t0 = now_ns();
        polar_decide(c, &d);
        uint64_t t1 = now_ns();
        sink += d.nchannels;
        s[i] = t1 - t0;
    }
    // batched: no per-call timer
    uint64_t b0 = now_ns();
    for (uint64_t i = 0; i < ncalls; ++i) {
        polar_decide(&ctxs[i % nctx], &d);
        sink += d.algo;
    }
    uint64_t b1 = now_ns();
    (void)sink;
    if (samples_ns) std::memcpy(samples_ns, s.data(), ncalls * sizeof(uint64_t));
    double sum = 0;
    uint64_t mn = ~0ull, mx = 0;
    for (uint64_t x : s) { sum += (double)x; mn = std::min(mn, x); mx = std::max(mx, x); }
    out->calls = ncalls;
    out->mean_ns = sum / (double)ncalls;
    out->min_ns = (double)mn;
    out->max_ns = (double)mx;
    out->p50_ns = pct(s, 0.50);
    out->p99_ns = pct(s, 0.99);
    out->timer_overhead_ns = pct(e, 0.50);
    out->batched_mean_ns = (double)(b1 - b0) / (double)ncalls;
    return POLAR_OK;
}

polar_status polar_bench_swap(uint32_t nthreads, uint64_t calls_per_thread, uint32_t nswaps,
                              const polar_policy_row* a, uint32_t na, const polar_policy_row* b, uint32_t nb,
                              polar_swap_stats* out) {
    if (!out || nthreads == 0 || nthreads > 64) return POLAR_EINVAL;
    if (polar::validate_rows(a, na) != POLAR_OK || polar::validate_rows(b, nb) != POLAR_OK) return POLAR_EINVAL;
    // contexts cycled by the invokers: sizes 2^3..2^30 x nranks {2,4,8}
    std::vector<polar_ctx> ctxs;
    for (uint32_t k = 3; k <= 30; ++k)
        for (uint32_t n : {2u, 4u, 8u}) ctxs.push_back({POLAR_COLL_ALLREDUCE, n, 1ull << k});
    const size_t nctx = ctxs.size();
    // expected decisions for table A / B (generation field ignored)
    std::vector<polar_decision> expA(nctx), expB(nctx);
    for (size_t i = 0; i < nctx; ++i) {
        polar::decide_rows(a, na, 0, &ctxs[i], &expA[i]);
        polar::decide_rows(b, nb, 0, &ctxs[i], &expB[i]);
    }
    // generation -> which table (0 = A, 1 = B); written BEFORE the swap publishes it
    const uint32_t g0 = polar_policy_generation();
    std::vector<std::atomic<int>> which(nswaps + 2);
    for (auto& w : which) w.store(-1, std::memory_order_relaxed);
    uint32_t gen = 0;
    if (polar_set_policy(a, na, &gen) != POLAR_OK) return POLAR_EINVAL;
    const uint32_t gbase = gen;
    which[0].store(0, std::memory_order_release);
    (void)g0;

    std::atomic<bool> go{false};
    std::atomic<uint64_t> progress{0};   // calls issued so far (all invokers), paces the reloader
    std::vector<uint64_t> calls(nthreads, 0), invalid(nthreads, 0), nonmono(nthreads, 0);
    std::vector<std::thread> th;
    for (uint32_t t = 0; t < nthreads; ++t) {
        th.emplace_back([&, t]() {
            while (!go.load(std::memory_order_acquire)) {}
            uint32_t last = 0;
            uint64_t c = 0, bad = 0, nm = 0;
            polar_decision d;
            for (uint64_t i = 0; i < calls_per_thread; ++i) {
                size_t k = (i * 7 + t) % nctx;
                if (polar_decide(&ctxs[k], &d) != POLAR_OK) { ++bad; continue; }
                ++c;
                if ((i & 255) == 255) progress.fetch_add(256, std::memory_order_relaxed);
                if (d.generation < last) ++nm;
                last = d.generation;
                uint32_t idx = d.generation - gbase;
                int w = idx < which.size() ? which[idx].load(std::memory_order_acquire) : -1;
                const polar_decision& e = (w == 1) ? expB[k] : expA[k];
                if (w < 0 || d.algo != e.algo || d.proto != e.proto || d.nchannels != e.nchannels) ++bad;
            }
            calls[t] = c; invalid[t] = bad; nonmono[t] = nm;
        });
    }
    // an invalid table (duplicate max_bytes): must be rejected without effect
    polar_policy_row badrows[2] = {{0, 0, 100, POLAR_ALGO_RING, POLAR_PROTO_LL, 1, 0},
                                   {0, 0, 100, POLAR_ALGO_RING, POLAR_PROTO_LL, 1, 0}};   // duplicate bound
    std::vector<uint64_t> swap_ns;
    swap_ns.reserve(nswaps);
    uint64_t rejected = 0, rejected_changed = 0, swaps = 0;
    go.store(true, std::memory_order_release);
    const uint64_t issued = (uint64_t)nthreads * calls_per_thread;
    // spread the swaps evenly over the invokers' run ("1000 swaps across 400k calls")
    for (uint32_t s = 1; s <= nswaps; ++s) {
        const uint64_t target = issued * s / ((uint64_t)nswaps + 1);
        while (progress.load(std::memory_order_relaxed) + 256ull * nthreads < target) std::this_thread::yield();
        const bool useB = (s % 2) == 1;
        // generation gbase + s will hold table (useB ? B : A)
        which[s].store(useB ? 1 : 0, std::memory_order_release);
        uint64_t t0 = now_ns();
        uint32_t g = 0;
        polar_status st = useB ? polar_set_policy(b, nb, &g) : polar_set_policy(a, na, &g);
        uint64_t t1 = now_ns();
        if (st == POLAR_OK) { ++swaps; swap_ns.push_back(t1 - t0); }
        if (s % 10 == 0) {
            uint32_t before = polar_policy_generation();
            if (polar_set_policy(badrows, 2, nullptr) != POLAR_OK) ++rejected;
            if (polar_policy_generation() != before) ++rejected_changed;
        }
    }
    for (auto& x : th) x.join();
    out->issued = issued;
    out->calls = out->invalid = out->nonmonotonic = 0;
    for (uint32_t t = 0; t < nthreads; ++t) {
        out->calls += calls[t];
        out->invalid += invalid[t];
        out->nonmonotonic += nonmono[t];
    }
    out->swaps = swaps;
    out->rejected = rejected;
    out->rejected_changed = rejected_changed;
    out->swap_p50_ns = pct(swap_ns, 0.50);
    out->swap_p99_ns = pct(swap_ns, 0.99);
    out->swap_max_ns = swap_ns.empty() ? 0.0 : (double)*std::max_element(swap_ns.begin(), swap_ns.end());
    out->final_generation = polar_policy_generation();
    return POLAR_OK;
}

}  // extern "C"
