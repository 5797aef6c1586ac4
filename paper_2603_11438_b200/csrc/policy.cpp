// Policy slot + decision hook (include/polar.h).
//
// The paper's tuner hook (§2; §3.3) is rebuilt as a
// native, bounded table scan: the policy is DATA (<= 64 rows), validated at
// install time instead of being verified bytecode.
// Hot reload (§4) is an atomic pointer exchange; retired
// tables are kept until process exit so no in-flight decide() can read freed
// memory (SPEC.md L446 drain safety).
#include <atomic>
#include <cstring>
#include <memory>
#include <mutex>
#include <vector>

#include "polar.h"
#include "polar_internal.h"

namespace {

struct Table {
    uint32_t generation;
    uint32_t nrows;
    polar_policy_row rows[POLAR_MAXROWS];
};

// Built-in default table: what every UNSET field and
// the empty policy (`noop`) defer to.
constexpr uint64_t KiB = 1024, MiB = 1024 * 1024;
const polar_policy_row kDefaultRows[] = {
    {POLAR_COLL_ALLREDUCE, 0, 64 * KiB, POLAR_ALGO_ONESHOT, POLAR_PROTO_LL, 4, 0},
    {POLAR_COLL_ALLREDUCE, 0, 1 * MiB, POLAR_ALGO_ONESHOT, POLAR_PROTO_SIMPLE, 8, 0},
    {POLAR_COLL_ALLREDUCE, 0, ~uint64_t(0), POLAR_ALGO_TWOSHOT, POLAR_PROTO_SIMPLE, 32, 0},
    // other collectives (f4): one direct all-to-all step
    {POLAR_COLL_ALLGATHER, 0, ~uint64_t(0), POLAR_ALGO_ONESHOT, POLAR_PROTO_SIMPLE, 32, 0},
    {POLAR_COLL_BROADCAST, 0, ~uint64_t(0), POLAR_ALGO_ONESHOT, POLAR_PROTO_SIMPLE, 32, 0},
    {POLAR_COLL_REDUCESCATTER, 0, ~uint64_t(0), POLAR_ALGO_ONESHOT, POLAR_PROTO_SIMPLE, 32, 0},
};
constexpr uint32_t kNumDefault = sizeof(kDefaultRows) / sizeof(kDefaultRows[0]);

const Table kEmpty = {0, 0, {}};
std::atomic<const Table*> g_active{&kEmpty};
std::mutex g_reload_mu;                       // one reloader at a time
std::vector<std::unique_ptr<Table>> g_retired;  // drain safety: never freed while running

inline const polar_policy_row* first_match(const polar_policy_row* rows, uint32_t n, uint32_t coll,
                                           uint32_t nranks, uint64_t bytes) {
    for (uint32_t i = 0; i < n; ++i) {
        const polar_policy_row& r = rows[i];
        if (r.coll == coll && (r.nranks == 0 || r.nranks == nranks) && bytes <= r.max_bytes) return &r;
    }
    return nullptr;
}

}  // namespace

namespace polar {

polar_status validate_rows(const polar_policy_row* rows, uint32_t nrows) {
    if (nrows > POLAR_MAXROWS) return POLAR_EINVAL;
    if (nrows && !rows) return POLAR_EINVAL;
    bool unsupported = false;
    for (uint32_t i = 0; i < nrows; ++i) {
        const polar_policy_row& r = rows[i];
        if (r.coll > POLAR_COLL_REDUCESCATTER) return POLAR_EINVAL;
        if (r.nranks > POLAR_MAXRANKS) return POLAR_EINVAL;
        if (r.flags & ~POLAR_ROW_ADAPTIVE_NCH) return POLAR_EINVAL;
        switch (r.algo) {
            case POLAR_ALGO_TREE: case POLAR_ALGO_RING: case POLAR_ALGO_ONESHOT:
            case POLAR_ALGO_TWOSHOT: case POLAR_UNSET: break;
            case POLAR_ALGO_NVLS:
                // accepted only while some comm holds a multicast object (nvls_host.cpp);
                // ReduceScatter / AllGather / Broadcast have no NVLS kernel
                if (!polar::nvls_available() || r.coll != POLAR_COLL_ALLREDUCE) unsupported = true;
                break;
            default: return POLAR_EINVAL;
        }
        switch (r.proto) {
            case POLAR_PROTO_LL: case POLAR_PROTO_LL128: case POLAR_PROTO_SIMPLE: case POLAR_UNSET: break;
            default: return POLAR_EINVAL;
        }
        // ReduceScatter / AllGather / Broadcast have one kernel: the direct
        // all-to-all step (ONESHOT / SIMPLE); any other choice would only fail
        // with EUNSUPPORTED at call time, so the table is refused now
        if (r.coll != POLAR_COLL_ALLREDUCE &&
            ((r.algo != POLAR_UNSET && r.algo != POLAR_ALGO_ONESHOT) ||
             (r.proto != POLAR_UNSET && r.proto != POLAR_PROTO_SIMPLE)))
            unsupported = true;
        // strictly ascending max_bytes within the (coll, nranks) group
        for (uint32_t j = 0; j < i; ++j) {
            if (rows[j].coll == r.coll && rows[j].nranks == r.nranks && r.max_bytes <= rows[j].max_bytes)
                return POLAR_EINVAL;
        }
    }
    return unsupported ? POLAR_EUNSUPPORTED : POLAR_OK;
}

// Decision against an explicit row set (used by decide() and the swap stress).
polar_status decide_rows(const polar_policy_row* rows, uint32_t nrows, uint32_t generation,
                         const polar_ctx* ctx, polar_decision* out) {
    if (ctx->nranks < 1 || ctx->nranks > POLAR_MAXRANKS) return POLAR_EINVAL;
    const polar_policy_row* d = first_match(kDefaultRows, kNumDefault, ctx->coll, ctx->nranks, ctx->bytes);
    if (!d) return POLAR_EUNSUPPORTED;
    uint32_t algo = d->algo, proto = d->proto, nch = d->nchannels, flags = 0;
    const polar_policy_row* m = first_match(rows, nrows, ctx->coll, ctx->nranks, ctx->bytes);
    if (m) {
        if (m->algo != POLAR_UNSET) algo = m->algo;
        if (m->proto != POLAR_UNSET) proto = m->proto;
        if (m->nchannels != 0) nch = m->nchannels;
        flags = m->flags;
    }
    if (nch < 1) nch = 1;
    if (nch > POLAR_MAXCH) nch = POLAR_MAXCH;
    out->algo = algo;
    out->proto = proto;
    out->nchannels = nch;
    out->generation = generation;
    out->flags = flags;
    out->_pad = 0;
    return POLAR_OK;
}

}  // namespace polar

extern "C" {

polar_status polar_set_policy(const polar_policy_row* rows, uint32_t nrows, uint32_t* generation_out) {
    polar_status st = polar::validate_rows(rows, nrows);
    if (st != POLAR_OK) return st;  // reject: the old policy continues
    std::lock_guard<std::mutex> lk(g_reload_mu);
    std::unique_ptr<Table> t(new (std::nothrow) Table);
    if (!t) return POLAR_ENOMEM;
    const Table* old = g_active.load(std::memory_order_acquire);
    t->generation = old->generation + 1;
    t->nrows = nrows;
    if (nrows) std::memcpy(t->rows, rows, nrows * sizeof(polar_policy_row));
    const Table* published = t.get();
    g_retired.emplace_back(std::move(t));
    g_active.store(published, std::memory_order_release);   // the swap
    if (generation_out) *generation_out = published->generation;
    return POLAR_OK;
}

polar_status polar_decide(const polar_ctx* ctx, polar_decision* out) {
    if (!ctx || !out) return POLAR_EINVAL;
    const Table* t = g_active.load(std::memory_order_acquire);
    return polar::decide_rows(t->rows, t->nrows, t->generation, ctx, out);
}

polar_status polar_decide_batch(const polar_ctx* ctx, polar_decision* out, size_t n) {
    if (n && (!ctx || !out)) return POLAR_EINVAL;
    for (size_t i = 0; i < n; ++i) {
        polar_status st = polar_decide(&ctx[i], &out[i]);
        if (st != POLAR_OK) return st;
    }
    return POLAR_OK;
}

uint32_t polar_policy_generation(void) { return g_active.load(std::memory_order_acquire)->generation; }

polar_status polar_get_policy(polar_policy_row* rows, uint32_t cap, uint32_t* nrows, uint32_t* generation) {
    const Table* t = g_active.load(std::memory_order_acquire);
    uint32_t n = t->nrows < cap ? t->nrows : cap;
    if (n && !rows) return POLAR_EINVAL;
    if (n) std::memcpy(rows, t->rows, n * sizeof(polar_policy_row));
    if (nrows) *nrows = t->nrows;
    if (generation) *generation = t->generation;
    return POLAR_OK;
}

const char* polar_status_string(polar_status s) {
    switch (s) {
        case POLAR_OK: return "POLAR_OK";
        case POLAR_EINVAL: return "POLAR_EINVAL: invalid argument or policy table";
        case POLAR_ECUDA: return "POLAR_ECUDA: CUDA call failed";
        case POLAR_EUNSUPPORTED: return "POLAR_EUNSUPPORTED: not built (NVLS, or an algorithm/protocol a collective has no kernel for)";
        case POLAR_ETIMEOUT: return "POLAR_ETIMEOUT: device wait for a peer timed out";
        case POLAR_EBUSY: return "POLAR_EBUSY: object in use";
        case POLAR_ESTATE: return "POLAR_ESTATE: comm unusable";
        case POLAR_ENOMEM: return "POLAR_ENOMEM: allocation failed";
    }
    return "POLAR_?: unknown status";
}

}  // extern "C"
