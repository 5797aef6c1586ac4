// NCCL tuner-plugin shim (§4): the same
// policy table that drives polar's own kernels, exported to NCCL 2.28.9 as a
// tuner plugin so it can steer NCCL's ring / tree / NVLS kernels on B200.
//
//   "NCCL's tuner API uses cost arrays rather than direct algorithm IDs: the
//    tuner sets costs to zero for preferred choices and to a sentinel value
//    (1e9) for others, allowing NCCL to fall back gracefully if the requested
//    combination is unavailable. [...] NCCL also passes a maximum channel count
//    that the tuner must respect; our native baseline layer clamps the
//    policy's request."
//
// getCollInfo(coll, nBytes):
//   * the first policy row (libpolar's process-global table, or POLAR_POLICY=
//     file.json read at init) matching (coll, nranks, nBytes) decides;
//   * a row's algorithm maps TREE -> NCCL_ALGO_TREE, RING -> RING, NVLS -> NVLS;
//     its protocol LL / LL128 / SIMPLE maps 1:1.  UNSET fields — and polar's own
//     ONESHOT / TWOSHOT, which NCCL does not have — leave that dimension to NCCL;
//   * cost cells: the preferred (algo, proto) cell(s) keep their meaning, every
//     other available cell becomes 1e9; NCCL_ALGO_PROTO_IGNORE (-1) cells are
//     never touched; if no preferred cell is available the table is left as is
//     (NCCL falls back to its own choice);
//   * nChannels: the row's count (0 = UNSET: untouched), clamped to the maximum
//     NCCL passed in *nChannels (when > 0) and to [1, 32].
// No row matches -> nothing changes (NCCL's default, the paper's `noop`).
// Exported as ncclTunerPlugin_v3 and _v4 (v4 adds regBuff; same behaviour).
#include <atomic>
#include <cstdint>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <mutex>
#include <string>
#include <vector>

#include "polar.h"

extern "C" {
typedef enum { ncclSuccess = 0, ncclInternalError = 3, ncclInvalidArgument = 4 } ncclResult_t;
typedef void (*ncclDebugLogger_t)(int level, unsigned long flags, const char* file, int line, const char* fmt, ...);
typedef enum {
    ncclFuncBroadcast = 0, ncclFuncReduce = 1, ncclFuncAllGather = 2, ncclFuncReduceScatter = 3,
    ncclFuncAllReduce = 4, ncclFuncSendRecv = 5, ncclFuncSend = 6, ncclFuncRecv = 7
} ncclFunc_t;
typedef struct {
    const char* name;
    ncclResult_t (*init)(size_t nRanks, size_t nNodes, ncclDebugLogger_t logFunction, void** context);
    ncclResult_t (*getCollInfo)(void* context, ncclFunc_t collType, size_t nBytes, int numPipeOps,
                                float** collCostTable, int numAlgo, int numProto, int* nChannels);
    ncclResult_t (*destroy)(void* context);
} ncclTunerPlugin_v3_t;
typedef struct {
    const char* name;
    ncclResult_t (*init)(size_t nRanks, size_t nNodes, ncclDebugLogger_t logFunction, void** context);
    ncclResult_t (*getCollInfo)(void* context, ncclFunc_t collType, size_t nBytes, int numPipeOps,
                                float** collCostTable, int numAlgo, int numProto, int regBuff, int* nChannels);
    ncclResult_t (*destroy)(void* context);
} ncclTunerPlugin_v4_t;
}

namespace {

constexpr int kNcclAlgoTree = 0, kNcclAlgoRing = 1, kNcclAlgoNvls = 4;
constexpr int kNcclNumProtocols = 3;
constexpr float kIgnore = -1.0f;     // NCCL_ALGO_PROTO_IGNORE
constexpr float kSentinel = 1e9f;

struct Ctx {
    size_t nranks, nnodes;
    ncclDebugLogger_t log;
    uint64_t id;                     // stable id derived from the context pointer
};

// the table the plugin decides with: libpolar's active rows, refreshed when its generation moves
std::mutex g_mu;
std::vector<polar_policy_row> g_rows;
uint32_t g_gen = 0xFFFFFFFFu;
bool g_file = false;                 // POLAR_POLICY file loaded: it wins over libpolar's table

// {"rows": [[coll, nranks, max_bytes, algo, proto, nch(, flags)], ...]} — a plain scan
bool load_policy_file(const char* path, std::vector<polar_policy_row>& out) {
    FILE* f = std::fopen(path, "rb");
    if (!f) return false;
    std::string s;
    char buf[4096];
    size_t k;
    while ((k = std::fread(buf, 1, sizeof(buf), f)) > 0) s.append(buf, k);
    std::fclose(f);
    const size_t at = s.find("\"rows\"");
    if (at == std::string::npos) return false;
    size_t i = s.find('[', at);
    if (i == std::string::npos) return false;
    int depth = 0;
    std::vector<unsigned long long> vals;
    for (; i < s.size(); ++i) {
        const char ch = s[i];
        if (ch == '[') { ++depth; if (depth == 2) vals.clear(); }
        else if (ch == ']') {
            if (depth == 2) {
                if (vals.size() < 6 || vals.size() > 7) return false;
                polar_policy_row r{};
                r.coll = (uint32_t)vals[0]; r.nranks = (uint32_t)vals[1]; r.max_bytes = vals[2];
                r.algo = (uint32_t)vals[3]; r.proto = (uint32_t)vals[4]; r.nchannels = (uint32_t)vals[5];
                r.flags = vals.size() == 7 ? (uint32_t)vals[6] : 0;
                out.push_back(r);
            }
            if (--depth == 0) break;
        } else if (depth == 2 && ch >= '0' && ch <= '9') {
            char* end = nullptr;
            vals.push_back(std::strtoull(&s[i], &end, 10));
            i = (size_t)(end - s.data()) - 1;
        }
    }
    return depth == 0;
}

void refresh_rows() {
    if (g_file) return;
    const uint32_t gen = polar_policy_generation();
    if (gen == g_gen) return;
    polar_policy_row rows[POLAR_MAXROWS];
    uint32_t n = 0, g = 0;
    if (polar_get_policy(rows, POLAR_MAXROWS, &n, &g) != POLAR_OK) return;
    g_rows.assign(rows, rows + n);
    g_gen = g;
}

int coll_of(ncclFunc_t f) {
    switch (f) {
        case ncclFuncAllReduce: return POLAR_COLL_ALLREDUCE;
        case ncclFuncAllGather: return POLAR_COLL_ALLGATHER;
        case ncclFuncBroadcast: return POLAR_COLL_BROADCAST;
        case ncclFuncReduceScatter: return POLAR_COLL_REDUCESCATTER;
        default: return -1;
    }
}

int nccl_algo(uint32_t a) {
    switch (a) {
        case POLAR_ALGO_TREE: return kNcclAlgoTree;
        case POLAR_ALGO_RING: return kNcclAlgoRing;
        case POLAR_ALGO_NVLS: return kNcclAlgoNvls;
        default: return -1;          // UNSET, ONESHOT, TWOSHOT: NCCL decides
    }
}

ncclResult_t tuner_init(size_t nRanks, size_t nNodes, ncclDebugLogger_t logFunction, void** context) {
    if (!context) return ncclInvalidArgument;
    Ctx* c = new (std::nothrow) Ctx{nRanks, nNodes, logFunction, 0};
    if (!c) return ncclInternalError;
    uint64_t h = reinterpret_cast<uintptr_t>(c) * 0x9E3779B97F4A7C15ull;
    c->id = h ^ (h >> 29);
    {
        std::lock_guard<std::mutex> lk(g_mu);
        const char* path = std::getenv("POLAR_POLICY");
        if (path && *path && !g_file) {
            std::vector<polar_policy_row> rows;
            // the same validation as polar_set_policy; a rejected file leaves libpolar's table in charge
            if (load_policy_file(path, rows) && polar_set_policy(rows.data(), (uint32_t)rows.size(), nullptr) == POLAR_OK) {
                g_rows = rows;
                g_file = true;
            }
        }
    }
    *context = c;
    if (logFunction)   // NCCL_LOG_INFO (3), subsystem NCCL_INIT (0x1)
        logFunction(3, 0x1, __FILE__, __LINE__, "polar tuner: init nRanks %zu nNodes %zu, policy %s (generation %u)",
                    nRanks, nNodes, g_file ? "from POLAR_POLICY" : "libpolar's active table", polar_policy_generation());
    return ncclSuccess;
}

ncclResult_t tuner_get(void* context, ncclFunc_t collType, size_t nBytes, int, float** collCostTable, int numAlgo,
                       int numProto, int* nChannels) {
    const Ctx* c = static_cast<const Ctx*>(context);
    if (!c || !collCostTable) return ncclInvalidArgument;
    const int coll = coll_of(collType);
    if (coll < 0) return ncclSuccess;
    polar_policy_row row{};
    bool hit = false;
    {
        std::lock_guard<std::mutex> lk(g_mu);
        refresh_rows();
        for (const polar_policy_row& r : g_rows)
            if ((int)r.coll == coll && (r.nranks == 0 || r.nranks == c->nranks) && (uint64_t)nBytes <= r.max_bytes) {
                row = r;
                hit = true;
                break;
            }
    }
    if (!hit) return ncclSuccess;    // noop: NCCL's own choice
    // NCCL hands the table as float (*)[NCCL_NUM_PROTOCOLS] behind a float**
    float (*table)[kNcclNumProtocols] = reinterpret_cast<float (*)[kNcclNumProtocols]>(collCostTable);
    const int pa = nccl_algo(row.algo);
    const int pp = (row.proto <= POLAR_PROTO_SIMPLE) ? (int)row.proto : -1;
    if (numProto > kNcclNumProtocols) numProto = kNcclNumProtocols;
    if ((pa >= 0 && pa < numAlgo) || (pp >= 0 && pp < numProto)) {
        bool avail = false;
        for (int a = 0; a < numAlgo; ++a)
            for (int p = 0; p < numProto; ++p)
                if ((pa < 0 || a == pa) && (pp < 0 || p == pp) && table[a][p] != kIgnore) avail = true;
        if (avail)
            for (int a = 0; a < numAlgo; ++a)
                for (int p = 0; p < numProto; ++p) {
                    if (table[a][p] == kIgnore) continue;
                    const bool pref = (pa < 0 || a == pa) && (pp < 0 || p == pp);
                    if (!pref) table[a][p] = kSentinel;
                    else if (pa >= 0 && pp >= 0) table[a][p] = 0.0f;   // the one preferred cell
                }
    }
    if (c->log)        // NCCL_LOG_INFO (3), subsystem NCCL_TUNING (0x40)
        c->log(3, 0x40, __FILE__, __LINE__, "polar tuner: coll %d bytes %zu -> row algo %u proto %u nch %u", (int)collType,
               nBytes, row.algo, row.proto, row.nchannels);
    if (row.nchannels && nChannels) {
        int want = row.nchannels > POLAR_MAXCH ? POLAR_MAXCH : (int)row.nchannels;
        if (*nChannels > 0 && want > *nChannels) want = *nChannels;   // NCCL's maximum
        *nChannels = want < 1 ? 1 : want;
    }
    return ncclSuccess;
}

ncclResult_t tuner_get_v4(void* context, ncclFunc_t collType, size_t nBytes, int numPipeOps, float** collCostTable,
                          int numAlgo, int numProto, int, int* nChannels) {
    return tuner_get(context, collType, nBytes, numPipeOps, collCostTable, numAlgo, numProto, nChannels);
}

ncclResult_t tuner_destroy(void* context) {
    delete static_cast<Ctx*>(context);
    return ncclSuccess;
}

}  // namespace

extern "C" {
__attribute__((visibility("default"))) ncclTunerPlugin_v3_t ncclTunerPlugin_v3 = {"polar", tuner_init, tuner_get,
                                                                                     tuner_destroy};
__attribute__((visibility("default"))) ncclTunerPlugin_v4_t ncclTunerPlugin_v4 = {"polar", tuner_init, tuner_get_v4,
                                                                                     tuner_destroy};
}
