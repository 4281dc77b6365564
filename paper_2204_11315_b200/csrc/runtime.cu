// Plan lifetime, device arena ("single working buffer" allocator), pinned
// compressed host store, and the stream/event executor of the lowered
// Algorithm-1 schedule (plan.cpp).  C ABI: include/oocs.h.
#include <cuda_runtime.h>

#include <algorithm>
#include <cstdio>
#include <cstdlib>
#include <chrono>
#include <cstring>
#include <mutex>
#include <new>
#include <string>
#include <thread>
#include <unordered_map>
#include <vector>

#include <unistd.h>

#include "oocs_internal.h"

namespace oocs {

static thread_local std::string g_last_error;
void set_error(const std::string &msg) { g_last_error = msg; }

struct Arena {
    char *base = nullptr;
    size_t cap = 0, used = 0;
    bool owned = false;
    void *take(size_t bytes) {
        const size_t off = (used + 255) & ~size_t(255);
        if (off + bytes > cap) return nullptr;
        used = off + bytes;
        return base + off;
    }
};

struct KernelTiming {
    int kind;  // 0 decode, 1 step, 2 encode
    cudaEvent_t a, b;
};

struct Plan {
    Geometry geo;
    Arena arena;
    uint64_t arena_bytes = 0, ws_bytes = 0, staging_bytes = 0, store_bytes = 0;
    float *ws[MAX_LANES][N_ARRAYS] = {};     // working sets (fl_buf); [set][array]
    uint8_t *hf[MAX_LANES] = {};       // hf_buf[0:3]: per-lane compressed buffer, used for the
                                     // chunk coming in (3 arrays x max_ext planes) and, once decoded,
                                     // for the owned planes going out (2 arrays x max_own planes)
    uint8_t *dstore[2][N_ARRAYS] = {};  // device store (double-buffered pressures; velocity once)
    int cur = 0;
    uint8_t *hstore[N_ARRAYS] = {};  // pinned host store, store_planes x plane_bytes per array
    uint8_t *dvel = nullptr;         // OOCS_FLAG_RESIDENT_VELOCITY: compressed velocity kept in HBM
    bool resident_vel = false;
    float *vdec = nullptr;           // OOCS_FLAG_DECODED_VELOCITY: the rank's velocity decoded (store planes)
    // multi-GPU exchange region (its own cudaMalloc, so that it can be exported by CUDA IPC): four
    // sequence flags and the ghost slots the neighbours write (oocs.h "multi-GPU")
    uint8_t *xreg = nullptr;
    uint64_t xreg_bytes = 0, gh_bytes = 0;  // gh_bytes = kR planes x plane_bytes (one pressure array)
    uint32_t *xflags = nullptr;             // [READY_LO, READY_HI, FREE_LO, FREE_HI]
    uint8_t *gh[2][2][2] = {};              // own ghost slots [side 0 = below / 1 = above][parity][pressure]
    struct Peer {
        uint8_t *base = nullptr;  // the neighbour's exchange region as mapped here
        bool ipc = false;         // opened with cudaIpcOpenMemHandle (closed at destroy)
        uint8_t *slot[2][2] = {}; // the neighbour's ghost slots this rank writes [parity][pressure]
        uint32_t *flags = nullptr;
    } peer[2];                              // 0 = rank-1, 1 = rank+1
    bool connected = false;
    int64_t seq = 0;                        // index t of the state S_t the store holds (sweeps so far)
    int *d_err = nullptr;
    uint32_t *d_vmax = nullptr;           // oocs_load of the velocity: max|v| of the loaded planes (float bits)
    bool ext_klane[MAX_LANES] = {};       // lane's kernel stream is the caller's (oocs_config.ext_streams)
    cudaStream_t lanes[MAX_LANES] = {};   // copy stream of each lane (and its kernels with LANE_SINGLE_STREAM)
    cudaStream_t klanes[MAX_LANES] = {};  // kernel stream of each lane (== lanes[] with LANE_SINGLE_STREAM)
    cudaEvent_t xfer_ev[MAX_LANES] = {}, kdone[MAX_LANES] = {};
    bool split = false;
    cudaStream_t cstream[3] = {};           // dispatcher: H2D, D2H and D2D (carry) copy streams
    cudaEvent_t cdone[3] = {};
    std::vector<cudaEvent_t> op_done[2];    // dispatcher: completion event of every op of a run, per run slot
    uint64_t copy_chunk = 0;  // pipeline PCIe copies are issued in pieces of this many bytes (0: whole)
    std::vector<cudaEvent_t> ev[6];  // per oocs_event_kind, rings indexed by block counter / DAG node
    int ev_ring = 0;
    cudaEvent_t t0[2] = {}, t1[2] = {}, lane_done[MAX_LANES] = {};
    cudaStream_t tstream = nullptr;  // run marks: t0, and t1 after joining every stream of the run
    bool poisoned = false;
    std::vector<KernelTiming> timing_pool[2];
    size_t timing_used[2] = {0, 0};
    // Runs issued and not yet finalized, one per slot (oocs_run_async chains at most two in flight: a run
    // is issued only after the previous one's last op was issued, and the one before that is finalized).
    // The dispatcher state a chained run needs from its predecessor: every lane's last work op and the op
    // that produced each event instance (indices into that slot's op_done).
    struct RunRec {
        bool active = false;
        int64_t steps = 0;
        oocs_stats stats{};
        std::vector<int64_t> lane_last;
        std::unordered_map<int64_t, int64_t> producer[6];
    } runs[2];
    int slot = 1;              // slot of the most recent run (the first run goes to slot 0)
    int64_t g_next = 0;        // global chunk counter of the next run's first chunk (chainable plans)
    std::vector<oocs_stats> finished;  // stats of runs finalized since the last oocs_wait
    // OOCS_FLAG_TIMELINE: one event pair per work op (pool reused across runs) and the last run's spans
    std::vector<std::pair<cudaEvent_t, cudaEvent_t>> span_events;
    std::vector<oocs_span> spans;
    std::chrono::steady_clock::time_point host_t0;
};

}  // namespace oocs

// the opaque ABI handle is the plan itself
struct oocs_plan : public oocs::Plan {};

namespace oocs {

#define CU(call)                                                                       \
    do {                                                                               \
        cudaError_t e_ = (call);                                                       \
        if (e_ != cudaSuccess) {                                                       \
            set_error(std::string(#call) + ": " + cudaGetErrorString(e_));             \
            return OOCS_ERR_CUDA;                                                      \
        }                                                                              \
    } while (0)

static size_t al(size_t b) { return (b + 255) & ~size_t(255); }

// ---------------------------------------------------------------------------
// helpers on the geometry
// ---------------------------------------------------------------------------
static inline uint64_t pb(const Plan *p) { return (uint64_t)p->geo.plane_bytes; }
// Bytes of one plane of one array in the store.  The uncompressed BASELINE keeps its pinned host store
// in the working buffer's own pitched layout (rows of `pitch` floats, data at column XOFF), so that its
// H2D / D2H / carry are 1-D copies straight between store and working set: a pitched 2-D H2D of
// 4 KB rows was measured at 30.7 GB/s vs 55.5 GB/s for a 1-D copy (tools/memcpy2d_micro.py).  Every
// other store holds the codec's planes (plane_bytes).
static inline bool pitched_store(const Geometry &g) { return g.host_store && g.cfg.mode == OOCS_MODE_BASELINE; }
static inline uint64_t store_pb(const Geometry &g) {
    return pitched_store(g) ? (uint64_t)g.ay * g.pitch * 4 : (uint64_t)g.plane_bytes;
}
static inline uint64_t spb(const Plan *p) { return store_pb(p->geo); }
// byte offset of interior plane z inside one array of the store
static inline uint64_t hoff(const Plan *p, int64_t z) { return (uint64_t)(z - p->geo.store_lo) * spb(p); }
// device store: same indexing
static inline float *wsa(Plan *p, int set, int a) { return p->ws[set][a]; }
// velocity of chunk b for the stencil: working-set array 0, or the resident decoded velocity at the
// chunk's first extent plane (OOCS_FLAG_DECODED_VELOCITY)
static inline float *vel_of(Plan *p, int set, const oocs_block &b) {
    return p->vdec ? p->vdec + (b.ext_lo - p->geo.store_lo) * p->geo.pstride : p->ws[set][0];
}

static cudaEvent_t evt(Plan *p, int kind, int64_t g) { return p->ev[kind][(size_t)(g % (int64_t)p->ev[kind].size())]; }

// ---------------------------------------------------------------------------
// multi-GPU exchange region: layout, stream memory operations, ghost predicates
// ---------------------------------------------------------------------------
enum { F_READY_LO = 0, F_READY_HI = 1, F_FREE_LO = 2, F_FREE_HI = 3 };
// byte offset of ghost slot [side][parity][pressure] inside an exchange region (same on every rank)
static inline uint64_t slot_off(uint64_t gh_bytes, int side, int par, int j) {
    return 256 + (uint64_t)((side * 2 + par) * 2 + j) * al(gh_bytes);
}
static inline uint64_t xreg_size(uint64_t gh_bytes) { return 256 + 8 * al(gh_bytes); }

// cuStreamWaitValue32 / cuStreamWriteValue32 through the runtime's driver entry point (no libcuda link
// dependency).  The wait is done by the stream's front end (no SM is held); the write is fenced, so
// every earlier write of the stream (the ghost-slot stores) is visible before the flag.
typedef int (*StreamValueFn)(cudaStream_t, unsigned long long, uint32_t, unsigned);
static StreamValueFn stream_value_fn(const char *name) {
    void *fp = nullptr;
    cudaDriverEntryPointQueryResult qr;
    if (cudaGetDriverEntryPoint(name, &fp, cudaEnableDefault, &qr) == cudaSuccess && qr == cudaDriverEntryPointSuccess)
        return reinterpret_cast<StreamValueFn>(fp);
    return nullptr;
}
static oocs_status wait_geq(cudaStream_t st, const uint32_t *flag, uint32_t v) {
    static const StreamValueFn fn = stream_value_fn("cuStreamWaitValue32");
    if (!fn) {
        set_error("cuStreamWaitValue32 unavailable");
        return OOCS_ERR_CUDA;
    }
    const int r = fn(st, (unsigned long long)(uintptr_t)flag, v, 0 /* CU_STREAM_WAIT_VALUE_GEQ (wrap-safe) */);
    if (r) {
        set_error("cuStreamWaitValue32 failed (" + std::to_string(r) + ")");
        return OOCS_ERR_CUDA;
    }
    return OOCS_OK;
}
static oocs_status write_flag(cudaStream_t st, uint32_t *flag, uint32_t v) {
    static const StreamValueFn fn = stream_value_fn("cuStreamWriteValue32");
    if (!fn) {
        set_error("cuStreamWriteValue32 unavailable");
        return OOCS_ERR_CUDA;
    }
    const int r = fn(st, (unsigned long long)(uintptr_t)flag, v, 0 /* CU_STREAM_WRITE_VALUE_DEFAULT: fenced */);
    if (r) {
        set_error("cuStreamWriteValue32 failed (" + std::to_string(r) + ")");
        return OOCS_ERR_CUDA;
    }
    return OOCS_OK;
}
// does chunk b take its pressure planes below (above) its owned range from a ghost slot?
static inline bool ghost_lo(const Plan *p, const oocs_block &b) {
    return p->geo.cfg.world > 1 && p->geo.cfg.rank > 0 && &b == &p->geo.blocks[p->geo.b_lo];
}
static inline bool ghost_hi(const Plan *p, const oocs_block &b) {
    return p->geo.cfg.world > 1 && p->geo.cfg.rank + 1 < p->geo.cfg.world && &b == &p->geo.blocks[p->geo.b_hi - 1];
}

static oocs_status poison(Plan *p, oocs_status st) {
    if (st == OOCS_ERR_CUDA) p->poisoned = true;
    return st;
}

// Pipeline PCIe copies can go out in pieces of `chunk` bytes (OOCS_COPY_CHUNK_MB, default 0 = whole
// copies): an experiment against the copy-engine stalls of DESIGN.md §8 -- measured, pieces of 2-32 MB
// lower the achieved PCIe rate and do not remove the stalls (the host dispatcher does).
static cudaError_t copy_1d(void *dst, const void *src, uint64_t bytes, cudaMemcpyKind kind, cudaStream_t st,
                           uint64_t chunk) {
    if (!chunk) chunk = bytes;
    for (uint64_t o = 0; o < bytes; o += chunk) {
        cudaError_t e = cudaMemcpyAsync(static_cast<uint8_t *>(dst) + o, static_cast<const uint8_t *>(src) + o,
                                        std::min(chunk, bytes - o), kind, st);
        if (e != cudaSuccess) return e;
    }
    return cudaSuccess;
}

// pitched 2D copy of `planes` allocated planes between raw (row = ax floats) and working-buffer
// layout, in pieces of whole rows of about `chunk` bytes
static cudaError_t copy_raw_to_ws(float *ws_plane0, const void *raw, const Geometry &g, int64_t planes,
                                  cudaMemcpyKind kind, cudaStream_t st, uint64_t chunk = 0) {
    const int64_t rows = planes * g.ay, step = chunk ? std::max<int64_t>(1, (int64_t)(chunk / (g.ax * 4))) : rows;
    for (int64_t r = 0; r < rows; r += step) {
        cudaError_t e = cudaMemcpy2DAsync(ws_plane0 + XOFF + r * g.pitch, g.pitch * 4,
                                          static_cast<const float *>(raw) + r * g.ax, g.ax * 4, g.ax * 4,
                                          std::min(step, rows - r), kind, st);
        if (e != cudaSuccess) return e;
    }
    return cudaSuccess;
}
static cudaError_t copy_ws_to_raw(void *raw, const float *ws_plane0, const Geometry &g, int64_t planes,
                                  cudaMemcpyKind kind, cudaStream_t st, uint64_t chunk = 0) {
    const int64_t rows = planes * g.ay, step = chunk ? std::max<int64_t>(1, (int64_t)(chunk / (g.ax * 4))) : rows;
    for (int64_t r = 0; r < rows; r += step) {
        cudaError_t e = cudaMemcpy2DAsync(static_cast<float *>(raw) + r * g.ax, g.ax * 4,
                                          ws_plane0 + XOFF + r * g.pitch, g.pitch * 4, g.ax * 4,
                                          std::min(step, rows - r), kind, st);
        if (e != cudaSuccess) return e;
    }
    return cudaSuccess;
}

// ---------------------------------------------------------------------------
// kernel launch wrappers with optional event timing
// ---------------------------------------------------------------------------
static KernelTiming *timing_slot(Plan *p, int kind) {
    if (!(p->geo.cfg.flags & OOCS_FLAG_PROFILE)) return nullptr;
    auto &pool = p->timing_pool[p->slot];
    size_t &used = p->timing_used[p->slot];
    if (used == pool.size()) {
        KernelTiming t{kind, nullptr, nullptr};
        if (cudaEventCreate(&t.a) != cudaSuccess || cudaEventCreate(&t.b) != cudaSuccess) return nullptr;
        pool.push_back(t);
    }
    KernelTiming *t = &pool[used++];
    t->kind = kind;
    return t;
}

// n arrays of `planes` planes each, one launch for BlockQuant (stats count launches as issued)
static oocs_status k_decode(Plan *p, const void *const *src, float *const *dst, int n, int64_t planes,
                            cudaStream_t st, oocs_stats *stats) {
    KernelTiming *t = timing_slot(p, 0);
    if (t) CU(cudaEventRecord(t->a, st));
    CU(launch_decode(src, dst, n, p->geo.ax, p->geo.ay, planes, p->geo.pitch, p->geo.codec, p->geo.q, st));
    if (t) CU(cudaEventRecord(t->b, st));
    if (stats) {
        stats->kernel_launches[0] += p->geo.codec == OOCS_CODEC_BLOCKQUANT ? 1 : n;
        const uint64_t vals = (uint64_t)planes * p->geo.ax * p->geo.ay;
        stats->alg_bytes[0] += n * ((uint64_t)planes * pb(p) + vals * 4);
    }
    return OOCS_OK;
}
static oocs_status k_decode(Plan *p, const void *src, float *dst, int64_t planes, cudaStream_t st,
                            oocs_stats *stats) {
    return k_decode(p, &src, &dst, 1, planes, st, stats);
}

static oocs_status k_encode(Plan *p, const float *const *src, void *const *dst, int n, int64_t planes,
                            cudaStream_t st, oocs_stats *stats) {
    KernelTiming *t = timing_slot(p, 2);
    if (t) CU(cudaEventRecord(t->a, st));
    CU(launch_encode(src, dst, n, p->geo.ax, p->geo.ay, planes, p->geo.pitch, p->geo.codec, p->geo.q, p->d_err,
                     st));
    if (t) CU(cudaEventRecord(t->b, st));
    if (stats) {
        stats->kernel_launches[2] += p->geo.codec == OOCS_CODEC_BLOCKQUANT ? 1 : n;
        const uint64_t vals = (uint64_t)planes * p->geo.ax * p->geo.ay;
        stats->alg_bytes[2] += n * (vals * 4 + (uint64_t)planes * pb(p));
    }
    return OOCS_OK;
}
static oocs_status k_encode(Plan *p, const float *src, void *dst, int64_t planes, cudaStream_t st,
                            oocs_stats *stats) {
    return k_encode(p, &src, &dst, 1, planes, st, stats);
}

static oocs_status k_step(Plan *p, const float *v, float *pp, const float *pc, int64_t zlo, int64_t zhi,
                          cudaStream_t st, oocs_stats *stats) {
    KernelTiming *t = timing_slot(p, 1);
    if (t) CU(cudaEventRecord(t->a, st));
    CU(launch_step(v, pp, pc, p->geo.ax, p->geo.ay, p->geo.pitch, p->geo.max_ext, zlo, zhi, p->geo.cfg.dt,
                   p->geo.cfg.stencil, st));
    if (t) CU(cudaEventRecord(t->b, st));
    if (stats) {
        stats->kernel_launches[1]++;
        const uint64_t cells = (uint64_t)(zhi - zlo) * p->geo.nx * p->geo.ny;
        stats->cell_updates_computed += cells;
        stats->alg_bytes[1] += cells * 16;  // read p_curr, p_prev, v; write p_next
    }
    return OOCS_OK;
}

// decode only the x/y ring of one BlockQuant array (OOCS_FLAG_FUSE_DECODE)
static oocs_status k_decode_ring(Plan *p, const void *src, float *dst, int64_t planes, cudaStream_t st,
                                 oocs_stats *stats) {
    KernelTiming *t = timing_slot(p, 0);
    if (t) CU(cudaEventRecord(t->a, st));
    CU(launch_decode_ring(src, dst, p->geo.ax, p->geo.ay, planes, p->geo.pitch, p->geo.q, st));
    if (t) CU(cudaEventRecord(t->b, st));
    if (stats) {
        stats->kernel_launches[0]++;
        // the ring launch decodes 8 block rows of every line at each y edge and one line (8 blocks) of every
        // block row at each x edge: about 16 (nbx + nby) blocks per slab
        const uint64_t blocks = (uint64_t)(planes / 4) * 16 * (uint64_t)(p->geo.ax / 4 + p->geo.ay / 4);
        stats->alg_bytes[0] += blocks * (64 * 4 + 4 * pb(p) / ((uint64_t)(p->geo.ax / 4) * (p->geo.ay / 4)));
    }
    return OOCS_OK;
}

// the first step of a chunk with p_prev read from its compressed records (OOCS_FLAG_FUSE_DECODE)
static oocs_status k_step_fused(Plan *p, const float *v, float *pp, const float *pc, const void *rec_pp, int64_t zlo,
                                int64_t zhi, cudaStream_t st, oocs_stats *stats) {
    KernelTiming *t = timing_slot(p, 1);
    if (t) CU(cudaEventRecord(t->a, st));
    CU(launch_step_fused(v, pp, pc, rec_pp, p->geo.ax, p->geo.ay, p->geo.pitch, p->geo.max_ext, zlo, zhi,
                         p->geo.cfg.dt, p->geo.q, st));
    if (t) CU(cudaEventRecord(t->b, st));
    if (stats) {
        stats->kernel_launches[1]++;
        const uint64_t cells = (uint64_t)(zhi - zlo) * p->geo.nx * p->geo.ny;
        stats->cell_updates_computed += cells;
        // read p_curr, v and p_prev's records (rate/8 B per value); write p_next
        stats->alg_bytes[1] += cells * 12 + cells * (uint64_t)p->geo.cfg.rate_bits / 8;
    }
    return OOCS_OK;
}

// ---------------------------------------------------------------------------
// plan create / destroy
// ---------------------------------------------------------------------------
static void free_plan(Plan *p) {
    if (!p) return;
    int cur_dev = -1;
    cudaGetDevice(&cur_dev);
    cudaSetDevice(p->geo.cfg.device);
    for (int c = 0; c < 3; ++c) {
        if (p->cstream[c]) cudaStreamDestroy(p->cstream[c]);
        if (p->cdone[c]) cudaEventDestroy(p->cdone[c]);
    }
    for (auto &v : p->op_done)
        for (auto e : v) cudaEventDestroy(e);
    for (int l = 0; l < MAX_LANES; ++l) {
        if (p->split && p->klanes[l] && !p->ext_klane[l]) cudaStreamDestroy(p->klanes[l]);
        if (p->xfer_ev[l]) cudaEventDestroy(p->xfer_ev[l]);
        if (p->kdone[l]) cudaEventDestroy(p->kdone[l]);
    }
    for (int l = 0; l < MAX_LANES; ++l)
        if (p->lanes[l] && (p->split || !p->ext_klane[l])) cudaStreamDestroy(p->lanes[l]);
    for (auto &v : p->ev)
        for (auto e : v) cudaEventDestroy(e);
    for (auto e : p->lane_done)
        if (e) cudaEventDestroy(e);
    for (int k = 0; k < 2; ++k) {
        if (p->t0[k]) cudaEventDestroy(p->t0[k]);
        if (p->t1[k]) cudaEventDestroy(p->t1[k]);
        for (auto &t : p->timing_pool[k]) {
            cudaEventDestroy(t.a);
            cudaEventDestroy(t.b);
        }
    }
    if (p->tstream) cudaStreamDestroy(p->tstream);
    for (auto &e : p->span_events) {
        cudaEventDestroy(e.first);
        cudaEventDestroy(e.second);
    }
    for (auto &pr : p->peer)
        if (pr.ipc && pr.base) cudaIpcCloseMemHandle(pr.base);
    if (p->xreg) cudaFree(p->xreg);
    if (p->arena.owned && p->arena.base) cudaFree(p->arena.base);
    for (auto h : p->hstore)
        if (h) cudaFreeHost(h);
    if (cur_dev >= 0) cudaSetDevice(cur_dev);
    delete static_cast<oocs_plan *>(p);
}

// Device arena sizing ("single working buffer" allocator): one pure function shared by
// oocs_plan_create (which then allocates exactly this) and oocs_plan_estimate (which does not).
struct Sizes {
    size_t ws_array = 0, ws_bytes = 0, hfb = 0, staging = 0, arr_store = 0, store_bytes = 0, vdec = 0, total = 0;
    size_t xreg = 0;  // exchange region, allocated apart from the arena (part of `total`, the device peak)
    uint64_t xbytes = 0;
    bool codec_staging = false, resident_vel = false;
};
static Sizes compute_sizes(const Geometry &g) {
    Sizes z;
    z.ws_array = (size_t)g.max_ext * g.pstride * 4;
    z.ws_bytes = N_ARRAYS * al(z.ws_array);
    z.total = g.n_ws * z.ws_bytes;
    z.codec_staging = g.host_store && g.cfg.mode != OOCS_MODE_BASELINE;
    if (z.codec_staging) {
        z.hfb = al((size_t)N_ARRAYS * g.max_ext * g.plane_bytes);
        z.staging = g.lanes * z.hfb;
        z.total += z.staging;
    }
    z.arr_store = (size_t)g.store_planes() * store_pb(g);
    z.store_bytes = N_ARRAYS * z.arr_store;
    if (!g.host_store) z.total += al(z.arr_store) * 5;  // v + 2x(p_prev, p_curr)
    z.resident_vel = (g.cfg.flags & OOCS_FLAG_RESIDENT_VELOCITY) != 0;
    if (z.resident_vel) z.total += al(z.arr_store);
    if (g.cfg.flags & OOCS_FLAG_DECODED_VELOCITY) {
        z.vdec = (size_t)g.store_planes() * g.pstride * 4;
        z.total += al(z.vdec);
    }
    if (g.cfg.world > 1) {  // the exchange region (allocated on its own for CUDA IPC; counted here)
        z.xbytes = (uint64_t)g.k * R * store_pb(g);
        z.xreg = al(xreg_size(z.xbytes));
        z.total += z.xreg;
    }
    z.total += 256;  // error flag
    return z;
}

static void fill_info(const Geometry &g, const Sizes &z, oocs_plan_info *info) {
    std::memset(info, 0, sizeof(*info));
    info->ax = g.ax;
    info->ay = g.ay;
    info->az = g.az;
    info->pitch = g.pitch;
    info->plane_bytes = g.plane_bytes;
    info->z_lo = g.blocks[g.b_lo].own_lo;
    info->z_hi = g.blocks[g.b_hi - 1].own_hi;
    info->store_lo = g.store_lo;
    info->store_hi = g.store_hi;
    info->block_lo = g.b_lo;
    info->block_hi = g.b_hi;
    info->max_ext_planes = g.max_ext;
    info->arena_bytes = z.total;
    info->working_set_bytes = z.ws_bytes;
    info->staging_bytes = z.staging;
    info->store_bytes = z.store_bytes;
    info->n_working_sets = g.n_ws;
    info->n_lanes = g.lanes;
}

static oocs_status create(const oocs_config *cfg, Plan **out, void *ext_arena = nullptr, uint64_t ext_bytes = 0) {
    *out = nullptr;
    oocs_plan *p = new (std::nothrow) oocs_plan();
    if (!p) return OOCS_ERR_HOST_OOM;
    std::string err;
    oocs_status st = make_geometry(cfg, &p->geo, &err);
    if (st != OOCS_OK) {
        set_error(err);
        delete p;
        return st;
    }
    const Geometry &g = p->geo;
    if (cudaSetDevice(g.cfg.device) != cudaSuccess) {
        cudaGetLastError();
        set_error("cudaSetDevice failed for the plan's device");
        delete p;
        return OOCS_ERR_CUDA;
    }
    const Sizes z = compute_sizes(g);
    const size_t ws_array = z.ws_array, hfb = z.hfb, arr_store = z.arr_store, total = z.total - z.xreg;
    const bool codec_staging = z.codec_staging;
    p->ws_bytes = z.ws_bytes;
    p->staging_bytes = z.staging;
    p->store_bytes = z.store_bytes;
    p->resident_vel = z.resident_vel;
    p->gh_bytes = z.xbytes;
    p->arena_bytes = z.total;
    if (g.cfg.device_capacity && z.total > g.cfg.device_capacity) {
        set_error("device arena (" + std::to_string(z.total) + " B) exceeds device_capacity");
        delete p;
        return OOCS_ERR_DEVICE_OOM;
    }
    cudaError_t ce = cudaSuccess;
    if (ext_arena) {  // caller-owned device memory (e.g. a torch tensor), kept alive by the caller
        if (ext_bytes < total || (reinterpret_cast<uintptr_t>(ext_arena) & 255)) {
            set_error("external arena too small (need " + std::to_string(total) + " B, see oocs_plan_estimate) or "
                      "not 256-byte aligned");
            delete p;
            return OOCS_ERR_CONFIG;
        }
        cudaPointerAttributes pa{};
        if (cudaPointerGetAttributes(&pa, ext_arena) != cudaSuccess || pa.type != cudaMemoryTypeDevice ||
            pa.device != g.cfg.device) {
            cudaGetLastError();
            set_error("external arena is not device memory of the plan's device");
            delete p;
            return OOCS_ERR_CONFIG;
        }
        p->arena.base = static_cast<char *>(ext_arena);
        p->arena.owned = false;
    } else {
        ce = cudaMalloc((void **)&p->arena.base, total);
        if (ce != cudaSuccess) {
            cudaGetLastError();
            set_error(std::string("cudaMalloc of the device arena failed: ") + cudaGetErrorString(ce));
            delete p;
            return OOCS_ERR_DEVICE_OOM;
        }
        p->arena.owned = true;
    }
    p->arena.cap = total;
    for (int s = 0; s < g.n_ws; ++s)
        for (int a = 0; a < N_ARRAYS; ++a) p->ws[s][a] = (float *)p->arena.take(ws_array);
    if (codec_staging)
        for (int l = 0; l < g.lanes; ++l) p->hf[l] = (uint8_t *)p->arena.take(hfb);
    if (!g.host_store) {
        p->dstore[0][0] = (uint8_t *)p->arena.take(arr_store);
        p->dstore[1][0] = p->dstore[0][0];
        for (int b = 0; b < 2; ++b)
            for (int a = 1; a < N_ARRAYS; ++a) p->dstore[b][a] = (uint8_t *)p->arena.take(arr_store);
    }
    if (p->resident_vel) p->dvel = (uint8_t *)p->arena.take(arr_store);
    if (z.vdec) p->vdec = (float *)p->arena.take(z.vdec);
    p->d_err = (int *)p->arena.take(2 * sizeof(int));
    p->d_vmax = p->d_err ? reinterpret_cast<uint32_t *>(p->d_err + 1) : nullptr;
    if (!p->d_err) {
        set_error("internal: arena carve-out overflow");
        free_plan(p);
        return OOCS_ERR_STATE;
    }
    // zero the working sets so halo columns / padding are defined
    if (cudaMemset(p->arena.base, 0, p->arena.used) != cudaSuccess) {
        set_error("cudaMemset of the arena failed");
        free_plan(p);
        return OOCS_ERR_CUDA;
    }
    if (g.cfg.world > 1) {
        p->xreg_bytes = xreg_size(p->gh_bytes);
        ce = cudaMalloc((void **)&p->xreg, p->xreg_bytes);
        if (ce != cudaSuccess || cudaMemset(p->xreg, 0, p->xreg_bytes) != cudaSuccess) {
            cudaGetLastError();
            p->xreg = ce == cudaSuccess ? p->xreg : nullptr;
            set_error("allocation of the multi-GPU exchange region failed");
            free_plan(p);
            return OOCS_ERR_DEVICE_OOM;
        }
        p->xflags = reinterpret_cast<uint32_t *>(p->xreg);
        for (int side = 0; side < 2; ++side)
            for (int par = 0; par < 2; ++par)
                for (int j = 0; j < 2; ++j) p->gh[side][par][j] = p->xreg + slot_off(p->gh_bytes, side, par, j);
    }
    if (g.host_store) {
        for (int a = 0; a < N_ARRAYS; ++a) {
            ce = cudaHostAlloc((void **)&p->hstore[a], std::max<size_t>(arr_store, 1), cudaHostAllocDefault);
            if (ce != cudaSuccess) {
                cudaGetLastError();
                set_error(std::string("pinned host store allocation failed: ") + cudaGetErrorString(ce));
                free_plan(p);
                return OOCS_ERR_HOST_OOM;
            }
            std::memset(p->hstore[a], 0, arr_store);
        }
    }
    // a kernel stream per lane for the dispatcher and the split replay; the lane's own stream otherwise
    p->split = !(g.cfg.flags & OOCS_FLAG_LANE_SINGLE_STREAM);
    for (int c = 0; c < 3; ++c)
        if (cudaStreamCreateWithFlags(&p->cstream[c], cudaStreamNonBlocking) != cudaSuccess ||
            cudaEventCreateWithFlags(&p->cdone[c], cudaEventDisableTiming) != cudaSuccess) {
            set_error("stream/event creation failed");
            free_plan(p);
            return OOCS_ERR_CUDA;
        }
    {
        // piece size of the pipeline's PCIe copies (OOCS_COPY_CHUNK_MB overrides; 0 = whole copies)
        const char *env = std::getenv("OOCS_COPY_CHUNK_MB");
        p->copy_chunk = env ? (uint64_t)(std::strtod(env, nullptr) * 1048576.0) & ~uint64_t(15) : 0;
    }
    for (int l = 0; l < g.nstreams; ++l) {
        // a caller stream (oocs_config.ext_streams) is the lane's kernel stream (its only stream with
        // LANE_SINGLE_STREAM); it must belong to the plan's device
        cudaStream_t ext = static_cast<cudaStream_t>(g.cfg.ext_streams[l]);
        if (ext) {
            int sdev = -1;
            if (cudaStreamGetDevice(ext, &sdev) != cudaSuccess || sdev != g.cfg.device) {
                cudaGetLastError();
                set_error("ext_streams[" + std::to_string(l) + "] is not a stream of the plan's device");
                free_plan(p);
                return OOCS_ERR_CONFIG;
            }
            p->ext_klane[l] = true;
        }
        if ((!(ext && !p->split) && cudaStreamCreateWithFlags(&p->lanes[l], cudaStreamNonBlocking) != cudaSuccess) ||
            cudaEventCreateWithFlags(&p->lane_done[l], cudaEventDisableTiming) != cudaSuccess ||
            cudaEventCreateWithFlags(&p->xfer_ev[l], cudaEventDisableTiming) != cudaSuccess ||
            cudaEventCreateWithFlags(&p->kdone[l], cudaEventDisableTiming) != cudaSuccess ||
            (p->split && !ext && cudaStreamCreateWithFlags(&p->klanes[l], cudaStreamNonBlocking) != cudaSuccess)) {
            set_error("stream/event creation failed");
            free_plan(p);
            return OOCS_ERR_CUDA;
        }
        if (ext) (p->split ? p->klanes[l] : p->lanes[l]) = ext;
        if (!p->split) p->klanes[l] = p->lanes[l];
    }
    p->ev_ring = g.nb() + 8;
    // DAG node events: a wait always refers to a node at most `window` chunks back (plan.cpp)
    const int node_ring = (std::max(std::max(g.lanes, g.n_ws), g.nb()) + 4) * (g.k + 10);
    for (int k = 0; k < 6; ++k) {
        p->ev[k].resize(k == OOCS_EV_NODE ? node_ring : p->ev_ring);
        for (auto &e : p->ev[k])
            if (cudaEventCreateWithFlags(&e, cudaEventDisableTiming) != cudaSuccess) {
                set_error("event creation failed");
                free_plan(p);
                return OOCS_ERR_CUDA;
            }
    }
    if (cudaEventCreate(&p->t0[0]) != cudaSuccess || cudaEventCreate(&p->t1[0]) != cudaSuccess ||
        cudaEventCreate(&p->t0[1]) != cudaSuccess || cudaEventCreate(&p->t1[1]) != cudaSuccess ||
        cudaStreamCreateWithFlags(&p->tstream, cudaStreamNonBlocking) != cudaSuccess) {
        set_error("event creation failed");
        free_plan(p);
        return OOCS_ERR_CUDA;
    }
    *out = p;
    return OOCS_OK;
}

// ---------------------------------------------------------------------------
// executor
// ---------------------------------------------------------------------------
// STEP s updates array (s odd ? 1 : 2) from the other one (leapfrog in place).
static inline int upd_array(int s) { return (s & 1) ? 1 : 2; }

// compressed source of interior plane z of array a for chunk b (staging slot s, or the device store's S_t)
static inline const void *comp_src(Plan *p, int s, const oocs_block &b, int a, int64_t z) {
    const Geometry &g = p->geo;
    if (a == 0 && p->resident_vel) return p->dvel + hoff(p, z);
    if (g.host_store) return p->hf[s] + ((uint64_t)a * g.max_ext + (z - b.ext_lo)) * pb(p);
    return p->dstore[p->cur][a] + hoff(p, z);
}

// OOCS_FLAG_FUSE_DECODE applies to this chunk: no multi-GPU ghost planes (their p_{t-1} comes from a ghost
// slot in a second decode), and p_{t-1}'s records of the extent 16-byte aligned
static inline bool fused_first_step(Plan *p, const oocs_block &b) {
    return (p->geo.cfg.flags & OOCS_FLAG_FUSE_DECODE) && !ghost_lo(p, b) && !ghost_hi(p, b) && step_fused_ok(p->geo.q);
}

// Issue one work op (H2D, CARRY, DECODE, STEP, ENCODE, D2H, SEND) on stream st.  The device
// store's read/write buffers follow from the op's sweep: S_t = dstore[cur0 ^ (sweep & 1)].
static oocs_status issue_work(Plan *p, const oocs_op &o, cudaStream_t st, int cur0, oocs_stats *stats) {
    const Geometry &g = p->geo;
    const uint64_t PB = pb(p);
    const oocs_block &b = g.blocks[o.block];
    const int64_t E = b.ext_hi - b.ext_lo;
    const int w = (int)(o.g % g.n_ws);
    const int s = (int)(o.g % g.lanes);
    p->cur = cur0 ^ (o.sweep & 1);
    switch (o.kind) {
    case OOCS_OP_WAIT:
        CU(cudaStreamWaitEvent(st, evt(p, o.arg, o.ev_g), 0));
        break;
    case OOCS_OP_RECORD:
        CU(cudaEventRecord(evt(p, o.arg, o.ev_g), st));
        break;
    case OOCS_OP_H2D: {
        const int64_t nplanes = b.body_hi - b.body_lo, off = b.body_lo - b.ext_lo;
        if (g.cfg.mode == OOCS_MODE_BASELINE) {  // pitched store: one 1-D copy per array
            for (int a = 0; a < N_ARRAYS; ++a)
                CU(copy_1d(wsa(p, w, a) + off * g.pstride, p->hstore[a] + hoff(p, b.body_lo), nplanes * spb(p),
                           cudaMemcpyHostToDevice, st, p->copy_chunk));
            if (stats) stats->bytes_h2d += (uint64_t)N_ARRAYS * nplanes * spb(p);
        } else {
            // multi-GPU edge chunks: the pressure planes beyond the slab come from the ghost slots
            // (written by the neighbour over NVLink), never from the host store
            const int64_t plo = ghost_lo(p, b) ? std::max(b.body_lo, b.own_lo) : b.body_lo;
            const int64_t phi = ghost_hi(p, b) ? std::min(b.body_hi, b.own_hi) : b.body_hi;
            for (int a = p->resident_vel ? 1 : 0; a < N_ARRAYS; ++a) {
                const int64_t lo = a ? plo : b.body_lo, hi = a ? phi : b.body_hi;
                if (hi <= lo) continue;
                CU(copy_1d(p->hf[s] + ((uint64_t)a * g.max_ext + (lo - b.ext_lo)) * PB, p->hstore[a] + hoff(p, lo),
                           (hi - lo) * PB, cudaMemcpyHostToDevice, st, p->copy_chunk));
                if (stats) stats->bytes_h2d += (uint64_t)(hi - lo) * PB;
            }
        }
        break;
    }
    case OOCS_OP_CARRY: {
        // overlap of this chunk with the previous chunk's extent, already on the GPU
        const oocs_block &pbk = g.blocks[o.block - 1];
        const int64_t nplanes = b.carry_hi - b.carry_lo;
        const int64_t src_off = b.carry_lo - pbk.ext_lo, dst_off = b.carry_lo - b.ext_lo;
        if (g.cfg.mode == OOCS_MODE_BASELINE) {
            // lane of o is the previous chunk's lane; destination is chunk g's working set
            const int wprev = (int)((o.g - 1) % g.n_ws);
            const uint64_t nb = (uint64_t)nplanes * g.pstride * 4;
            auto sa = [&](int a) { return wsa(p, wprev, a) + src_off * g.pstride; };
            auto da = [&](int a) { return wsa(p, w, a) + dst_off * g.pstride; };
            CU(launch_peer_copy(sa(0), da(0), sa(1), da(1), nb, st));
            CU(launch_peer_copy(sa(2), da(2), nullptr, nullptr, nb, st, 1));
            if (stats) {
                stats->bytes_d2d += (uint64_t)N_ARRAYS * nplanes * g.ax * g.ay * 4;
                stats->copy_launches += 2;
            }
        } else {
            const int sp = (int)((o.g - 1) % g.lanes);
            auto sa = [&](int a) { return p->hf[sp] + ((uint64_t)a * g.max_ext + src_off) * PB; };
            auto da = [&](int a) { return p->hf[s] + ((uint64_t)a * g.max_ext + dst_off) * PB; };
            const uint64_t nb = (uint64_t)nplanes * PB;
            if (p->resident_vel) {
                CU(launch_peer_copy(sa(1), da(1), sa(2), da(2), nb, st));
            } else {
                CU(launch_peer_copy(sa(0), da(0), sa(1), da(1), nb, st));
                CU(launch_peer_copy(sa(2), da(2), nullptr, nullptr, nb, st, 1));
            }
            if (stats) stats->copy_launches += p->resident_vel ? 1 : 2;
            if (stats) stats->bytes_d2d += (uint64_t)(N_ARRAYS - (p->resident_vel ? 1 : 0)) * nplanes * PB;
        }
        break;
    }
    case OOCS_OP_DECODE: {
        auto src_of = [&](int a, int64_t z) { return comp_src(p, s, b, a, z); };
        // with the velocity kept decoded only the two pressures are decoded
        const int a0 = p->vdec ? 1 : 0;
        const bool glo = ghost_lo(p, b), ghi = ghost_hi(p, b);
        if (fused_first_step(p, b)) {
            // the velocity and p_t in one launch; of p_{t-1} only what the later steps read beyond the fused
            // first step's output: the x/y ring, and the physical z-halo planes of a boundary chunk
            const void *src[2];
            float *dst[2];
            int n = 0;
            if (!a0) {
                src[n] = src_of(0, b.ext_lo);
                dst[n++] = wsa(p, w, 0);
            }
            src[n] = src_of(2, b.ext_lo);
            dst[n++] = wsa(p, w, 2);
            if (oocs_status r = k_decode(p, src, dst, n, E, st, stats)) return r;
            if (oocs_status r = k_decode_ring(p, src_of(1, b.ext_lo), wsa(p, w, 1), E, st, stats)) return r;
            if (b.ext_lo == -R)
                if (oocs_status r = k_decode(p, src_of(1, b.ext_lo), wsa(p, w, 1), R, st, stats)) return r;
            if (b.ext_hi == g.nz + R)
                if (oocs_status r = k_decode(p, src_of(1, b.ext_hi - R), wsa(p, w, 1) + (E - R) * g.pstride, R, st,
                                             stats))
                    return r;
            break;
        }
        if (!glo && !ghi) {
            const void *src[N_ARRAYS];
            float *dst[N_ARRAYS];
            for (int a = 0; a < N_ARRAYS; ++a) {
                src[a] = src_of(a, b.ext_lo);
                dst[a] = wsa(p, w, a);
            }
            oocs_status r = k_decode(p, src + a0, dst + a0, N_ARRAYS - a0, E, st, stats);
            if (r) return r;
            break;
        }
        // multi-GPU edge chunk: the pressure planes beyond the slab are decoded straight out of the ghost
        // slots of state S_t, once the neighbour has written them (READY >= t); the neighbour's FREE flag
        // then releases the slot for S_{t+2}
        const uint32_t t_idx = (uint32_t)(p->seq + o.sweep);
        const int par = (int)(t_idx & 1u);
        const int64_t kR = (int64_t)g.k * R, mlo = glo ? b.own_lo : b.ext_lo, mhi = ghi ? b.own_hi : b.ext_hi;
        if (a0 == 0) {
            oocs_status r = k_decode(p, src_of(0, b.ext_lo), wsa(p, w, 0), E, st, stats);
            if (r) return r;
        }
        {
            const void *src[2] = {src_of(1, mlo), src_of(2, mlo)};
            float *dst[2] = {wsa(p, w, 1) + (mlo - b.ext_lo) * g.pstride, wsa(p, w, 2) + (mlo - b.ext_lo) * g.pstride};
            oocs_status r = k_decode(p, src, dst, 2, mhi - mlo, st, stats);
            if (r) return r;
        }
        for (int side = 0; side < 2; ++side) {
            if (!(side ? ghi : glo)) continue;
            if (oocs_status r = wait_geq(st, &p->xflags[side ? F_READY_HI : F_READY_LO], t_idx)) return r;
            const int64_t z0 = side ? b.own_hi : b.ext_lo;
            const void *src[2] = {p->gh[side][par][0], p->gh[side][par][1]};
            float *dst[2] = {wsa(p, w, 1) + (z0 - b.ext_lo) * g.pstride, wsa(p, w, 2) + (z0 - b.ext_lo) * g.pstride};
            oocs_status r = k_decode(p, src, dst, 2, kR, st, stats);
            if (r) return r;
            // the lower neighbour's upper sends / the upper neighbour's lower sends are consumed up to S_t
            Plan::Peer &pr = p->peer[side];
            if (oocs_status r2 = write_flag(st, pr.flags + (side ? F_FREE_LO : F_FREE_HI), t_idx + 1)) return r2;
        }
        break;
    }
    case OOCS_OP_STEP: {
        // step s is valid on [lo_s, hi_s): the trapezoid shrinks by R per step except at
        // the physical boundary (P:L85 temporal blocking)
        const int sidx = o.arg;
        const int64_t lo = (b.ext_lo == -R) ? 0 : b.ext_lo + (int64_t)sidx * R;
        const int64_t hi = (b.ext_hi == g.nz + R) ? g.nz : b.ext_hi - (int64_t)sidx * R;
        const int up = upd_array(sidx), other = 3 - up;
        oocs_status r = sidx == 1 && fused_first_step(p, b)
                            ? k_step_fused(p, vel_of(p, w, b), wsa(p, w, up), wsa(p, w, other),
                                           comp_src(p, s, b, up, b.ext_lo), lo - b.ext_lo, hi - b.ext_lo, st, stats)
                            : k_step(p, vel_of(p, w, b), wsa(p, w, up), wsa(p, w, other), lo - b.ext_lo,
                                     hi - b.ext_lo, st, stats);
        if (r) return r;
        break;
    }
    case OOCS_OP_ENCODE: {
        // after k steps: level t0+k in array upd(k), level t0+k-1 in the other
        const int curr = upd_array(g.k), prev = 3 - curr;
        const int64_t W = b.own_hi - b.own_lo, off = b.own_lo - b.ext_lo;
        const int src_arr[2] = {prev, curr};
        const float *src[2];
        void *dst[2];
        for (int j = 0; j < 2; ++j) {
            src[j] = wsa(p, w, src_arr[j]) + off * g.pstride;
            if (g.host_store)
                dst[j] = p->hf[s] + (uint64_t)j * g.max_own * PB;
            else
                dst[j] = p->dstore[p->cur ^ 1][1 + j] + hoff(p, b.own_lo);
        }
        oocs_status r = k_encode(p, src, dst, 2, W, st, stats);
        if (r) return r;
        break;
    }
    case OOCS_OP_D2H: {
        const int64_t W = b.own_hi - b.own_lo;
        if (g.cfg.mode == OOCS_MODE_BASELINE) {
            const int curr = upd_array(g.k), prev = 3 - curr;
            const int64_t off = b.own_lo - b.ext_lo;
            CU(copy_1d(p->hstore[1] + hoff(p, b.own_lo), wsa(p, w, prev) + off * g.pstride, W * spb(p),
                       cudaMemcpyDeviceToHost, st, p->copy_chunk));
            CU(copy_1d(p->hstore[2] + hoff(p, b.own_lo), wsa(p, w, curr) + off * g.pstride, W * spb(p),
                       cudaMemcpyDeviceToHost, st, p->copy_chunk));
        } else {
            for (int j = 0; j < 2; ++j)
                CU(copy_1d(p->hstore[1 + j] + hoff(p, b.own_lo), p->hf[s] + (uint64_t)j * g.max_own * PB, W * PB,
                           cudaMemcpyDeviceToHost, st, p->copy_chunk));
        }
        if (stats) stats->bytes_d2h += (uint64_t)2 * W * spb(p);
        break;
    }
    case OOCS_OP_SEND: {
        // multi-GPU: this edge chunk's first (arg bit 0) / last (bit 1) kR encoded planes of S_{t+1},
        // straight from the encode output into the neighbour's ghost slot over NVLink (peer stores from
        // a copy kernel on this stream), then the neighbour's READY flag.  The slot of parity (t+1)&1
        // last held S_{t-1}: wait until the neighbour has consumed it (our FREE flag >= t).
        const uint32_t t1 = (uint32_t)(p->seq + o.sweep + 1);
        const int par = (int)(t1 & 1u);
        const int64_t kR = (int64_t)g.k * R, W = b.own_hi - b.own_lo;
        auto enc_out = [&](int j, int64_t plane_off) -> const uint8_t * {
            if (g.host_store) return p->hf[s] + ((uint64_t)j * g.max_own + plane_off) * PB;
            return p->dstore[p->cur ^ 1][1 + j] + hoff(p, b.own_lo + plane_off);
        };
        for (int side = 0; side < 2; ++side) {
            if (!((o.arg >> side) & 1)) continue;
            Plan::Peer &pr = p->peer[side];
            if (t1 >= 2)
                if (oocs_status r = wait_geq(st, &p->xflags[side ? F_FREE_HI : F_FREE_LO], t1 - 1)) return r;
            const int64_t off = side ? W - kR : 0;
            CU(launch_peer_copy(enc_out(0, off), pr.slot[par][0], enc_out(1, off), pr.slot[par][1], p->gh_bytes, st));
            if (stats) stats->copy_launches++;
            if (oocs_status r = write_flag(st, pr.flags + (side ? F_READY_LO : F_READY_HI), t1)) return r;
            if (stats) stats->bytes_exchange += 2 * p->gh_bytes;
        }
        break;
    }
    default:
        set_error("internal: unknown op");
        return OOCS_ERR_STATE;
    }
    return OOCS_OK;
}

// SEND and CARRY are kernel-stream ops too: SM copy kernels (SEND plus stream memory operations)
static bool is_kernel_op(int k) {
    return k == OOCS_OP_DECODE || k == OOCS_OP_STEP || k == OOCS_OP_ENCODE || k == OOCS_OP_SEND ||
           k == OOCS_OP_CARRY;
}
static bool is_work_op(int k) { return k != OOCS_OP_WAIT && k != OOCS_OP_RECORD; }

// OOCS_FLAG_TIMELINE: event pair around a work op
static oocs_status span_begin(Plan *p, const oocs_op &o, cudaStream_t st, size_t *idx) {
    const size_t n = p->spans.size();
    if (n == p->span_events.size()) {
        cudaEvent_t a, e;
        CU(cudaEventCreate(&a));
        if (cudaEventCreate(&e) != cudaSuccess) {
            cudaEventDestroy(a);
            CU(cudaErrorMemoryAllocation);
        }
        p->span_events.emplace_back(a, e);
    }
    oocs_span sp{};
    sp.kind = o.kind;
    sp.lane = o.lane;
    sp.g = o.g;
    sp.block = o.block;
    sp.sweep = o.sweep;
    sp.arg = o.arg;
    sp.host_ms = std::chrono::duration<double, std::milli>(std::chrono::steady_clock::now() - p->host_t0).count();
    p->spans.push_back(sp);
    CU(cudaEventRecord(p->span_events[n].first, st));
    *idx = n;
    return OOCS_OK;
}

// Executor 1 (OOCS_FLAG_LANE_SINGLE_STREAM / OOCS_FLAG_LANE_SPLIT_STREAMS): the schedule replayed onto
// CUDA streams in list order -- every lane one stream (Alg. 1 literally), or a copy and a kernel
// stream per lane joined by an event at every switch.  WAIT/RECORD become cudaStreamWaitEvent /
// cudaEventRecord.
static oocs_status execute_streams(Plan *p, const std::vector<oocs_op> &ops, int cur0, oocs_stats *stats) {
    const Geometry &g = p->geo;
    const bool tl = g.cfg.flags & OOCS_FLAG_TIMELINE;
    // a WAIT goes to the stream of the lane's next work op, a RECORD to the stream of its previous one
    auto work_stream = [&](const oocs_op &o) {
        return is_kernel_op(o.kind) ? p->klanes[o.lane] : p->lanes[o.lane];
    };
    std::vector<cudaStream_t> op_stream(ops.size());
    {
        std::vector<cudaStream_t> next(g.nstreams, nullptr), prev(g.nstreams, nullptr);
        for (size_t i = ops.size(); i-- > 0;) {
            const oocs_op &o = ops[i];
            if (is_work_op(o.kind)) next[o.lane] = work_stream(o);
            else if (o.kind == OOCS_OP_WAIT) op_stream[i] = next[o.lane] ? next[o.lane] : p->lanes[o.lane];
        }
        for (size_t i = 0; i < ops.size(); ++i) {
            const oocs_op &o = ops[i];
            if (is_work_op(o.kind)) op_stream[i] = prev[o.lane] = work_stream(o);
            else if (o.kind == OOCS_OP_RECORD) op_stream[i] = prev[o.lane] ? prev[o.lane] : p->lanes[o.lane];
        }
    }
    std::vector<cudaStream_t> last_work(g.nstreams, nullptr);
    for (size_t oi = 0; oi < ops.size(); ++oi) {
        const oocs_op &o = ops[oi];
        cudaStream_t st = op_stream[oi];
        if (o.kind == OOCS_OP_WAIT) {
            CU(cudaStreamWaitEvent(st, evt(p, o.arg, o.ev_g), 0));
            continue;
        }
        if (o.kind == OOCS_OP_RECORD) {
            CU(cudaEventRecord(evt(p, o.arg, o.ev_g), st));
            continue;
        }
        {
            // program order within the lane across its two streams
            cudaStream_t &lw = last_work[o.lane];
            if (lw && lw != st) {
                CU(cudaEventRecord(p->xfer_ev[o.lane], lw));
                CU(cudaStreamWaitEvent(st, p->xfer_ev[o.lane], 0));
            }
            lw = st;
        }
        size_t sp = 0;
        if (tl) {
            oocs_status r = span_begin(p, o, st, &sp);
            if (r) return r;
        }
        oocs_status r = issue_work(p, o, st, cur0, stats);
        if (r) return r;
        if (tl) CU(cudaEventRecord(p->span_events[sp].second, st));
    }
    return OOCS_OK;
}

// Watchdog: a run that makes no progress for OOCS_WATCHDOG_S seconds (default 600; 0 disables) is
// aborted -- in a multi-GPU job that means a neighbour stopped writing its flags.
static bool stalled_ok(Plan *p, std::chrono::steady_clock::time_point since) {
    static const double limit = [] {
        const char *e = std::getenv("OOCS_WATCHDOG_S");
        return e ? std::strtod(e, nullptr) : 600.0;
    }();
    if (limit <= 0) return true;
    if (std::chrono::duration<double>(std::chrono::steady_clock::now() - since).count() < limit) return true;
    set_error("no progress for " + std::to_string((int)limit) + " s (a multi-GPU neighbour stopped?); plan poisoned");
    p->poisoned = true;
    return false;
}

// Executor 2 (default): a host dispatcher over the schedule's dependency graph.  Every WAIT of the
// lowered schedule is resolved to the work op whose completion its event marks, and every work op
// depends on the previous work op of its lane (the lane's program order).  Kernels are issued in list
// order on their lane's kernel stream as soon as their dependencies are issued, with device-side
// waits on the dependencies' completion events.  A copy (H2D, CARRY, D2H) is issued only once its
// dependencies have COMPLETED (polled with cudaEventQuery), onto one stream per direction, so no copy
// stream ever holds a pending cross-stream wait: a copy channel blocked on a wait is re-examined by
// the copy-engine scheduler only between DMA commands, and with stream-mapped waits the decode of chunk
// g was measured to start only once the H2D of chunk g+1 had finished.  Same
// dependencies as the stream-mapped replay, so the same bytes.
static oocs_status execute_dispatch(Plan *p, const std::vector<oocs_op> &ops, int cur0, oocs_stats *stats,
                                    Plan::RunRec *prev) {
    const Geometry &g = p->geo;
    const bool tl = g.cfg.flags & OOCS_FLAG_TIMELINE;
    const size_t n = ops.size();
    const int slot = p->slot;
    Plan::RunRec &me = p->runs[slot];
    // producer of every event instance (kind, block counter) and the dependency lists; `fdeps` are the
    // dependencies on ops of the previous run (chained runs, `prev`): that run's ops are all issued, its
    // events live in the other slot's op_done pool
    std::vector<int64_t> dep_start(n + 1, 0), deps, fdep_start(n + 1, 0), fdeps;
    {
        std::vector<int64_t> last_work(g.nstreams, -1);
        for (auto &m : me.producer) m.clear();
        std::vector<std::vector<int64_t>> lane_waits(g.nstreams), lane_fwaits(g.nstreams);
        for (size_t i = 0; i < n; ++i) {
            const oocs_op &o = ops[i];
            dep_start[i] = (int64_t)deps.size();
            fdep_start[i] = (int64_t)fdeps.size();
            if (o.kind == OOCS_OP_RECORD) {
                if (last_work[o.lane] >= 0) me.producer[o.arg][o.ev_g] = last_work[o.lane];  // else records nothing
            } else if (o.kind == OOCS_OP_WAIT) {
                auto it = me.producer[o.arg].find(o.ev_g);
                if (it != me.producer[o.arg].end()) {
                    lane_waits[o.lane].push_back(it->second);
                } else if (prev) {  // an event of the previous run (cross-run RAW, working-buffer hand-off)
                    auto jt = prev->producer[o.arg].find(o.ev_g);
                    if (jt != prev->producer[o.arg].end()) lane_fwaits[o.lane].push_back(jt->second);
                }  // else: never recorded, or recorded by a run that has completed: a no-op
            } else {
                if (last_work[o.lane] >= 0) deps.push_back(last_work[o.lane]);
                else if (prev && o.lane < (int)prev->lane_last.size() && prev->lane_last[o.lane] >= 0)
                    fdeps.push_back(prev->lane_last[o.lane]);  // the lane's program continues across runs
                for (int64_t d : lane_waits[o.lane]) deps.push_back(d);
                for (int64_t d : lane_fwaits[o.lane]) fdeps.push_back(d);
                lane_waits[o.lane].clear();
                lane_fwaits[o.lane].clear();
                last_work[o.lane] = (int64_t)i;
            }
        }
        dep_start[n] = (int64_t)deps.size();
        fdep_start[n] = (int64_t)fdeps.size();
        // a run of a plan with no chained successor keeps lanes that never worked pointing at the
        // predecessor's last op on them (chains skip none, but keep the state total)
        me.lane_last.assign(g.nstreams, -1);
        for (int l = 0; l < g.nstreams; ++l) me.lane_last[l] = last_work[l];
    }
    std::vector<cudaEvent_t> &done_ev = p->op_done[slot];
    if (done_ev.size() < n) {
        const size_t old = done_ev.size();
        done_ev.resize(n, nullptr);
        for (size_t i = old; i < n; ++i)
            if (cudaEventCreateWithFlags(&done_ev[i], cudaEventDisableTiming) != cudaSuccess) {
                done_ev.resize(i);
                CU(cudaErrorMemoryAllocation);
            }
    }
    const std::vector<cudaEvent_t> *prev_ev = prev ? &p->op_done[slot ^ 1] : nullptr;
    auto stream_of = [&](const oocs_op &o) -> cudaStream_t {
        switch (o.kind) {
        case OOCS_OP_H2D: return p->cstream[0];
        case OOCS_OP_D2H: return p->cstream[1];
        default: return p->klanes[o.lane];  // kernels, and the SM-copy CARRY / SEND
        }
    };
    std::vector<char> issued(n, 0), done(n, 0);
    std::vector<cudaStream_t> where(n, nullptr);
    std::unordered_map<int64_t, char> fdone;  // completion of the previous run's ops polled so far
    for (size_t i = 0; i < n; ++i)
        if (!is_work_op(ops[i].kind)) issued[i] = done[i] = 1;
    // a query error other than NotReady is a sticky device fault: stop and poison the plan
    cudaError_t qerr = cudaSuccess;
    auto query = [&](cudaEvent_t e) -> bool {
        const cudaError_t r = cudaEventQuery(e);
        if (r == cudaSuccess) return true;
        if (r != cudaErrorNotReady) {
            qerr = r;
            (void)cudaGetLastError();
        }
        return false;
    };
    auto complete = [&](int64_t d) -> bool {
        if (done[d]) return true;
        if (query(done_ev[d])) done[d] = 1;
        return done[d];
    };
    auto fcomplete = [&](int64_t d) -> bool {
        char &f = fdone[d];
        if (!f && query((*prev_ev)[d])) f = 1;
        return f;
    };
    size_t first = 0;
    auto last_progress = std::chrono::steady_clock::now();
    // Run tail of a chainable plan: once only write-backs (D2H) are left, they are issued at once behind
    // device-side waits, so that the call returns -- and a chained next run starts its H2Ds -- without
    // waiting on the host for the last chunks' encodes (the D2H stream then holds those waits alone)
    // (same-box A/B, profiles/r02_tail_ab.json: chained c3 steps 2031-2037 vs 2076-2080 ms)
    const bool tail_ok = chainable(g) && !tl;
    bool tail = false;
    while (first < n) {
        if (tail_ok && !tail) {
            tail = true;
            for (size_t i = first; i < n && tail; ++i)
                if (!issued[i] && ops[i].kind != OOCS_OP_D2H) tail = false;
        }
        if (qerr != cudaSuccess) {
            set_error(std::string("device fault while executing the schedule: ") + cudaGetErrorString(qerr));
            return OOCS_ERR_CUDA;
        }
        if (!stalled_ok(p, last_progress)) return OOCS_ERR_EXCHANGE;
        bool progress = false;
        for (size_t i = first; i < n; ++i) {
            if (issued[i]) continue;
            const oocs_op &o = ops[i];
            const bool copy = !is_kernel_op(o.kind) && !tail;
            bool ready = true;
            for (int64_t k = dep_start[i]; k < dep_start[i + 1] && ready; ++k) {
                const int64_t d = deps[k];
                ready = issued[d] && (!copy || complete(d));
            }
            if (copy)
                for (int64_t k = fdep_start[i]; k < fdep_start[i + 1] && ready; ++k) ready = fcomplete(fdeps[k]);
            if (!ready) continue;
            cudaStream_t st = stream_of(o);
            if (!copy) {
                for (int64_t k = dep_start[i]; k < dep_start[i + 1]; ++k) {
                    const int64_t d = deps[k];
                    if (where[d] != st && !done[d]) CU(cudaStreamWaitEvent(st, done_ev[d], 0));
                }
                for (int64_t k = fdep_start[i]; k < fdep_start[i + 1]; ++k)
                    if (!fdone[fdeps[k]]) CU(cudaStreamWaitEvent(st, (*prev_ev)[fdeps[k]], 0));
            }
            size_t sp = 0;
            if (tl) {
                oocs_status r = span_begin(p, o, st, &sp);
                if (r) return r;
            }
            oocs_status r = issue_work(p, o, st, cur0, stats);
            if (r) return r;
            if (tl) CU(cudaEventRecord(p->span_events[sp].second, st));
            CU(cudaEventRecord(done_ev[i], st));
            issued[i] = 1;
            where[i] = st;
            progress = true;
        }
        while (first < n && issued[first]) ++first;
        if (progress) last_progress = std::chrono::steady_clock::now();
        else std::this_thread::yield();
    }
    return OOCS_OK;
}

static oocs_status execute(Plan *p, const std::vector<oocs_op> &ops, oocs_stats *stats, Plan::RunRec *prev) {
    const Geometry &g = p->geo;
    const int cur0 = p->cur;
    int64_t sweeps = 0;
    for (const oocs_op &o : ops) sweeps = std::max<int64_t>(sweeps, o.sweep + 1);
    oocs_status r = (g.cfg.flags & (OOCS_FLAG_LANE_SINGLE_STREAM | OOCS_FLAG_LANE_SPLIT_STREAMS))
                        ? execute_streams(p, ops, cur0, stats)
                        : execute_dispatch(p, ops, cur0, stats, prev);
    if (r) return r;
    p->cur = g.host_store ? cur0 : cur0 ^ (int)(sweeps & 1);
    return OOCS_OK;
}

// Complete the run in slot k (if it is still in flight): wait for its t1 mark, then its device time,
// kernel timings, spans and busy fractions; the stats go to p->finished.
static oocs_status finalize(Plan *p, int k) {
    Plan::RunRec &r = p->runs[k];
    if (!r.active) return OOCS_OK;
    r.active = false;
    const Geometry &g = p->geo;
    {
        // poll instead of blocking: a multi-GPU neighbour that never writes its flag must not hang the
        // process (the watchdog turns it into OOCS_ERR_EXCHANGE and a poisoned plan)
        const auto t_start = std::chrono::steady_clock::now();
        for (;;) {
            const cudaError_t e = cudaEventQuery(p->t1[k]);
            if (e == cudaSuccess) break;
            if (e != cudaErrorNotReady) CU(e);
            if (!stalled_ok(p, t_start)) return poison(p, OOCS_ERR_EXCHANGE);
            std::this_thread::sleep_for(std::chrono::microseconds(g.cfg.world > 1 ? 20 : 100));
        }
    }
    oocs_stats &stats = r.stats;
    float ms = 0.f;
    CU(cudaEventElapsedTime(&ms, p->t0[k], p->t1[k]));
    stats.wall_ms = ms;
    for (size_t i = 0; i < p->timing_used[k]; ++i) {
        float t = 0.f;
        CU(cudaEventElapsedTime(&t, p->timing_pool[k][i].a, p->timing_pool[k][i].b));
        stats.kernel_ms[p->timing_pool[k][i].kind] += t;
    }
    if (g.cfg.flags & OOCS_FLAG_TIMELINE) {  // timeline runs are never chained: p->spans are this run's
        for (size_t i = 0; i < p->spans.size(); ++i) {
            float a = 0.f, b = 0.f;
            CU(cudaEventElapsedTime(&a, p->t0[k], p->span_events[i].first));
            CU(cudaEventElapsedTime(&b, p->t0[k], p->span_events[i].second));
            p->spans[i].start_ms = a;
            p->spans[i].end_ms = b;
        }
        // busy time per engine = length of the union of its spans
        std::vector<std::pair<double, double>> iv[4];
        for (const oocs_span &sp : p->spans) {
            const int e = sp.kind == OOCS_OP_H2D ? 0 : sp.kind == OOCS_OP_D2H ? 1
                        : (sp.kind == OOCS_OP_DECODE || sp.kind == OOCS_OP_STEP || sp.kind == OOCS_OP_ENCODE) ? 2
                        : sp.kind == OOCS_OP_SEND ? 3 : -1;
            if (e >= 0) iv[e].emplace_back(sp.start_ms, sp.end_ms);
        }
        for (int e = 0; e < 4; ++e) {
            std::sort(iv[e].begin(), iv[e].end());
            double tot = 0, lo = 0, hi = -1;
            for (auto &x : iv[e]) {
                if (x.first > hi) {
                    if (hi > lo) tot += hi - lo;
                    lo = x.first;
                    hi = x.second;
                } else {
                    hi = std::max(hi, x.second);
                }
            }
            if (hi > lo) tot += hi - lo;
            stats.busy_ms[e] = tot;
        }
    }
    int herr = 0;
    CU(cudaMemcpy(&herr, p->d_err, sizeof(int), cudaMemcpyDeviceToHost));
    stats.data_error = herr;
    int64_t owned = 0;
    for (int i = g.b_lo; i < g.b_hi; ++i) owned += g.blocks[i].own_hi - g.blocks[i].own_lo;
    stats.cell_updates = (uint64_t)g.nx * g.ny * owned * r.steps;
    p->finished.push_back(stats);
    if (herr) {
        set_error("encoder rejected a non-finite or |x| >= 2^126 value (S:L200)");
        return OOCS_ERR_DATA;
    }
    return OOCS_OK;
}

// every run in flight, oldest first
static oocs_status finalize_all(Plan *p) {
    oocs_status st = finalize(p, p->slot ^ 1);
    const oocs_status st2 = finalize(p, p->slot);
    return st ? st : st2;
}

// Issue a run.  chain: the caller allows it to start while the previous run drains (oocs_run_async);
// it does so only for chainable plans (host store, codec modes, Algorithm 1, one rank) on the host
// dispatcher without a timeline.  Otherwise the previous run is finalized first.  Returns once every
// op of the run is issued; the run's t1 mark completes with its last op.
static oocs_status submit(Plan *p, int64_t steps, bool chain) {
    const Geometry &g = p->geo;
    if (steps < 0 || steps % g.k) {
        set_error("steps must be a non-negative multiple of tb_depth (S:L448)");
        return OOCS_ERR_CONFIG;
    }
    if (g.cfg.world > 1 && !p->connected) {
        set_error("world > 1: connect the neighbours first (oocs_peer_handle / oocs_peer_connect)");
        return OOCS_ERR_EXCHANGE;
    }
    CU(cudaSetDevice(g.cfg.device));
    const bool can = chain && chainable(g) &&
                     !(g.cfg.flags & (OOCS_FLAG_TIMELINE | OOCS_FLAG_LANE_SINGLE_STREAM | OOCS_FLAG_LANE_SPLIT_STREAMS));
    const int prev = p->slot;
    const bool chained = can && p->runs[prev].active;
    if (p->runs[prev].active && !chained)
        if (oocs_status st = finalize(p, prev)) return st;
    const int slot = prev ^ 1;
    if (p->runs[slot].active)  // two runs back: long done when chaining (its successor is fully issued)
        if (oocs_status st = finalize(p, slot)) return st;
    std::vector<oocs_op> ops;
    const int64_t sweeps = steps / g.k;
    lower_schedule(g, sweeps, ops, p->g_next);
    if (chainable(g)) p->g_next += sweeps * g.nb();
    p->slot = slot;
    p->timing_used[slot] = 0;
    p->spans.clear();
    p->host_t0 = std::chrono::steady_clock::now();
    Plan::RunRec &r = p->runs[slot];
    std::memset(&r.stats, 0, sizeof(r.stats));
    r.steps = steps;
    if (!chained) {
        // nothing in flight: clear the error flag, and anchor every stream at the run's start mark
        CU(cudaMemsetAsync(p->d_err, 0, sizeof(int), p->tstream));
        CU(cudaEventRecord(p->t0[slot], p->tstream));
        for (int l = 0; l < g.nstreams; ++l) CU(cudaStreamWaitEvent(p->lanes[l], p->t0[slot], 0));
        if (p->split)
            for (int l = 0; l < g.nstreams; ++l) CU(cudaStreamWaitEvent(p->klanes[l], p->t0[slot], 0));
        for (int c = 0; c < 3; ++c) CU(cudaStreamWaitEvent(p->cstream[c], p->t0[slot], 0));
    } else {
        // the mark follows the previous run's t1 on the timing stream: the time this run's first ops
        // overlap with the previous run's drain is counted once, in the previous run
        CU(cudaEventRecord(p->t0[slot], p->tstream));
    }
    oocs_status st = execute(p, ops, &r.stats, chained ? &p->runs[prev] : nullptr);
    if (st) return poison(p, st);
    // t1: after every stream's share of this run
    for (int l = 0; l < g.nstreams; ++l) {
        CU(cudaEventRecord(p->lane_done[l], p->lanes[l]));
        CU(cudaStreamWaitEvent(p->tstream, p->lane_done[l], 0));
        if (p->split) {
            CU(cudaEventRecord(p->kdone[l], p->klanes[l]));
            CU(cudaStreamWaitEvent(p->tstream, p->kdone[l], 0));
        }
    }
    for (int c = 0; c < 3; ++c) {
        CU(cudaEventRecord(p->cdone[c], p->cstream[c]));
        CU(cudaStreamWaitEvent(p->tstream, p->cdone[c], 0));
    }
    CU(cudaEventRecord(p->t1[slot], p->tstream));
    r.active = true;
    p->seq += sweeps;  // the store holds S_{seq} once this run completes
    return OOCS_OK;
}

static oocs_status run(Plan *p, int64_t steps, oocs_stats *out) {
    if (oocs_status st = submit(p, steps, false)) return st;
    p->finished.clear();
    oocs_status st = finalize(p, p->slot);
    if (out && !p->finished.empty()) *out = p->finished.back();
    p->finished.clear();
    return st;
}

// ---------------------------------------------------------------------------
// load / store
// ---------------------------------------------------------------------------
static oocs_status check_range(const Plan *p, int32_t array, int64_t a_lo, int64_t a_hi) {
    const Geometry &g = p->geo;
    if (array < 0 || array >= N_ARRAYS) {
        set_error("array must be 0 (velocity), 1 (p_prev) or 2 (p_curr)");
        return OOCS_ERR_CONFIG;
    }
    if (a_lo < g.a_store_lo() || a_hi > g.a_store_lo() + g.store_planes() || a_lo > a_hi || a_lo % 4 || a_hi % 4) {
        set_error("plane range outside this rank's store or not 4-aligned");
        return OOCS_ERR_CONFIG;
    }
    return OOCS_OK;
}

// Multi-GPU: the pressure ghost planes of a rank's store are a mirror of its ghost slots (the slots are
// what the pipeline reads and the neighbours write).  After a write into the store (load, write_raw) the
// ghost planes go to the slots of the current state; before a read they come back from them.
static oocs_status sync_ghosts(Plan *p, int32_t array, int64_t a_lo, int64_t a_hi, bool to_slots) {
    const Geometry &g = p->geo;
    if (g.cfg.world == 1 || array == 0) return OOCS_OK;
    const int64_t kR = (int64_t)g.k * R;
    const int par = (int)(p->seq & 1);
    for (int side = 0; side < 2; ++side) {
        if (side == 0 && g.cfg.rank == 0) continue;
        if (side == 1 && g.cfg.rank + 1 == g.cfg.world) continue;
        const int64_t z0 = side ? g.store_hi - kR : g.store_lo;  // interior planes of the ghost range
        if (a_hi <= z0 + R || z0 + kR + R <= a_lo) continue;
        uint8_t *slot = p->gh[side][par][array - 1];
        if (g.host_store) {
            uint8_t *h = p->hstore[array] + hoff(p, z0);
            if (to_slots) CU(cudaMemcpy(slot, h, p->gh_bytes, cudaMemcpyHostToDevice));
            else CU(cudaMemcpy(h, slot, p->gh_bytes, cudaMemcpyDeviceToHost));
        } else {
            uint8_t *d = p->dstore[p->cur][array] + hoff(p, z0);
            CU(cudaMemcpy(to_slots ? slot : d, to_slots ? d : slot, p->gh_bytes, cudaMemcpyDeviceToDevice));
        }
    }
    return OOCS_OK;
}

static oocs_status load(Plan *p, int32_t array, const float *src, int64_t a_lo, int64_t a_hi, bool dev_src) {
    oocs_status st = check_range(p, array, a_lo, a_hi);
    if (st) return st;
    const Geometry &g = p->geo;
    CU(cudaSetDevice(g.cfg.device));
    cudaStream_t s = p->lanes[0];
    const int64_t chunk = g.max_ext / 4 * 4;
    float *ws = p->ws[0][0];
    CU(cudaMemsetAsync(p->d_err, 0, 2 * sizeof(int), s));  // error flag and max|v|
    // staging for the compressed result (host store): reuse a slice of ws[0][1]
    uint8_t *stage = reinterpret_cast<uint8_t *>(p->ws[0][1]);
    for (int64_t a = a_lo; a < a_hi; a += chunk) {
        const int64_t n = std::min(chunk, a_hi - a);
        CU(copy_raw_to_ws(ws, src + (a - a_lo) * g.ax * g.ay, g, n,
                          dev_src ? cudaMemcpyDeviceToDevice : cudaMemcpyHostToDevice, s));
        if (array == 0) CU(launch_absmax(ws + XOFF, n * g.ay, g.ax, g.pitch, p->d_vmax, s));  // CFL check below
        const int64_t z = a - R;
        if (pitched_store(g)) {  // BASELINE: the store holds working-buffer rows
            CU(cudaMemcpyAsync(p->hstore[array] + hoff(p, z), ws, n * spb(p), cudaMemcpyDeviceToHost, s));
        } else if (g.host_store) {
            oocs_status r = k_encode(p, ws, stage, n, s, nullptr);
            if (r) return r;
            CU(cudaMemcpyAsync(p->hstore[array] + hoff(p, z), stage, n * pb(p), cudaMemcpyDeviceToHost, s));
            if (array == 0 && p->resident_vel)
                CU(cudaMemcpyAsync(p->dvel + hoff(p, z), stage, n * pb(p), cudaMemcpyDeviceToDevice, s));
        } else {
            for (int b = 0; b < (array == 0 ? 1 : 2); ++b) {
                oocs_status r = k_encode(p, ws, p->dstore[b][array] + hoff(p, z), n, s, nullptr);
                if (r) return r;
            }
            if (array == 0 && p->vdec) {  // the resident decoded velocity: decode of the same records
                oocs_status r = k_decode(p, p->dstore[0][0] + hoff(p, z), p->vdec + (z - g.store_lo) * g.pstride, n,
                                         s, nullptr);
                if (r) return r;
            }
        }
        CU(cudaStreamSynchronize(s));
    }
    if (oocs_status r = sync_ghosts(p, array, a_lo, a_hi, true)) return r;
    int herr[2] = {0, 0};
    CU(cudaMemcpy(herr, p->d_err, sizeof(herr), cudaMemcpyDeviceToHost));
    if (herr[0]) {
        set_error("oocs_load: non-finite or |x| >= 2^126 value for a lossy codec (S:L200)");
        return OOCS_ERR_DATA;
    }
    if (array == 0) {
        float vmax;
        std::memcpy(&vmax, &herr[1], sizeof(vmax));
        if (!((double)g.cfg.dt * (double)vmax <= cfl_limit(g.cfg.stencil))) {  // NaN fails too
            set_error("oocs_load: dt * max|v| = " + std::to_string((double)g.cfg.dt * vmax) +
                      " exceeds the stencil's CFL limit " + std::to_string(cfl_limit(g.cfg.stencil)) + " (DESIGN.md Q1)");
            return OOCS_ERR_CONFIG;
        }
    }
    return OOCS_OK;
}

static oocs_status store(Plan *p, int32_t array, float *dst, int64_t a_lo, int64_t a_hi, bool dev_dst) {
    oocs_status st = check_range(p, array, a_lo, a_hi);
    if (st) return st;
    const Geometry &g = p->geo;
    CU(cudaSetDevice(g.cfg.device));
    if (oocs_status r = sync_ghosts(p, array, a_lo, a_hi, false)) return r;
    cudaStream_t s = p->lanes[0];
    const int64_t chunk = g.max_ext / 4 * 4;
    float *ws = p->ws[0][0];
    uint8_t *stage = reinterpret_cast<uint8_t *>(p->ws[0][1]);
    for (int64_t a = a_lo; a < a_hi; a += chunk) {
        const int64_t n = std::min(chunk, a_hi - a);
        const int64_t z = a - R;
        const void *src;
        if (pitched_store(g)) {
            CU(cudaMemcpyAsync(ws, p->hstore[array] + hoff(p, z), n * spb(p), cudaMemcpyHostToDevice, s));
        } else {
            if (g.host_store) {
                CU(cudaMemcpyAsync(stage, p->hstore[array] + hoff(p, z), n * pb(p), cudaMemcpyHostToDevice, s));
                src = stage;
            } else {
                src = p->dstore[array == 0 ? 0 : p->cur][array] + hoff(p, z);
            }
            oocs_status r = k_decode(p, src, ws, n, s, nullptr);
            if (r) return r;
        }
        CU(copy_ws_to_raw(dst + (a - a_lo) * g.ax * g.ay, ws, g, n,
                          dev_dst ? cudaMemcpyDeviceToDevice : cudaMemcpyDeviceToHost, s));
        CU(cudaStreamSynchronize(s));
    }
    return OOCS_OK;
}

static oocs_status raw_io(Plan *p, int32_t array, void *host, int64_t a_lo, int64_t a_hi, bool write) {
    oocs_status st = check_range(p, array, a_lo, a_hi);
    if (st) return st;
    const Geometry &g = p->geo;
    CU(cudaSetDevice(g.cfg.device));
    if (!write)
        if (oocs_status r = sync_ghosts(p, array, a_lo, a_hi, false)) return r;
    const uint64_t off = hoff(p, a_lo - R), n = (uint64_t)(a_hi - a_lo) * pb(p);
    if (pitched_store(g)) {  // raw bytes are the identity codec's planes (rows of ax floats)
        const int64_t rows = (a_hi - a_lo) * g.ay;
        uint8_t *base = p->hstore[array] + off + XOFF * 4;
        for (int64_t r = 0; r < rows; ++r) {
            uint8_t *st_row = base + (uint64_t)r * g.pitch * 4;
            uint8_t *h_row = static_cast<uint8_t *>(host) + (uint64_t)r * g.ax * 4;
            if (write) std::memcpy(st_row, h_row, g.ax * 4);
            else std::memcpy(h_row, st_row, g.ax * 4);
        }
        return OOCS_OK;
    }
    if (g.host_store) {
        if (write) {
            std::memcpy(p->hstore[array] + off, host, n);
            if (array == 0 && p->resident_vel) CU(cudaMemcpy(p->dvel + off, host, n, cudaMemcpyHostToDevice));
        } else {
            std::memcpy(host, p->hstore[array] + off, n);
        }
        return OOCS_OK;
    }
    if (write) {
        for (int b = 0; b < (array == 0 ? 1 : 2); ++b)
            CU(cudaMemcpy(p->dstore[b][array] + off, host, n, cudaMemcpyHostToDevice));
        if (array == 0 && p->vdec) {
            oocs_status r = k_decode(p, p->dstore[0][0] + off, p->vdec + (a_lo - R - g.store_lo) * g.pstride,
                                     a_hi - a_lo, p->lanes[0], nullptr);
            if (r) return r;
            CU(cudaStreamSynchronize(p->lanes[0]));
        }
    } else {
        CU(cudaMemcpy(host, p->dstore[array == 0 ? 0 : p->cur][array] + off, n, cudaMemcpyDeviceToHost));
    }
    return OOCS_OK;
}

}  // namespace oocs

// ===========================================================================
// C ABI
// ===========================================================================
using namespace oocs;

// the exchange-region handle oocs_peer_handle exports (OOCS_PEER_HANDLE_BYTES)
constexpr uint64_t PEER_MAGIC = 0x5245455053434f4fULL;  // "OOCSPEER"
struct PeerBlob {
    uint64_t magic;
    uint32_t version, pid;
    int32_t device, rank, world, k, codec, pad;
    int64_t nx, ny, nz, plane_bytes;
    uint64_t gh_bytes, xreg_bytes, dev_ptr;
    cudaIpcMemHandle_t ipc;
};
static_assert(sizeof(PeerBlob) <= OOCS_PEER_HANDLE_BYTES, "peer handle blob too large");

static oocs_status guard(const oocs_plan *p) {
    if (!p) {
        set_error("plan is NULL");
        return OOCS_ERR_STATE;
    }
    if (p->poisoned) {
        set_error("plan poisoned by an earlier CUDA error; only oocs_destroy is valid");
        return OOCS_ERR_STATE;
    }
    return OOCS_OK;
}

extern "C" {

oocs_status oocs_plan_create(const oocs_config *cfg, oocs_plan **out) {
    if (!out) {
        set_error("out is NULL");
        return OOCS_ERR_CONFIG;
    }
    *out = nullptr;
    Plan *p = nullptr;
    oocs_status st = create(cfg, &p);
    if (st == OOCS_OK) *out = static_cast<oocs_plan *>(p);
    return st;
}

oocs_status oocs_plan_create_in(const oocs_config *cfg, void *arena, uint64_t arena_bytes, oocs_plan **out) {
    if (!out || !arena) {
        set_error("out or arena is NULL");
        return OOCS_ERR_CONFIG;
    }
    *out = nullptr;
    Plan *p = nullptr;
    oocs_status st = create(cfg, &p, arena, arena_bytes);
    if (st == OOCS_OK) *out = static_cast<oocs_plan *>(p);
    return st;
}

oocs_status oocs_plan_query(const oocs_plan *plan, oocs_plan_info *info) {
    if (oocs_status st = guard(plan)) return st;
    if (!info) return OOCS_ERR_CONFIG;
    fill_info(plan->geo, compute_sizes(plan->geo), info);
    return OOCS_OK;
}

oocs_status oocs_plan_estimate(const oocs_config *cfg, oocs_plan_info *info) {
    if (!info) return OOCS_ERR_CONFIG;
    Geometry g;
    std::string err;
    oocs_status st = make_geometry(cfg, &g, &err);
    if (st != OOCS_OK) {
        set_error(err);
        return st;
    }
    fill_info(g, compute_sizes(g), info);
    return OOCS_OK;
}

oocs_status oocs_peer_handle(const oocs_plan *plan, void *out) {
    if (oocs_status st = guard(plan)) return st;
    if (!out) {
        set_error("oocs_peer_handle: out is NULL");
        return OOCS_ERR_CONFIG;
    }
    if (!plan->xreg) {
        set_error("oocs_peer_handle: world == 1, the plan has no exchange region");
        return OOCS_ERR_STATE;
    }
    const Geometry &g = plan->geo;
    CU(cudaSetDevice(g.cfg.device));
    PeerBlob b;
    std::memset(&b, 0, sizeof(b));
    b.magic = PEER_MAGIC;
    b.version = OOCS_ABI_VERSION;
    b.pid = (uint32_t)getpid();
    b.device = g.cfg.device;
    b.rank = g.cfg.rank;
    b.world = g.cfg.world;
    b.k = g.k;
    b.nx = g.nx;
    b.ny = g.ny;
    b.nz = g.nz;
    b.plane_bytes = g.plane_bytes;
    b.gh_bytes = plan->gh_bytes;
    b.xreg_bytes = plan->xreg_bytes;
    b.dev_ptr = (uint64_t)(uintptr_t)plan->xreg;
    b.codec = g.codec;
    CU(cudaIpcGetMemHandle(&b.ipc, plan->xreg));
    std::memset(out, 0, OOCS_PEER_HANDLE_BYTES);
    std::memcpy(out, &b, sizeof(b));
    return OOCS_OK;
}

oocs_status oocs_peer_connect(oocs_plan *plan, const void *lower, const void *upper) {
    if (oocs_status st = guard(plan)) return st;
    const Geometry &g = plan->geo;
    if (!plan->xreg) {
        set_error("oocs_peer_connect: world == 1, nothing to connect");
        return OOCS_ERR_STATE;
    }
    const void *blob[2] = {lower, upper};
    const bool need[2] = {g.cfg.rank > 0, g.cfg.rank + 1 < g.cfg.world};
    PeerBlob pb2[2];
    for (int side = 0; side < 2; ++side) {
        if (!need[side]) continue;
        if (!blob[side]) {
            set_error(side ? "oocs_peer_connect: upper (rank+1) handle missing" : "oocs_peer_connect: lower (rank-1) handle missing");
            return OOCS_ERR_CONFIG;
        }
        std::memcpy(&pb2[side], blob[side], sizeof(PeerBlob));
        const PeerBlob &b = pb2[side];
        if (b.magic != PEER_MAGIC || b.version != OOCS_ABI_VERSION || b.world != g.cfg.world ||
            b.rank != g.cfg.rank + (side ? 1 : -1) || b.k != g.k || b.nx != g.nx || b.ny != g.ny || b.nz != g.nz ||
            b.plane_bytes != g.plane_bytes || b.codec != g.codec || b.gh_bytes != plan->gh_bytes ||
            b.xreg_bytes != plan->xreg_bytes) {
            set_error("oocs_peer_connect: the handle is not the neighbour's of the same job geometry");
            return OOCS_ERR_CONFIG;
        }
    }
    CU(cudaSetDevice(g.cfg.device));
    for (auto &pr : plan->peer) {  // re-connect: drop the previous mappings
        if (pr.ipc && pr.base) cudaIpcCloseMemHandle(pr.base);
        pr = Plan::Peer{};
    }
    plan->connected = false;
    for (int side = 0; side < 2; ++side) {
        if (!need[side]) continue;
        const PeerBlob &b = pb2[side];
        Plan::Peer &pr = plan->peer[side];
        if (b.pid == (uint32_t)getpid()) {  // same process: the pointer itself
            if (b.device == g.cfg.device) {
                // one context would hold both ranks' streams: a rank's flag wait at the head of a hardware
                // queue could block the neighbour's producing work queued behind it (false dependency)
                set_error("oocs_peer_connect: ranks sharing one device must be separate processes");
                return OOCS_ERR_CONFIG;
            }
            pr.base = reinterpret_cast<uint8_t *>((uintptr_t)b.dev_ptr);
            if (b.device != g.cfg.device) {
                const cudaError_t e = cudaDeviceEnablePeerAccess(b.device, 0);
                if (e != cudaSuccess && e != cudaErrorPeerAccessAlreadyEnabled) {
                    cudaGetLastError();
                    set_error(std::string("oocs_peer_connect: peer access failed: ") + cudaGetErrorString(e));
                    return OOCS_ERR_EXCHANGE;
                }
                cudaGetLastError();
            }
        } else {
            void *ptr = nullptr;
            const cudaError_t e = cudaIpcOpenMemHandle(&ptr, b.ipc, cudaIpcMemLazyEnablePeerAccess);
            if (e != cudaSuccess) {
                cudaGetLastError();
                set_error(std::string("oocs_peer_connect: cudaIpcOpenMemHandle failed: ") + cudaGetErrorString(e));
                return OOCS_ERR_EXCHANGE;
            }
            pr.base = static_cast<uint8_t *>(ptr);
            pr.ipc = true;
        }
        // we write the lower neighbour's upper slots and the upper neighbour's lower slots
        for (int par = 0; par < 2; ++par)
            for (int j = 0; j < 2; ++j) pr.slot[par][j] = pr.base + slot_off(plan->gh_bytes, 1 - side, par, j);
        pr.flags = reinterpret_cast<uint32_t *>(pr.base);
    }
    plan->connected = true;
    return OOCS_OK;
}

oocs_status oocs_destroy(oocs_plan *plan) {
    if (plan && !plan->poisoned) (void)finalize_all(plan);  // let runs in flight finish before freeing
    free_plan(static_cast<Plan *>(plan));
    return OOCS_OK;
}

oocs_status oocs_load(oocs_plan *plan, int32_t array, const float *src, int64_t a_lo, int64_t a_hi) {
    if (oocs_status st = guard(plan)) return st;
    if (oocs_status st = poison(plan, finalize_all(plan))) return st;  // runs in flight complete first
    return poison(plan, load(plan, array, src, a_lo, a_hi, false));
}

oocs_status oocs_load_device(oocs_plan *plan, int32_t array, const float *src, int64_t a_lo, int64_t a_hi) {
    if (oocs_status st = guard(plan)) return st;
    if (oocs_status st = poison(plan, finalize_all(plan))) return st;  // runs in flight complete first
    return poison(plan, load(plan, array, src, a_lo, a_hi, true));
}

oocs_status oocs_store(oocs_plan *plan, int32_t array, float *dst, int64_t a_lo, int64_t a_hi) {
    if (oocs_status st = guard(plan)) return st;
    if (oocs_status st = poison(plan, finalize_all(plan))) return st;  // runs in flight complete first
    return poison(plan, store(plan, array, dst, a_lo, a_hi, false));
}

oocs_status oocs_store_device(oocs_plan *plan, int32_t array, float *dst, int64_t a_lo, int64_t a_hi) {
    if (oocs_status st = guard(plan)) return st;
    if (oocs_status st = poison(plan, finalize_all(plan))) return st;  // runs in flight complete first
    return poison(plan, store(plan, array, dst, a_lo, a_hi, true));
}

oocs_status oocs_store_read_raw(oocs_plan *plan, int32_t array, void *dst, int64_t a_lo, int64_t a_hi) {
    if (oocs_status st = guard(plan)) return st;
    if (oocs_status st = poison(plan, finalize_all(plan))) return st;  // runs in flight complete first
    return poison(plan, raw_io(plan, array, dst, a_lo, a_hi, false));
}

oocs_status oocs_store_write_raw(oocs_plan *plan, int32_t array, const void *src, int64_t a_lo, int64_t a_hi) {
    if (oocs_status st = guard(plan)) return st;
    if (oocs_status st = poison(plan, finalize_all(plan))) return st;  // runs in flight complete first
    return poison(plan, raw_io(plan, array, const_cast<void *>(src), a_lo, a_hi, true));
}

oocs_status oocs_run(oocs_plan *plan, int64_t steps, oocs_stats *out) {
    if (oocs_status st = guard(plan)) return st;
    return poison(plan, run(plan, steps, out));
}

oocs_status oocs_run_async(oocs_plan *plan, int64_t steps) {
    if (oocs_status st = guard(plan)) return st;
    return poison(plan, submit(plan, steps, true));
}

oocs_status oocs_wait(oocs_plan *plan, oocs_stats *out, int64_t cap, int64_t *n_runs) {
    if (oocs_status st = guard(plan)) return st;
    if (cap < 0 || (cap > 0 && !out)) {
        set_error("oocs_wait: out is NULL or cap < 0");
        return OOCS_ERR_CONFIG;
    }
    const oocs_status st = poison(plan, finalize_all(plan));
    const int64_t n = (int64_t)plan->finished.size();
    if (n_runs) *n_runs = n;
    for (int64_t i = 0; i < std::min(n, cap); ++i) out[i] = plan->finished[i];
    plan->finished.clear();
    return st;
}

oocs_status oocs_timeline(const oocs_plan *plan, oocs_span *out, int64_t cap, int64_t *n_spans) {
    if (oocs_status st = guard(plan)) return st;
    if (oocs_status st = finalize_all(const_cast<oocs_plan *>(plan))) return st;
    if (!n_spans || cap < 0) {
        set_error("oocs_timeline: n_spans is NULL or cap < 0");
        return OOCS_ERR_CONFIG;
    }
    const int64_t n = (int64_t)plan->spans.size();
    *n_spans = n;
    if (out)
        for (int64_t i = 0; i < std::min(n, cap); ++i) out[i] = plan->spans[i];
    return OOCS_OK;
}

oocs_status oocs_decode(const void *src, float *dst, int64_t ax, int64_t ay, int64_t planes, int64_t pitch,
                        int32_t codec, int32_t rate_bits, void *stream) {
    if (ax % 4 || ay % 4 || planes % 4 || pitch < ax + XOFF || pitch % 32 || codec < 0 || codec > 3 ||
        (codec == 1 && (rate_bits < 2 || rate_bits > 24)) || (codec == 2 && (rate_bits < 1 || rate_bits > 32)) ||
        (codec == 3 && rate_bits != 16)) {
        set_error("oocs_decode: bad geometry or codec");
        return OOCS_ERR_CONFIG;
    }
    const int qk = codec == 1 ? rate_bits - 1 : codec == 2 ? rate_bits : 0;
    CU(launch_decode(&src, &dst, 1, ax, ay, planes, pitch, codec, qk, (cudaStream_t)stream));
    return OOCS_OK;
}

oocs_status oocs_encode(const float *src, void *dst, int64_t ax, int64_t ay, int64_t planes, int64_t pitch,
                        int32_t codec, int32_t rate_bits, int32_t *err_flag, void *stream) {
    if (ax % 4 || ay % 4 || planes % 4 || pitch < ax + XOFF || pitch % 32 || codec < 0 || codec > 3 ||
        (codec == 1 && (rate_bits < 2 || rate_bits > 24)) || (codec == 2 && (rate_bits < 1 || rate_bits > 32)) ||
        (codec == 3 && rate_bits != 16)) {
        set_error("oocs_encode: bad geometry or codec");
        return OOCS_ERR_CONFIG;
    }
    const int qk = codec == 1 ? rate_bits - 1 : codec == 2 ? rate_bits : 0;
    int *flag = err_flag;
    if (!flag) {
        // the caller does not want the flag: a per-device scratch word, allocated once
        static std::mutex mu;
        static int *scratch[64] = {};
        int dev = 0;
        CU(cudaGetDevice(&dev));
        std::lock_guard<std::mutex> lk(mu);
        if (dev < 0 || dev >= 64) {
            set_error("device ordinal out of range");
            return OOCS_ERR_CONFIG;
        }
        if (!scratch[dev]) CU(cudaMalloc((void **)&scratch[dev], sizeof(int)));
        flag = scratch[dev];
    }
    CU(launch_encode(&src, &dst, 1, ax, ay, planes, pitch, codec, qk, flag, (cudaStream_t)stream));
    return OOCS_OK;
}

oocs_status oocs_step(const float *vel, float *p_prev, const float *p_curr, int64_t ax, int64_t ay, int64_t planes,
                      int64_t pitch, float dt, int64_t z_lo, int64_t z_hi, int32_t stencil, void *stream) {
    if (ax % 4 || ay % 4 || pitch < ax + XOFF || pitch % 32 || z_lo < R || z_hi > planes - R || z_lo > z_hi ||
        (stencil != OOCS_STENCIL_ACOUSTIC25 && stencil != OOCS_STENCIL_STAR7)) {
        set_error("oocs_step: bad geometry, plane range or stencil");
        return OOCS_ERR_CONFIG;
    }
    CU(launch_step(vel, p_prev, p_curr, ax, ay, pitch, planes, z_lo, z_hi, dt, stencil, (cudaStream_t)stream));
    return OOCS_OK;
}

const char *oocs_last_error(void) { return g_last_error.c_str(); }
int32_t oocs_abi_version(void) { return OOCS_ABI_VERSION; }

void oocs_abi_sizes(int64_t out[6]) {
    out[0] = sizeof(oocs_config);
    out[1] = sizeof(oocs_stats);
    out[2] = sizeof(oocs_plan_info);
    out[3] = sizeof(oocs_block);
    out[4] = sizeof(oocs_op);
    out[5] = sizeof(oocs_span);
}

}  // extern "C"
