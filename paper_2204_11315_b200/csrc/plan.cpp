// Host-side planning: configuration validation, z-chunk decomposition with
// temporal-blocking halos and region-sharing overlaps (§3.1,
// S:L42-61), and the lowering of Algorithm 1 plus the hazard
// edges it leaves implicit to a per-lane
// operation list.  Pure functions: no CUDA calls, testable on a CPU box
// through oocs_plan_table / oocs_schedule.
#include <algorithm>
#include <cmath>
#include <cstring>
#include <functional>

#include "oocs_internal.h"

namespace oocs {

static bool bad(std::string *err, const std::string &msg) {
    if (err) *err = msg;
    return false;
}

static bool validate(const oocs_config *c, std::string *err) {
    if (!c) return bad(err, "config is NULL");
    if (c->struct_size != sizeof(oocs_config)) return bad(err, "oocs_config.struct_size mismatch (ABI version)");
    if (c->nx <= 0 || c->ny <= 0 || c->nz <= 0) return bad(err, "grid dimensions must be positive");
    if (c->nx % 4 || c->ny % 4 || c->nz % 4) return bad(err, "nx, ny, nz must be multiples of 4 (4x4x4 codec blocks)");
    if (!(c->dt > 0.0f) || !std::isfinite(c->dt)) return bad(err, "dt must be positive and finite");
    if (c->stencil != OOCS_STENCIL_ACOUSTIC25 && c->stencil != OOCS_STENCIL_STAR7) return bad(err, "unknown stencil");
    if (!(c->v_max >= 0.0f) || !std::isfinite(c->v_max)) return bad(err, "v_max must be finite and >= 0 (0 = undeclared)");
    if ((double)c->dt * (double)c->v_max > cfl_limit(c->stencil))
        return bad(err, "dt * v_max exceeds the stencil's CFL limit (" + std::to_string(cfl_limit(c->stencil)) +
                            "; DESIGN.md Q1)");
    if (c->codec != OOCS_CODEC_IDENTITY && c->codec != OOCS_CODEC_BLOCKQUANT && c->codec != OOCS_CODEC_ZFP &&
        c->codec != OOCS_CODEC_TRUNC16)
        return bad(err, "unknown codec");
    if (c->codec == OOCS_CODEC_TRUNC16 && c->rate_bits != 16) return bad(err, "Truncate-16 has rate_bits 16");
    if (c->codec == OOCS_CODEC_ZFP && (c->rate_bits < 1 || c->rate_bits > 32))
        return bad(err, "ZFP rate_bits must be in [1, 32] (64*rate bits per 4x4x4 block)");
    if (c->codec == OOCS_CODEC_BLOCKQUANT && (c->rate_bits < 2 || c->rate_bits > 24))
        return bad(err, "BlockQuant rate_bits must be in [2, 24] (q = rate-1 code bits)");
    if (c->mode < OOCS_MODE_BASELINE || c->mode > OOCS_MODE_COMPRESS_DWB) return bad(err, "unknown mode");
    if (c->mode == OOCS_MODE_BASELINE && c->codec != OOCS_CODEC_IDENTITY)
        return bad(err, "BASELINE mode (fig:3ver(a)) moves uncompressed data: codec must be identity");
    if (c->store != OOCS_STORE_HOST && c->store != OOCS_STORE_DEVICE) return bad(err, "unknown store kind");
    if (c->store == OOCS_STORE_HOST && !c->region_sharing)
        return bad(err, "an in-place host store requires region sharing (the overlap of chunk i+1 is overwritten "
                        "by chunk i's write-back; SURVEY §8(a) a3)");
    if (c->n_blocks < 1 || c->tb_depth < 1) return bad(err, "n_blocks and tb_depth must be >= 1");
    if (c->nz / 4 < c->n_blocks) return bad(err, "more chunks than 4-plane units: empty chunk (S:L57)");
    if (c->world < 1 || c->rank < 0 || c->rank >= c->world) return bad(err, "bad rank/world");
    if (c->n_blocks % c->world) return bad(err, "world must divide n_blocks (whole chunks per GPU)");
    if (c->world > 1 && c->mode == OOCS_MODE_BASELINE)
        return bad(err, "the uncompressed BASELINE (fig:3ver(a)) is a single-GPU comparison: world must be 1");
    if (c->device < 0) return bad(err, "bad device ordinal");
    if (c->flags & ~(uint32_t)(OOCS_FLAG_PROFILE | OOCS_FLAG_RESIDENT_VELOCITY | OOCS_FLAG_TIMELINE |
                               OOCS_FLAG_LANE_SINGLE_STREAM | OOCS_FLAG_LANE_SPLIT_STREAMS | OOCS_FLAG_DECODED_VELOCITY |
                               OOCS_FLAG_FUSE_DECODE))
        return bad(err, "unknown or retired flag (4 = ABI 1's fused last step + encode, removed)");
    if ((c->flags & OOCS_FLAG_RESIDENT_VELOCITY) && (c->store != OOCS_STORE_HOST || c->mode == OOCS_MODE_BASELINE))
        return bad(err, "OOCS_FLAG_RESIDENT_VELOCITY applies to host-store codec modes only");
    if ((c->flags & OOCS_FLAG_DECODED_VELOCITY) && c->store != OOCS_STORE_DEVICE)
        return bad(err, "OOCS_FLAG_DECODED_VELOCITY applies to the device store only");
    if ((c->flags & OOCS_FLAG_FUSE_DECODE) &&
        (c->mode == OOCS_MODE_BASELINE || c->codec != OOCS_CODEC_BLOCKQUANT || c->rate_bits > 16 || (c->rate_bits & 1) ||
         c->stencil != OOCS_STENCIL_ACOUSTIC25))
        return bad(err, "OOCS_FLAG_FUSE_DECODE applies to codec modes with BlockQuant at an even rate <= 16 and the "
                        "25-point stencil");
    if (c->schedule < OOCS_SCHED_ALG1 || c->schedule > OOCS_SCHED_DAG_FUNC) return bad(err, "unknown schedule kind");
    if (c->n_lanes != 0 && (c->n_lanes < 2 || c->n_lanes > MAX_LANES)) return bad(err, "n_lanes must be 0 (=3) or 2..8");
    return true;
}

oocs_status make_geometry(const oocs_config *cfg, Geometry *g, std::string *err) {
    if (!validate(cfg, err)) return OOCS_ERR_CONFIG;
    const oocs_config &c = *cfg;
    g->cfg = c;
    g->nx = c.nx;
    g->ny = c.ny;
    g->nz = c.nz;
    g->ax = c.nx + 2 * R;
    g->ay = c.ny + 2 * R;
    g->az = c.nz + 2 * R;
    g->pitch = (XOFF + g->ax + 31) / 32 * 32;
    g->pstride = g->ay * g->pitch;
    g->codec = c.codec;
    // kernel parameter: q = r - 1 code bits for BlockQuant, the rate itself for ZFP
    g->q = c.codec == OOCS_CODEC_BLOCKQUANT ? c.rate_bits - 1 : c.codec == OOCS_CODEC_ZFP ? c.rate_bits : 0;
    g->plane_bytes = c.codec == OOCS_CODEC_IDENTITY  ? g->ax * g->ay * 4
                     : c.codec == OOCS_CODEC_TRUNC16 ? g->ax * g->ay * 2
                                                     : (g->ax / 4) * (g->ay / 4) * 8 * c.rate_bits / 4;
    g->k = c.tb_depth;
    const int n = c.n_blocks;
    const int64_t kR = (int64_t)c.tb_depth * R;
    // owned planes: 4-plane units, remainder to the leading chunks (Q5)
    const int64_t units = c.nz / 4, base = units / n, rem = units % n;
    g->blocks.assign(n, oocs_block{});
    int64_t lo = 0;
    for (int i = 0; i < n; ++i) {
        const int64_t w = 4 * (base + (i < rem ? 1 : 0));
        if (kR >= w) {
            if (err) *err = "k*R must be smaller than every chunk's owned width (S:L57)";
            return OOCS_ERR_CONFIG;
        }
        oocs_block &b = g->blocks[i];
        b.own_lo = lo;
        b.own_hi = lo + w;
        b.ext_lo = std::max<int64_t>(-R, b.own_lo - kR);
        b.ext_hi = std::min<int64_t>(c.nz + R, b.own_hi + kR);
        // the previous chunk's extent reaches own_lo + kR: that overlap stays on the GPU
        if (i > 0 && c.region_sharing) {
            b.carry_lo = b.own_lo - kR;
            b.carry_hi = b.own_lo + kR;
        } else {
            b.carry_lo = b.carry_hi = b.ext_lo;
        }
        b.body_lo = b.carry_hi;
        b.body_hi = b.ext_hi;
        lo = b.own_hi;
    }
    g->b_lo = (int)((int64_t)c.rank * n / c.world);
    g->b_hi = (int)((int64_t)(c.rank + 1) * n / c.world);
    // a rank's first chunk has no predecessor on this GPU: no carry (its pressure halo below the slab
    // arrives in a ghost slot from rank-1, its velocity halo is in the store)
    oocs_block &first = g->blocks[g->b_lo];
    first.carry_lo = first.carry_hi = first.body_lo = first.ext_lo;
    g->store_lo = std::max<int64_t>(-R, g->blocks[g->b_lo].own_lo - kR);
    g->store_hi = std::min<int64_t>(c.nz + R, g->blocks[g->b_hi - 1].own_hi + kR);
    g->max_ext = g->max_own = 0;
    for (int i = g->b_lo; i < g->b_hi; ++i) {
        g->max_ext = std::max(g->max_ext, g->blocks[i].ext_hi - g->blocks[i].ext_lo);
        g->max_own = std::max(g->max_own, g->blocks[i].own_hi - g->blocks[i].own_lo);
    }
    g->host_store = c.store == OOCS_STORE_HOST;
    g->lanes = c.n_lanes ? c.n_lanes : 3;
    // the by-function DAG schedule runs its ops on three streams (H2D + carry / kernels / D2H) whatever the
    // number of staging slots
    g->nstreams = (g->host_store && c.schedule == OOCS_SCHED_DAG_FUNC) ? std::max(g->lanes, 3) : g->lanes;
    if (!g->host_store)
        g->n_ws = 1;
    else  // SWB: one working buffer; DWB: two; BASELINE / COMPRESS: one per stream (fig:3ver)
        g->n_ws = c.mode == OOCS_MODE_COMPRESS_SWB ? 1 : c.mode == OOCS_MODE_COMPRESS_DWB ? 2 : g->lanes;
    return OOCS_OK;
}

// ---------------------------------------------------------------------------
// Lowering.  g = global block counter (sweep * nb + local block), lane
// s(g) = g mod 3 (S:L425 repair of Algorithm 1's never-updated si), working
// set w(g) = g mod n_ws.  Codec modes follow Algorithm 1 line by line:
//   iteration g:  [lane s(g)] WAIT evt_h2d(g-1); CARRY(g); RECORD evt_carry(g)
//                      (region sharing: the overlap is copied GPU-side out of the
//                      previous chunk's half-size buffer before that buffer is reused)
//                 [deferred tail of g-1 on lane s(g-1)]
//                 WAIT evt_carry(g); ENCODE(g-1) into hf_buf[s(g-1)]; RECORD evt_enc(g-1);
//                 D2H(g-1); RECORD evt_d2h(g-1)
//                 [head of g on lane s(g)]
//                 WAIT evt_d2h of the previous sweep's chunks whose owned planes this
//                      H2D reads (cross-sweep RAW on the in-place host store, a10)
//                 H2D(g) body into hf_buf[s(g)]; RECORD evt_h2d(g)
//                 WAIT evt_enc(g - n_ws)         (working-buffer hand-off)
//                 DECODE(g); RECORD evt_dec(g); STEP(g, 1..k)
//   drain epilogue after the loop.
// ---------------------------------------------------------------------------
namespace {
struct Emitter {
    std::vector<oocs_op> &ops;
    void emit(int kind, int lane, int64_t g, int block, int sweep, int arg = 0, int64_t ev_g = -1) {
        oocs_op o;
        std::memset(&o, 0, sizeof(o));
        o.kind = kind;
        o.lane = lane;
        o.g = g;
        o.block = block;
        o.sweep = sweep;
        o.arg = arg;
        o.ev_g = ev_g;
        ops.push_back(o);
    }
};
}  // namespace

// multi-GPU: which of a chunk's edges go to a neighbour's ghost slot after its encode (bit 0: its first
// kR owned planes to rank-1, bit 1: its last kR owned planes to rank+1)
static int send_mask(const Geometry &geo, int blk) {
    int m = 0;
    if (geo.cfg.world > 1) {
        if (blk == geo.b_lo && geo.cfg.rank > 0) m |= 1;
        if (blk == geo.b_hi - 1 && geo.cfg.rank + 1 < geo.cfg.world) m |= 2;
    }
    return m;
}

// g0: global chunk counter of the run's first chunk (a multiple of the rank's chunk count): lanes,
// working sets and event instances continue across runs, and the first sweep's cross-sweep waits name
// the previous run's write-backs, so a run can be issued while the previous one drains (oocs_run_async).
// The ops' `sweep` field stays run-local.  Host store, codec modes only (0 elsewhere).
static void lower_alg1(const Geometry &geo, int64_t sweeps, std::vector<oocs_op> &ops, int64_t g0) {
    ops.clear();
    Emitter E{ops};
    const int nb = geo.nb();
    const int64_t G = sweeps * nb;
    if (!geo.host_store) {
        for (int64_t g = 0; g < G; ++g) {
            const int t = (int)(g / nb), blk = geo.b_lo + (int)(g % nb);
            E.emit(OOCS_OP_DECODE, 0, g, blk, t);
            for (int s = 1; s <= geo.k; ++s) E.emit(OOCS_OP_STEP, 0, g, blk, t, s);
            E.emit(OOCS_OP_ENCODE, 0, g, blk, t);
            if (const int m = send_mask(geo, blk)) E.emit(OOCS_OP_SEND, 0, g, blk, t, m);
        }
        return;
    }
    const int L = geo.lanes;
    auto lane = [L](int64_t g) { return (int)(g % L); };
    auto blk_of = [&](int64_t g) { return geo.b_lo + (int)(g % nb); };
    // previous sweep's chunks whose owned planes intersect [lo, hi) (global sweep index; the op keeps
    // its run-local sweep)
    auto raw_waits = [&](int64_t g, int64_t lo, int64_t hi) {
        const int64_t tg = g / nb;
        if (tg == 0) return;
        const int t = (int)((g - g0) / nb);
        for (int j = 0; j < nb; ++j) {
            const oocs_block &b = geo.blocks[geo.b_lo + j];
            if (b.own_lo < hi && lo < b.own_hi)
                E.emit(OOCS_OP_WAIT, lane(g), g, blk_of(g), t, OOCS_EV_D2H, (tg - 1) * nb + j);
        }
    };
    if (geo.cfg.mode == OOCS_MODE_BASELINE) {
        // fig:3ver(a): three private working sets, H2D straight into them; the
        // overlap is copied GPU-side from the previous chunk's working set
        // before that chunk's compute overwrites it.
        for (int64_t g = 0; g < G; ++g) {
            const int t = (int)(g / nb), i = (int)(g % nb), blk = blk_of(g), s = lane(g);
            const oocs_block &b = geo.blocks[blk];
            raw_waits(g, b.body_lo, b.body_hi);
            E.emit(OOCS_OP_H2D, s, g, blk, t);
            if (i > 0) E.emit(OOCS_OP_WAIT, s, g, blk, t, OOCS_EV_CARRY, g);
            if (i + 1 < nb) {  // the next chunk's working set was last used by chunk g+1-L
                if (g + 1 >= L) E.emit(OOCS_OP_WAIT, s, g, blk, t, OOCS_EV_D2H, g + 1 - L);
                E.emit(OOCS_OP_CARRY, s, g + 1, blk + 1, t);
                E.emit(OOCS_OP_RECORD, s, g + 1, blk + 1, t, OOCS_EV_CARRY, g + 1);
            }
            for (int st = 1; st <= geo.k; ++st) E.emit(OOCS_OP_STEP, s, g, blk, t, st);
            E.emit(OOCS_OP_D2H, s, g, blk, t);
            E.emit(OOCS_OP_RECORD, s, g, blk, t, OOCS_EV_D2H, g);
        }
        return;
    }
    int64_t pending = -1;
    // tail of chunk p on its lane.  The next chunk's carry copy reads hf_buf[s(p)], which
    // ENCODE(p) overwrites (one half-size buffer per stream for both directions): the carry is
    // issued on this same stream before the tail, so stream order protects it.
    auto tail = [&](int64_t p) {
        const int s = lane(p), blk = blk_of(p), t = (int)((p - g0) / nb);
        E.emit(OOCS_OP_ENCODE, s, p, blk, t);
        E.emit(OOCS_OP_RECORD, s, p, blk, t, OOCS_EV_ENC, p);
        // multi-GPU: the edge planes go to the neighbour's ghost slot straight from the encoded buffer,
        // before the D2H (the neighbour's edge chunk is waiting for them)
        if (const int m = send_mask(geo, blk)) E.emit(OOCS_OP_SEND, s, p, blk, t, m);
        E.emit(OOCS_OP_D2H, s, p, blk, t);
        E.emit(OOCS_OP_RECORD, s, p, blk, t, OOCS_EV_D2H, p);
    };
    for (int64_t g = g0; g < g0 + G; ++g) {
        const int t = (int)((g - g0) / nb), i = (int)(g % nb), blk = blk_of(g), s = lane(g);
        const oocs_block &b = geo.blocks[blk];
        const bool carry = i > 0 && b.carry_hi > b.carry_lo;
        // H2D(g) depends only on its stream's own earlier work (the D2H that emptied hf_buf[s], L chunks
        // back) and the cross-sweep RAW waits, so the H2D engine can queue it while chunk g-1 is still in
        // flight.  Algorithm 1 lists the previous chunk's compress / record / transfer first,
        // on another stream: per-stream programs and events are unchanged.  Exception: when H2D(g) reads
        // host planes that the pending chunk g-1's D2H writes (a cross-sweep RAW with one or two chunks per
        // sweep), that D2H's record must precede the wait, so the tail goes first.
        bool raw_on_pending = false;
        if (pending >= 0 && g / nb > 0 && pending / nb == g / nb - 1) {
            const oocs_block &pb = geo.blocks[blk_of(pending)];
            raw_on_pending = pb.own_lo < b.body_hi && b.body_lo < pb.own_hi;
        }
        auto h2d = [&] {
            raw_waits(g, b.body_lo, b.body_hi);
            E.emit(OOCS_OP_H2D, s, g, blk, t);
            E.emit(OOCS_OP_RECORD, s, g, blk, t, OOCS_EV_H2D, g);
        };
        if (!raw_on_pending) h2d();
        if (carry) {
            // region sharing: the overlap is copied GPU-side out of chunk g-1's buffer, on chunk g-1's
            // stream (after its H2D and steps, before its encode overwrites the buffer: stream order),
            // into hf_buf[s(g)] once chunk g-L's D2H has emptied it.  Not on stream s(g) ahead of H2D(g):
            // that made every H2D wait for the previous chunk's carry (measured: 5.5 ms per chunk idle on
            // the binding PCIe direction at c3 with a copy-engine carry)
            const int sp = lane(g - 1);
            // (when 2kR > W the source planes include planes carried into chunk g-1 by its own carry copy:
            // ordered too, since chunk g-1's decode, earlier on this stream, waited for that copy)
            if (g >= L) E.emit(OOCS_OP_WAIT, sp, g, blk, t, OOCS_EV_D2H, g - L);
            E.emit(OOCS_OP_CARRY, sp, g, blk, t);
            E.emit(OOCS_OP_RECORD, sp, g, blk, t, OOCS_EV_CARRY, g);
        }
        if (pending >= 0) {
            tail(pending);
            pending = -1;
        }
        if (raw_on_pending) h2d();
        if (carry) E.emit(OOCS_OP_WAIT, s, g, blk, t, OOCS_EV_CARRY, g);
        if (g >= geo.n_ws) E.emit(OOCS_OP_WAIT, s, g, blk, t, OOCS_EV_ENC, g - geo.n_ws);
        E.emit(OOCS_OP_DECODE, s, g, blk, t);
        E.emit(OOCS_OP_RECORD, s, g, blk, t, OOCS_EV_DEC, g);
        for (int st = 1; st <= geo.k; ++st) E.emit(OOCS_OP_STEP, s, g, blk, t, st);
        pending = g;
    }
    if (pending >= 0) tail(pending);  // drain epilogue
}

// ---------------------------------------------------------------------------
// DAG schedules: "Task graph based methods can be used to schedule the GPU kernels to
// prevent resource conflicts ... We can schedule the operations by applying topological sorting to
// the DAG. CUDA events are used to realize fine-grained synchronizations between streams. At the
// beginning of an arrowed dotted line, we record an event with the stream the line starts from,
// whereas at the end of the arrowed dotted line, we wait for the event with the stream the arrow is
// pointed to."
//   nodes: the chunk operations in the order of the sequential program (Algorithm 1's order);
//   edges: every pair of nodes touching the same bytes with at least one write (footprints below,
//          the same model tests/schedule_check.py verifies against);
//   order: Kahn's algorithm with the program position as priority;
//   events: a record/wait pair for every cross-stream edge that stream order plus earlier waits do
//           not already imply (per-node vector clocks over the streams).
// ---------------------------------------------------------------------------
namespace {
struct Acc {
    int kind, idx, arr;  // kind 0 host store, 1 half-size buffer (arr unused), 2 working buffer
    int64_t lo, hi;      // plane range
    bool w;
};

static void footprint(const Geometry &geo, const oocs_op &o, std::vector<Acc> &f) {
    f.clear();
    const int L = geo.lanes;
    const int64_t g = o.g;
    const oocs_block &b = geo.blocks[o.block];
    const int s = (int)(g % L), w = (int)(g % geo.n_ws);
    const int64_t E = b.ext_hi - b.ext_lo, ME = geo.max_ext, MO = geo.max_own;
    const bool resv = (geo.cfg.flags & OOCS_FLAG_RESIDENT_VELOCITY) != 0;
    const int a0 = resv ? 1 : 0;
    const bool base = geo.cfg.mode == OOCS_MODE_BASELINE;
    auto step_range = [&](int st, int64_t &lo, int64_t &hi) {
        lo = (b.ext_lo == -R) ? 0 : b.ext_lo + (int64_t)st * R;
        hi = (b.ext_hi == geo.nz + R) ? geo.nz : b.ext_hi - (int64_t)st * R;
    };
    switch (o.kind) {
    case OOCS_OP_H2D:
        for (int a = base ? 0 : a0; a < N_ARRAYS; ++a) {
            f.push_back({0, 0, a, b.body_lo, b.body_hi, false});
            if (base)
                f.push_back({2, w, a, b.body_lo - b.ext_lo, E, true});
            else
                f.push_back({1, s, -1, a * ME + b.body_lo - b.ext_lo, a * ME + E, true});
        }
        break;
    case OOCS_OP_CARRY: {
        const oocs_block &pb = geo.blocks[o.block - 1];
        const int sp = (int)((g - 1) % L), wp = (int)((g - 1) % geo.n_ws);
        for (int a = base ? 0 : a0; a < N_ARRAYS; ++a) {
            if (base) {
                f.push_back({2, wp, a, b.carry_lo - pb.ext_lo, b.carry_hi - pb.ext_lo, false});
                f.push_back({2, w, a, b.carry_lo - b.ext_lo, b.carry_hi - b.ext_lo, true});
            } else {
                f.push_back({1, sp, -1, a * ME + b.carry_lo - pb.ext_lo, a * ME + b.carry_hi - pb.ext_lo, false});
                f.push_back({1, s, -1, a * ME + b.carry_lo - b.ext_lo, a * ME + b.carry_hi - b.ext_lo, true});
            }
        }
        break;
    }
    case OOCS_OP_DECODE:
        for (int a = 0; a < N_ARRAYS; ++a) {
            if (a >= a0) f.push_back({1, s, -1, a * ME, a * ME + E, false});
            f.push_back({2, w, a, 0, E, true});
        }
        break;
    case OOCS_OP_STEP: {
        int64_t lo, hi;
        step_range(o.arg, lo, hi);
        const int up = (o.arg & 1) ? 1 : 2;
        f.push_back({2, w, 0, lo - R - b.ext_lo, hi + R - b.ext_lo, false});
        f.push_back({2, w, 3 - up, lo - R - b.ext_lo, hi + R - b.ext_lo, false});
        f.push_back({2, w, up, lo - b.ext_lo, hi - b.ext_lo, true});
        // OOCS_FLAG_FUSE_DECODE: the first step reads p_{t-1}'s records in the staging buffer (edge chunks of
        // a multi-GPU run are not fused; the extra edge is then only conservative)
        if (o.arg == 1 && (geo.cfg.flags & OOCS_FLAG_FUSE_DECODE) && !base) f.push_back({1, s, -1, ME, ME + E, false});
        break;
    }
    case OOCS_OP_ENCODE:
        for (int j = 0; j < 2; ++j) {
            f.push_back({2, w, 1 + j, b.own_lo - b.ext_lo, b.own_hi - b.ext_lo, false});
            f.push_back({1, s, -1, j * MO, j * MO + b.own_hi - b.own_lo, true});
        }
        break;
    case OOCS_OP_SEND:
        for (int j = 0; j < 2; ++j) f.push_back({1, s, -1, j * MO, j * MO + b.own_hi - b.own_lo, false});
        break;
    case OOCS_OP_D2H:
        for (int j = 0; j < 2; ++j) {
            if (base)
                f.push_back({2, w, 1 + j, b.own_lo - b.ext_lo, b.own_hi - b.ext_lo, false});
            else
                f.push_back({1, s, -1, j * MO, j * MO + b.own_hi - b.own_lo, false});
            f.push_back({0, 0, 1 + j, b.own_lo, b.own_hi, true});
        }
        break;
    default:
        break;
    }
}

static bool conflict(const std::vector<Acc> &x, const std::vector<Acc> &y) {
    for (const Acc &a : x)
        for (const Acc &c : y)
            if (a.kind == c.kind && a.idx == c.idx && a.arr == c.arr && (a.w || c.w) && a.lo < c.hi && c.lo < a.hi)
                return true;
    return false;
}
}  // namespace

static void lower_dag(const Geometry &geo, int64_t sweeps, bool by_function, std::vector<oocs_op> &ops) {
    // 1. nodes = the sequential program (Algorithm 1's operation order, no synchronisation)
    std::vector<oocs_op> seq;
    lower_alg1(geo, sweeps, seq, 0);
    std::vector<oocs_op> nodes;
    for (const oocs_op &o : seq)
        if (o.kind != OOCS_OP_WAIT && o.kind != OOCS_OP_RECORD) nodes.push_back(o);
    const int N = (int)nodes.size();
    if (by_function)
        for (oocs_op &o : nodes)
            o.lane = (o.kind == OOCS_OP_H2D || o.kind == OOCS_OP_CARRY) ? 0 : (o.kind == OOCS_OP_D2H ? 2 : 1);
    // 2. data-dependence edges (u < v in program order); chunks further apart than the window
    //    share no buffer (ring sizes) and meet on the host store only across one sweep
    const int L = geo.lanes, nb = geo.nb();
    const int64_t window = std::max<int64_t>(std::max(L, geo.n_ws), nb) + 2;
    std::vector<std::vector<Acc>> fp(N);
    for (int i = 0; i < N; ++i) footprint(geo, nodes[i], fp[i]);
    std::vector<std::vector<int>> pred(N), succ(N);
    for (int v = 0; v < N; ++v) {
        for (int u = v - 1; u >= 0; --u) {
            if (nodes[v].g - nodes[u].g > window) break;
            if (conflict(fp[u], fp[v])) {
                pred[v].push_back(u);
                succ[u].push_back(v);
            }
        }
    }
    // 3. Kahn topological sort, ties broken by program position
    std::vector<int> indeg(N), order;
    for (int v = 0; v < N; ++v) indeg[v] = (int)pred[v].size();
    std::vector<int> ready;  // min-heap on index
    for (int v = 0; v < N; ++v)
        if (!indeg[v]) ready.push_back(v);
    std::make_heap(ready.begin(), ready.end(), std::greater<int>());
    while (!ready.empty()) {
        std::pop_heap(ready.begin(), ready.end(), std::greater<int>());
        const int u = ready.back();
        ready.pop_back();
        order.push_back(u);
        for (int v : succ[u])
            if (--indeg[v] == 0) {
                ready.push_back(v);
                std::push_heap(ready.begin(), ready.end(), std::greater<int>());
            }
    }
    // 4. streams + events: vector clock per node = latest position on every stream known to happen
    //    before it; a cross-stream edge u->v needs a record/wait unless already covered
    const int S = MAX_LANES;
    std::vector<std::vector<int64_t>> vc(N, std::vector<int64_t>(S, -1));
    std::vector<int64_t> lane_pos(S, -1);
    std::vector<int> lane_last(S, -1);
    std::vector<char> recorded(N, 0);
    std::vector<int64_t> pos(N, -1);
    std::vector<std::vector<int>> waits(N);
    for (int v : order) {
        const oocs_op &o = nodes[v];
        std::vector<int64_t> c(S, -1);
        const int l = o.lane;
        if (lane_last[l] >= 0) {
            c = vc[lane_last[l]];
            c[l] = std::max(c[l], pos[lane_last[l]]);
        }
        std::vector<int> ps = pred[v];
        std::sort(ps.begin(), ps.end(), [&](int a, int b2) { return pos[a] > pos[b2]; });
        for (int u : ps) {
            const int lu = nodes[u].lane;
            if (c[lu] >= pos[u]) continue;  // implied by stream order / earlier waits
            waits[v].push_back(u);
            recorded[u] = 1;
            for (int k = 0; k < S; ++k) c[k] = std::max(c[k], vc[u][k]);
            c[lu] = std::max(c[lu], pos[u]);
        }
        pos[v] = ++lane_pos[l];
        vc[v] = c;
        lane_last[l] = v;
    }
    // 5. emit: waits before the node, the node, its record after it
    ops.clear();
    Emitter E{ops};
    for (int v : order) {
        const oocs_op &o = nodes[v];
        for (int u : waits[v]) E.emit(OOCS_OP_WAIT, o.lane, o.g, o.block, o.sweep, OOCS_EV_NODE, u);
        ops.push_back(o);
        if (recorded[v]) E.emit(OOCS_OP_RECORD, o.lane, o.g, o.block, o.sweep, OOCS_EV_NODE, v);
    }
}

void lower_schedule(const Geometry &geo, int64_t sweeps, std::vector<oocs_op> &ops, int64_t g0) {
    if (geo.host_store && geo.cfg.schedule != OOCS_SCHED_ALG1)
        lower_dag(geo, sweeps, geo.cfg.schedule == OOCS_SCHED_DAG_FUNC, ops);
    else
        lower_alg1(geo, sweeps, ops, chainable(geo) ? g0 : 0);
}

bool chainable(const Geometry &geo) {
    return geo.host_store && geo.cfg.mode != OOCS_MODE_BASELINE && geo.cfg.schedule == OOCS_SCHED_ALG1 &&
           geo.cfg.world == 1;
}

}  // namespace oocs

using namespace oocs;

extern "C" oocs_status oocs_plan_table(const oocs_config *cfg, oocs_block *out) {
    Geometry g;
    std::string err;
    oocs_status st = make_geometry(cfg, &g, &err);
    if (st != OOCS_OK) {
        set_error(err);
        return st;
    }
    if (out) std::memcpy(out, g.blocks.data(), g.blocks.size() * sizeof(oocs_block));
    return OOCS_OK;
}

extern "C" oocs_status oocs_schedule(const oocs_config *cfg, int64_t steps, oocs_op *ops, int64_t cap,
                                     int64_t *n_ops) {
    return oocs_schedule_at(cfg, steps, 0, ops, cap, n_ops);
}

extern "C" oocs_status oocs_schedule_at(const oocs_config *cfg, int64_t steps, int64_t first_sweep, oocs_op *ops,
                                        int64_t cap, int64_t *n_ops) {
    Geometry g;
    std::string err;
    oocs_status st = make_geometry(cfg, &g, &err);
    if (st != OOCS_OK) {
        set_error(err);
        return st;
    }
    if (steps < 0 || steps % g.k) {
        set_error("steps must be a non-negative multiple of tb_depth (S:L448)");
        return OOCS_ERR_CONFIG;
    }
    if (first_sweep < 0) {
        set_error("first_sweep must be >= 0");
        return OOCS_ERR_CONFIG;
    }
    std::vector<oocs_op> v;
    lower_schedule(g, steps / g.k, v, first_sweep * g.nb());
    if (n_ops) *n_ops = (int64_t)v.size();
    if (ops && cap > 0) std::memcpy(ops, v.data(), std::min<int64_t>(cap, (int64_t)v.size()) * sizeof(oocs_op));
    return OOCS_OK;
}

extern "C" oocs_status oocs_encoded_bytes(const oocs_config *cfg, int64_t planes, uint64_t *bytes) {
    Geometry g;
    std::string err;
    oocs_status st = make_geometry(cfg, &g, &err);
    if (st != OOCS_OK) {
        set_error(err);
        return st;
    }
    if (planes < 0 || planes % 4) {
        set_error("planes must be a non-negative multiple of 4");
        return OOCS_ERR_CONFIG;
    }
    if (bytes) *bytes = (uint64_t)(planes * g.plane_bytes);
    return OOCS_OK;
}
