/*
 * oocs.h — C ABI of the B200-native out-of-core compressed stencil library
 * (arXiv 2204.11315, "Compression-Based Optimizations for Out-of-Core GPU
 * Stencil Computation", Shen, Deng, Wu, Okita, Ino).
 *
 * The library runs the paper's data-parallel hot path on one GPU per process:
 * for every z-chunk ("block") of a 3-D grid that does not fit the GPU, H2D of
 * the fixed-rate-compressed chunk (minus the overlap already resident on the
 * GPU, "region sharing"), GPU decompression, k temporally blocked steps
 * of a 25-point acoustic-wave stencil in a single working buffer (P:L85,
 * P:L170-173), GPU recompression of the owned planes and D2H, overlapped on
 * three CUDA streams with the event hand-off of Algorithm 1.
 *
 * Citations: "P:L<n>" = PAPER.md line n; "S:L<n>" = SPEC.md line n.
 *
 * General rules
 *  - Every call returns oocs_status; OOCS_OK = 0.  No C++ exception crosses
 *    the ABI.  On failure oocs_last_error() returns a thread-local message.
 *  - After a CUDA error inside oocs_run/oocs_load/oocs_store the plan is
 *    poisoned: every later call except oocs_destroy returns OOCS_ERR_STATE.
 *  - Pointers are plain host or device pointers as stated per argument; the
 *    library never retains caller pointers beyond the call.
 *  - Streams are passed as `void*` holding a cudaStream_t (NULL = legacy
 *    default stream).  No torch type appears in any signature.
 *  - One plan per host thread; plans on different devices may run
 *    concurrently.
 *
 * Grid layout (host side, "allocated layout"): an array of the grid is
 * (az, ay, ax) float32, x fastest, with ax = nx+2R, ay = ny+2R, az = nz+2R,
 * R = 4 (Table 1 "(1152+2xHALO)^3, HALO=4").  Allocated plane index
 * a = interior plane z + R.  The R-cell halo on all six faces is a Dirichlet
 * boundary: it keeps its initial value forever (pressure 0 by convention).
 *
 * Compressed format (docs/FORMAT.md): each array is stored slab by slab (4
 * allocated planes per slab), within a slab by 4x4x4 block in (by, bx) order,
 * so every 4-aligned plane range is one contiguous, independently decodable
 * byte range ("we compress the overlapped area of a chunk
 * separately").  BlockQuant block record = 8(q+1) bytes:
 *   [mn f32][mx f32][P_{q-1} u64] ... [P_0 u64],  P_b bit j = bit b of code_j,
 *   j = xi + 4 yi + 16 zi; rate r = q + 1 bits/value (r = 16 is the paper's
 *   "compression rate 32/64 = 1/2", applied to fp32).
 * Identity codec: raw float32 planes (ax*ay*4 bytes per plane).
 */
#ifndef OOCS_H
#define OOCS_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define OOCS_RADIUS 4      /* halo width of every grid and chunk extent: the 25-point star's radius (P:L212,
                              Table 1 HALO=4); every stencil below reaches at most this far */
#define OOCS_ABI_VERSION 2  /* 2: oocs_config.stencil / v_max / ext_streams, oocs_step's stencil argument */

typedef enum {
    OOCS_OK = 0,
    OOCS_ERR_CONFIG = 2,     /* invalid configuration */
    OOCS_ERR_DEVICE_OOM = 3, /* device capacity exceeded */
    OOCS_ERR_VERIFY = 4,     /* reserved: verification failure */
    OOCS_ERR_IO = 5,         /* host-side I/O / pinned allocation failure */
    OOCS_ERR_DATA = 6,       /* NaN/Inf or |x| >= 2^126 given to a lossy codec */
    OOCS_ERR_HOST_OOM = 7,   /* host (pinned) allocation failed */
    OOCS_ERR_CUDA = 8,       /* CUDA runtime error; plan poisoned */
    OOCS_ERR_EXCHANGE = 9,   /* multi-GPU: peers not connected, or a peer handle that cannot be opened */
    OOCS_ERR_STATE = 10      /* plan poisoned by an earlier failure, or call out of order */
} oocs_status;

typedef enum {
    OOCS_CODEC_IDENTITY = 0,   /* raw fp32 (rate 32) */
    OOCS_CODEC_BLOCKQUANT = 1, /* fixed-rate 4x4x4 block quantiser, rate_bits in [2, 24] */
    OOCS_CODEC_ZFP = 2,        /* ZFP fixed-rate (cuZFP's algorithm), rate_bits in [1, 32]; record = 8*rate B */
    OOCS_CODEC_TRUNC16 = 3     /* Truncate-16: fp32 -> bfloat16, round to nearest even, NaN -> 0x7FC0;
                                * rate_bits must be 16; raw bf16 planes (ax*ay*2 B per plane, x fastest); never
                                * reports OOCS_ERR_DATA (Inf stays Inf, finite values above the bf16 range round to Inf) */
} oocs_codec;

/* The stencil of the update p_next = 2 p - p_prev + (v dt)^2 L(p), h = 1 ("25-point stencil ...
 * acoustic wave propagation").  L is evaluated in difference form (DESIGN.md §3 "stencil
 * evaluation order").  Both use the same R = 4 halo, plane ranges and temporal-blocking extents (kR planes
 * per side with R = OOCS_RADIUS): STAR7 needs only 1 plane per step, so its chunks carry a conservative
 * halo (redundant but exact: blocked == in-core bitwise, DESIGN.md §3 "STAR7 geometry").
 * CFL limit of the leapfrog (v dt / h at most 2 / sqrt(3 |symbol(pi)|)): ACOUSTIC25 2/sqrt(3*2048/315) =
 * 0.452856, STAR7 2/sqrt(12) = 0.577350. */
typedef enum {
    OOCS_STENCIL_ACOUSTIC25 = 0, /* 2nd order in time, 8th in space: c = (-205/72, 8/5, -1/5, 8/315, -1/560), R = 4 */
    OOCS_STENCIL_STAR7 = 1       /* 2nd order in space: c = (-2, 1), radius 1: small exact tests */
} oocs_stencil;

/* Pipeline architectures of the paper (Fig. 6 `fig:3ver`, Fig. 7 `fig:swb`). */
typedef enum {
    OOCS_MODE_BASELINE = 0,     /* fig:3ver(a): no compression, 3 per-stream working buffers */
    OOCS_MODE_COMPRESS = 1,     /* fig:3ver(b): compression, 3 per-stream working buffers */
    OOCS_MODE_COMPRESS_SWB = 2, /* fig:swb: compression + single working buffer (the paper's method) */
    OOCS_MODE_COMPRESS_DWB = 3  /* compression + 2 ping-pong working buffers (BASELINE.json configs[4]) */
} oocs_mode;

typedef enum {
    OOCS_STORE_HOST = 0,  /* compressed state in pinned host memory, streamed over PCIe (the paper) */
    OOCS_STORE_DEVICE = 1 /* compressed state resident in HBM (double-buffered); kernels only */
} oocs_store_kind;

/* How the stream/event schedule is obtained (host store). */
typedef enum {
    OOCS_SCHED_ALG1 = 0,     /* Algorithm 1 lowered by hand, with the hazard edges it leaves implicit */
    OOCS_SCHED_DAG = 1,      /* the paper's general recipe: build the DAG of data dependencies
                                between chunk operations, Kahn topological sort, record/wait an event for
                                every cross-stream edge not already implied; one stream per chunk (g mod L) */
    OOCS_SCHED_DAG_FUNC = 2  /* same DAG, streams by function: H2D + carry / kernels / D2H */
} oocs_schedule_kind;

#define OOCS_FLAG_PROFILE 1u /* time every kernel launch with CUDA events (oocs_stats.kernel_ms) */
/* Host store only, codec modes: keep this rank's compressed velocity (the read-only dataset,
 * P:L244) resident in HBM instead of re-sending it every sweep (SPEC S:L508's config flag);
 * H2D then moves the two pressure arrays only.  Off by default (paper-faithful accounting). */
#define OOCS_FLAG_RESIDENT_VELOCITY 2u
/* Flag value 4 is retired (ABI 1's OOCS_FLAG_FUSE_ENCODE, the last step fused with the encode: measured
 * slower than step + encode on B200 and removed in ABI 2); it is rejected. */
/* Record a CUDA-event span around every work op (H2D, CARRY, DECODE, STEP, ENCODE, D2H, SEND) of a
 * run; read it back with oocs_timeline (the analog of the paper's pipeline figures fig:pipe1 /
 * fig:newbot).  Costs two event records per op. */
#define OOCS_FLAG_TIMELINE 8u
/* Executors.  By default a host dispatcher issues the schedule's work ops by dependency: kernels on
 * their lane's kernel stream with device-side waits, copies only once their dependencies have completed,
 * on one stream per direction -- so no copy stream ever holds a pending cross-stream wait (a copy channel
 * blocked on a wait was measured, OOCS_FLAG_TIMELINE, to be re-examined only when the copy engine's
 * current DMA ends: DESIGN.md §8) -- except, on chainable plans, a run's trailing write-backs: once only
 * D2H copies are left they are issued at once behind device-side waits on the D2H stream, so that the
 * call returns (and a chained next run's H2Ds start) without the host waiting for the last encodes.
 * These flags replay the schedule onto streams instead:
 * LANE_SINGLE_STREAM = one CUDA stream per lane, the literal mapping of Alg. 1's three streams;
 * LANE_SPLIT_STREAMS = a copy and a kernel stream per lane, joined by an event at every switch.  All
 * three execute the same dependencies and produce the same bytes. */
/* Device store only: keep this rank's velocity (the read-only dataset) decoded in HBM as fp32
 * (allocated planes x ay x pitch, +4 B per cell) instead of decoding it from the compressed store in
 * every chunk of every sweep.  The values are the same decode of the same records, so results are
 * bitwise identical; each chunk's decode then moves two arrays instead of three.  Decoded once per
 * oocs_load / oocs_store_write_raw of array 0.  Off by default (the compressed-state accounting). */
#define OOCS_FLAG_DECODED_VELOCITY 64u
/* Decode -> first step fusion: the first of a chunk's k steps reads p_{t-1} straight
 * from its compressed BlockQuant records (staged into shared memory by bulk copies, decoded with the decode
 * kernel's warp transpose and arithmetic) instead of a decoded working-buffer copy, and the chunk's decode
 * then writes only the velocity, p_t and the x/y ring of p_{t-1} (which later steps read as the boundary).
 * p_{t-1} is read once and then overwritten, so this saves 8 B per cell of decode write + step read.  Same
 * values, so results are bitwise identical.  Codec modes with BlockQuant at an even rate <= 16 (q odd,
 * 16-byte records) and the 25-point stencil; chunks with multi-GPU ghost planes run unfused. */
#define OOCS_FLAG_FUSE_DECODE 128u
#define OOCS_FLAG_LANE_SINGLE_STREAM 16u
#define OOCS_FLAG_LANE_SPLIT_STREAMS 32u

typedef struct {
    uint32_t struct_size;     /* sizeof(oocs_config): ABI versioning */
    int64_t nx, ny, nz;       /* interior cells; nx, ny, nz multiples of 4 */
    float dt;                 /* time step; update uses c = (v*dt)^2 with h = 1 */
    int32_t n_blocks;         /* global number of z-chunks n ("eight chunks") */
    int32_t tb_depth;         /* temporal-blocking depth k: steps per chunk visit */
    int32_t codec;            /* oocs_codec */
    int32_t rate_bits;        /* BlockQuant rate r (q = r - 1 code bits); ignored for identity */
    int32_t mode;             /* oocs_mode */
    int32_t region_sharing;   /* 1: reuse the 2kR-plane overlap on the GPU; 0: re-send it */
    int32_t n_lanes;          /* CUDA streams / half-size buffers of the pipeline: 0 = 3, max 8 */
    int32_t schedule;         /* oocs_schedule_kind */
    int32_t store;            /* oocs_store_kind */
    int32_t device;           /* CUDA device ordinal used by this plan */
    int32_t rank, world;      /* z-slab sharding: this process owns a contiguous run of blocks */
    uint32_t flags;           /* OOCS_FLAG_* */
    uint64_t device_capacity; /* 0 = unlimited; else the arena may not exceed this many bytes */
    /* ---- ABI 2 ---- */
    int32_t stencil;          /* oocs_stencil */
    float v_max;              /* declared bound on |v| (0 = undeclared).  oocs_plan_create rejects dt*v_max above
                               * the stencil's CFL limit; independently, every oocs_load / oocs_load_device of the
                               * velocity (array 0) measures max|v| of the loaded planes on the GPU and rejects
                               * dt*max|v| above the limit (OOCS_ERR_CONFIG; NaN velocity counts as above).
                               * oocs_store_write_raw (trusted checkpoints) is not checked. */
    void *ext_streams[8];     /* optional caller-owned cudaStream_t per lane (e.g. torch streams): entry l < n_lanes,
                               * if non-NULL, replaces the library's kernel stream of lane l (its decode, steps and
                               * encode are issued there, so work the caller queued on it earlier runs first).  The
                               * library never destroys them; they must outlive the plan and belong to
                               * cfg->device.  NULL entries: library-owned streams. */
} oocs_config;

typedef struct {
    int64_t ax, ay, az;         /* allocated extents */
    int64_t pitch;              /* working-buffer row pitch in floats (>= ax + 28, multiple of 32) */
    int64_t plane_bytes;        /* compressed bytes of one allocated plane of one array */
    int64_t z_lo, z_hi;         /* this rank's owned interior planes [z_lo, z_hi) */
    int64_t store_lo, store_hi; /* interior planes held in this rank's store (owned + ghost halo) */
    int32_t block_lo, block_hi; /* this rank's global blocks [block_lo, block_hi) */
    int64_t max_ext_planes;     /* largest extended extent (planes) = working-buffer depth */
    uint64_t arena_bytes;       /* device bytes the plan allocated (its peak: allocation is static) */
    uint64_t working_set_bytes; /* one working buffer (all arrays) = the paper's "1 unit" x datasets */
    uint64_t staging_bytes;     /* all compressed staging buffers (hf_buf) */
    uint64_t store_bytes;       /* compressed state (host pinned or device) */
    int32_t n_working_sets;     /* 3 (BASELINE/COMPRESS), 1 (SWB), 2 (DWB) */
    int32_t n_lanes;            /* CUDA streams of the pipeline (default 3) */
} oocs_plan_info;

typedef struct {
    double wall_ms;             /* device time of the run: its start mark .. the mark after its last op; a chained
                                 * run's start mark follows the previous run's end mark (oocs_run_async) */
    double kernel_ms[3];        /* [decode, step, encode] summed launch durations (OOCS_FLAG_PROFILE) */
    int64_t kernel_launches[3]; /* launches per kind */
    uint64_t bytes_h2d, bytes_d2h, bytes_d2d, bytes_exchange;
    uint64_t cell_updates;          /* useful: nx*ny*(owned planes)*steps on this rank */
    uint64_t cell_updates_computed; /* incl. redundant temporal-blocking halo updates */
    uint64_t alg_bytes[3];          /* algorithmic HBM bytes per kind */
    int32_t data_error;             /* 1 if the encoder saw NaN/Inf/|x|>=2^126 */
    int32_t copy_launches;          /* SM copy kernels launched: region-sharing carries, multi-GPU sends */
    double busy_ms[4];              /* OOCS_FLAG_TIMELINE: busy time (union of op spans) of the H2D copies, the
                                     * D2H copies, the kernels and the exchange; 0 without the flag */
} oocs_stats;

/* One entry of the decomposition table (interior plane coordinates,
 * half-open intervals). */
typedef struct {
    int64_t own_lo, own_hi;     /* owned planes: partition of [0, nz) */
    int64_t ext_lo, ext_hi;     /* own +- k*R, clamped to [-R, nz+R) */
    int64_t carry_lo, carry_hi; /* overlap with the previous chunk's extent, kept on the GPU */
    int64_t body_lo, body_hi;   /* ext \ carry: what crosses PCIe */
} oocs_block;

/* One operation of the lowered pipeline schedule (Algorithm 1 + repairs). */
typedef struct {
    int32_t kind;  /* oocs_op_kind */
    int32_t lane;  /* CUDA stream index */
    int64_t g;     /* global block counter (sweep * blocks + block) the op belongs to */
    int32_t block; /* global block index */
    int32_t sweep;
    int32_t arg;   /* STEP: step index s (1..k); WAIT/RECORD: event kind; else 0 */
    int32_t pad;
    int64_t ev_g;  /* WAIT/RECORD: block counter of the event */
} oocs_op;

/* One recorded op of the last oocs_run under OOCS_FLAG_TIMELINE: when its lane reached it (start) and
 * finished it (end), in ms from the run's first event.  A copy's start is when its stream issued it; it
 * may then queue behind another lane's copy on the same DMA engine. */
typedef struct {
    int32_t kind;  /* oocs_op_kind (H2D, CARRY, DECODE, STEP, ENCODE, D2H, SEND) */
    int32_t lane;
    int64_t g;     /* global block counter */
    int32_t block;
    int32_t sweep;
    int32_t arg;   /* STEP: step index s */
    int32_t pad;
    double start_ms, end_ms;
    double host_ms; /* host wall clock when the op was enqueued, ms from the run's start (enqueue lag) */
} oocs_span;

typedef enum {
    OOCS_OP_H2D = 0, OOCS_OP_CARRY = 1, OOCS_OP_DECODE = 2, OOCS_OP_STEP = 3,
    OOCS_OP_ENCODE = 4, OOCS_OP_D2H = 5, OOCS_OP_RECORD = 6, OOCS_OP_WAIT = 7,
    OOCS_OP_SEND = 8 /* multi-GPU: an edge chunk's kR encoded planes straight into the neighbour's ghost slot */
} oocs_op_kind;

typedef enum {
    OOCS_EV_H2D = 0,   /* body (+carry) of block g is in its staging/working buffer */
    OOCS_EV_DEC = 1,   /* block g decoded */
    OOCS_EV_ENC = 2,   /* block g encoded: working buffer free (Alg. 1 "Record evt[prev_s]") */
    OOCS_EV_D2H = 3,   /* owned planes of block g written back to the host store */
    OOCS_EV_CARRY = 4, /* BASELINE mode: carry of block g copied into its working buffer */
    OOCS_EV_NODE = 5   /* DAG schedules: completion of DAG node ev_g (index in the schedule's node list) */
} oocs_event_kind;

typedef struct oocs_plan oocs_plan;

/* ---- host-only calls (no GPU needed) ---------------------------------- */

/* Validate cfg and fill the decomposition table for ALL global blocks
 * (out[cfg->n_blocks], caller-owned).  Pure function of cfg.
 * Errors: OOCS_ERR_CONFIG for nx/ny/nz not multiples of 4, n_blocks > nz/4,
 * k*R >= owned width, rate outside [2,24], world not dividing
 * n_blocks, dt <= 0, unknown stencil, v_max < 0, or dt*v_max above the
 * stencil's CFL limit when v_max is declared (the velocity data itself is
 * checked by oocs_load). */
oocs_status oocs_plan_table(const oocs_config *cfg, oocs_block *out);

/* Lower the pipeline of `steps` time steps (steps % k == 0) for this rank
 * to its operation list (the exact list oocs_run issues for a HOST store).
 * Always sets *n_ops to the full count and writes the first min(cap, count)
 * ops to `ops` (ops may be NULL when cap == 0).
 * Errors: OOCS_ERR_CONFIG. */
oocs_status oocs_schedule(const oocs_config *cfg, int64_t steps, oocs_op *ops, int64_t cap,
                          int64_t *n_ops);

/* The same for a run that starts after `first_sweep` sweeps of earlier runs of the same plan: with a
 * host store, codec modes, Algorithm 1 and world == 1 ("chainable"), consecutive runs continue one
 * global chunk counter (lanes, working sets, event instances) and the run's first cross-sweep waits name
 * the previous run's write-backs -- what lets oocs_run_async issue a run while the previous one drains.
 * Other configurations restart at chunk 0 (identical to oocs_schedule).  Errors: OOCS_ERR_CONFIG. */
oocs_status oocs_schedule_at(const oocs_config *cfg, int64_t steps, int64_t first_sweep, oocs_op *ops,
                             int64_t cap, int64_t *n_ops);

/* What oocs_plan_create would allocate for cfg (arena = the device peak, pinned host store, working
 * sets, staging), without allocating anything: the paper's memory comparison for
 * configurations larger than this machine.  Errors: OOCS_ERR_CONFIG. */
oocs_status oocs_plan_estimate(const oocs_config *cfg, oocs_plan_info *info);

/* Compressed bytes of `planes` allocated planes of one array. */
oocs_status oocs_encoded_bytes(const oocs_config *cfg, int64_t planes, uint64_t *bytes);

/* ---- plan lifetime ----------------------------------------------------- */

/* Create a plan on cfg->device: validates, allocates the device arena
 * (working buffers, staging, [device store]) and the pinned host store,
 * creates streams and events.  *out = NULL on failure.
 * Errors: OOCS_ERR_CONFIG, OOCS_ERR_DEVICE_OOM (arena > device_capacity or
 * cudaMalloc failure), OOCS_ERR_HOST_OOM, OOCS_ERR_CUDA. */
oocs_status oocs_plan_create(const oocs_config *cfg, oocs_plan **out);

/* The same on a caller-owned device arena (SURVEY §8(b) "optional torch-owned arena"): `arena` is device
 * memory of cfg->device, 256-byte aligned, at least oocs_plan_estimate(cfg).arena_bytes long; the plan
 * carves its working sets, staging and device store out of it, zeroes it, and never frees it -- the
 * caller keeps it alive until oocs_destroy.  Errors: as oocs_plan_create, plus OOCS_ERR_CONFIG for a
 * NULL, short, misaligned or non-device arena. */
oocs_status oocs_plan_create_in(const oocs_config *cfg, void *arena, uint64_t arena_bytes, oocs_plan **out);

oocs_status oocs_plan_query(const oocs_plan *plan, oocs_plan_info *info);

/* ---- multi-GPU: z-slab sharding with a peer-memory halo exchange -----------------
 * Rank r of `world` owns a contiguous run of whole chunks.  The kR pressure planes it needs beyond its
 * slab (the neighbours' edge planes of S_t, P:L85 temporal-blocking halo) arrive in HBM "ghost slots"
 * (two per side, by parity of the sweep's state index), written directly by the neighbour over
 * NVLink (CUDA IPC peer memory; the same GPU when ranks share one): right after the neighbour's edge
 * chunk is encoded, a copy kernel on that chunk's stream stores its kR compressed planes into our
 * slot and then writes a sequence number into our READY flag (cuStreamWriteValue32, fenced).  Our
 * edge chunk's decode waits for that number on its own stream (cuStreamWaitValue32) and, once it has
 * read the slot, writes the neighbour's FREE flag so the slot can be reused two sweeps later.  No
 * host synchronisation, no drain between sweeps, no re-streaming of halos over PCIe: the multi-GPU
 * analogue of region sharing.  The static velocity ghosts are loaded once.
 *
 * Protocol: every rank calls oocs_peer_handle, the caller moves the blobs between processes (e.g.
 * torch.distributed all_gather_object: plumbing only), every rank calls oocs_peer_connect with its
 * neighbours' blobs.  Runs of all ranks must advance by the same steps; load/store/raw calls and
 * oocs_destroy must not overlap a neighbour's oocs_run (a barrier between them is the caller's).
 * The ranks may live in one process (same-process peers use plain pointers) or in several. */
#define OOCS_PEER_HANDLE_BYTES 256

/* Fill `out` (OOCS_PEER_HANDLE_BYTES, host memory) with this plan's exchange-region handle.
 * Errors: OOCS_ERR_STATE (world == 1: no exchange region), OOCS_ERR_CUDA. */
oocs_status oocs_peer_handle(const oocs_plan *plan, void *out);

/* Map the neighbours' exchange regions: `lower` = rank-1's handle (NULL for rank 0), `upper` = rank+1's
 * (NULL for the last rank).  Validates that the blobs come from the same job geometry.
 * Errors: OOCS_ERR_CONFIG (wrong / mismatched blob, missing neighbour), OOCS_ERR_EXCHANGE (IPC open
 * failed), OOCS_ERR_STATE. */
oocs_status oocs_peer_connect(oocs_plan *plan, const void *lower, const void *upper);

/* NULL-safe; frees streams, events, arena and pinned store. */
oocs_status oocs_destroy(oocs_plan *plan);

/* ---- state in / out ---------------------------------------------------- */

/* Compress allocated planes [a_lo, a_hi) (allocated coordinates, 4-aligned,
 * within this rank's store) of one array from HOST memory `src` laid out
 * (a_hi-a_lo, ay, ax) float32 into the store.  array: 0 = velocity
 * (read-only dataset), 1 = pressure at t-1, 2 = pressure at t.
 * The GPU encodes; host memory is only read during the call.
 * Errors: OOCS_ERR_CONFIG (range; for array 0 also dt*max|v| above the
 * stencil's CFL limit, see oocs_config.v_max -- the store is then undefined
 * for those planes), OOCS_ERR_DATA (non-finite input for a lossy codec),
 * OOCS_ERR_CUDA. */
oocs_status oocs_load(oocs_plan *plan, int32_t array, const float *src, int64_t a_lo, int64_t a_hi);

/* Decompress allocated planes [a_lo, a_hi) of one array into HOST `dst`
 * (same layout as oocs_load). */
oocs_status oocs_store(oocs_plan *plan, int32_t array, float *dst, int64_t a_lo, int64_t a_hi);

/* The same two calls with DEVICE memory of the plan's device on the caller's side (same raw layout):
 * state generated or consumed on the GPU never crosses PCIe uncompressed.  The library works on its own
 * streams: the caller's writes to `src` must be complete (e.g. its stream synchronized) before the call;
 * `dst` is complete when the call returns. */
oocs_status oocs_load_device(oocs_plan *plan, int32_t array, const float *src, int64_t a_lo, int64_t a_hi);
oocs_status oocs_store_device(oocs_plan *plan, int32_t array, float *dst, int64_t a_lo, int64_t a_hi);

/* Raw compressed bytes of allocated planes [a_lo, a_hi) of one array,
 * to / from HOST memory (bitstream parity tests, checkpoints). */
oocs_status oocs_store_read_raw(oocs_plan *plan, int32_t array, void *dst, int64_t a_lo, int64_t a_hi);
oocs_status oocs_store_write_raw(oocs_plan *plan, int32_t array, const void *src, int64_t a_lo,
                                 int64_t a_hi);

/* Advance the state by `steps` time steps (steps % k == 0) = steps/k sweeps
 * of Algorithm 1 over this rank's blocks, sweeps pipelined back to back.
 * Blocks the host until the device work is complete.  `out` may be NULL.
 * Errors: OOCS_ERR_CONFIG (steps), OOCS_ERR_DATA (encoder rejected a value;
 * state undefined), OOCS_ERR_CUDA, OOCS_ERR_EXCHANGE (world > 1 and not connected), OOCS_ERR_STATE. */
oocs_status oocs_run(oocs_plan *plan, int64_t steps, oocs_stats *out);

/* Issue `steps` steps and return once every operation is issued, without waiting for them (the run's
 * tail -- the last chunk's kernels and write-back -- may still be in flight).  A following
 * oocs_run_async on a chainable plan (host store, codec modes, OOCS_SCHED_ALG1, world == 1, host
 * dispatcher, no OOCS_FLAG_TIMELINE) starts while that tail drains: its first H2D waits only for what
 * it really depends on (the lane buffer's previous write-back, the previous sweep's write-back of the
 * planes it reads -- oocs_schedule_at), which overlaps the two runs' pipeline drain and fill
 * ("overlap the first H2D with the previous run's drain").  Otherwise it waits for the
 * previous run first.  Every other call on the plan (load, store, raw I/O, timeline, destroy) completes
 * the runs in flight first.  The result is bitwise that of the same steps in oocs_run calls.
 * Errors: as oocs_run (a data error is reported by oocs_wait). */
oocs_status oocs_run_async(oocs_plan *plan, int64_t steps);

/* Complete every run in flight and return their stats in issue order: min(cap, n) entries into out,
 * *n_runs = n (may be NULL).  A run's wall_ms counts from its start mark, which follows the previous
 * run's end mark, so the wall times of a chain add up to the chain's device time.
 * Errors: OOCS_ERR_CONFIG (cap < 0, or out NULL with cap > 0), OOCS_ERR_DATA, OOCS_ERR_CUDA,
 * OOCS_ERR_EXCHANGE, OOCS_ERR_STATE. */
oocs_status oocs_wait(oocs_plan *plan, oocs_stats *out, int64_t cap, int64_t *n_runs);

/* Spans of the last oocs_run made with OOCS_FLAG_TIMELINE, in schedule order.  Copies min(cap, n)
 * spans into out (out may be NULL to query n); *n_spans = n (0 if the flag was not set).
 * Errors: OOCS_ERR_CONFIG for NULL plan / n_spans, OOCS_ERR_STATE for a poisoned plan. */
oocs_status oocs_timeline(const oocs_plan *plan, oocs_span *out, int64_t cap, int64_t *n_spans);

/* ---- hot-path kernels, callable on caller device memory --------------- */
/* Working-buffer layout for these calls: planes x ay rows x `pitch` floats,
 * element (x) of a row at column x + 28 (so interior x = R starts on a
 * 128-byte boundary); pitch >= ax + 28 and a multiple of 32. */

/* Decompress `planes` (multiple of 4) allocated planes: src (DEVICE)
 * compressed bytes -> dst (DEVICE) working-buffer layout. */
oocs_status oocs_decode(const void *src, float *dst, int64_t ax, int64_t ay, int64_t planes,
                        int64_t pitch, int32_t codec, int32_t rate_bits, void *stream);

/* Compress `planes` allocated planes of src (DEVICE, working-buffer layout)
 * into dst (DEVICE).  *err_flag (DEVICE int32, may be NULL) is OR-ed with 1
 * if a value is rejected. */
oocs_status oocs_encode(const float *src, void *dst, int64_t ax, int64_t ay, int64_t planes,
                        int64_t pitch, int32_t codec, int32_t rate_bits, int32_t *err_flag,
                        void *stream);

/* One leapfrog step of the chosen stencil:
 *   p_prev[z] <- 2 p_curr[z] - p_prev[z] + (v dt)^2 L(p_curr)[z]
 * on buffer planes [z_lo, z_hi) (R <= z_lo, z_hi <= planes-R), interior x,y (R = OOCS_RADIUS for both
 * stencils).  All pointers DEVICE, working-buffer layout.  p_prev is updated in place.  stencil is an
 * oocs_stencil.  No CFL check (no velocity bound is known here). */
oocs_status oocs_step(const float *vel, float *p_prev, const float *p_curr, int64_t ax, int64_t ay,
                      int64_t planes, int64_t pitch, float dt, int64_t z_lo, int64_t z_hi,
                      int32_t stencil, void *stream);

/* ---- misc -------------------------------------------------------------- */
const char *oocs_last_error(void);
int32_t oocs_abi_version(void);

/* sizeof of the ABI structs, for bindings to check their mirrors: out[0..5] = oocs_config, oocs_stats,
 * oocs_plan_info, oocs_block, oocs_op, oocs_span.  Host-only. */
void oocs_abi_sizes(int64_t out[6]);

#ifdef __cplusplus
}
#endif
#endif /* OOCS_H */
