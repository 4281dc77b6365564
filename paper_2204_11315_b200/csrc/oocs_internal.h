// Internal declarations shared by the library's translation units.
#pragma once
#include <cuda_runtime.h>
#include <stdint.h>

#include <string>
#include <vector>

#include "../../include/oocs.h"

namespace oocs {

constexpr int R = OOCS_RADIUS;
constexpr int XOFF = 32 - R;  // column offset: interior x = R lands on a 128-byte boundary
constexpr int N_ARRAYS = 3;   // 0 velocity (read-only), 1 pressure t-1, 2 pressure t
constexpr int MAX_LANES = 8;  // strm[0:3] in the paper; configurable 2..8

// CFL limit of the leapfrog, v dt / h <= 2 / sqrt(3 |L1(pi)|), with L1(pi) = c0 + 2 sum_m (-1)^m c_m the 1-D
// operator's symbol at the Nyquist wavenumber: ACOUSTIC25 |L1(pi)| = 2048/315, STAR7 4 (oocs.h oocs_stencil)
inline double cfl_limit(int stencil) { return stencil == OOCS_STENCIL_STAR7 ? 0.5773502691896258 : 0.4528555233184199; }

// Geometry derived from a config (pure host; plan.cpp).
struct Geometry {
    oocs_config cfg;
    int64_t nx, ny, nz, ax, ay, az, pitch, pstride;  // pstride = ay * pitch (floats)
    int q;                  // BlockQuant code bits (rate_bits - 1); 0 for identity
    int codec;
    int64_t plane_bytes;    // compressed bytes of one allocated plane of one array
    int k;                  // temporal-blocking depth
    std::vector<oocs_block> blocks;  // all global blocks
    int b_lo, b_hi;         // this rank's blocks
    int64_t store_lo, store_hi;      // interior planes held by this rank's store (owned + ghost)
    int64_t max_ext, max_own;        // planes
    int n_ws;               // working sets
    int lanes;              // half-size buffers (chunk g uses slot g mod lanes) = CUDA streams of Alg. 1
    int nstreams;           // op lanes of the schedule: lanes, or 3 for OOCS_SCHED_DAG_FUNC (H2D+carry / kernels
                            // / D2H) when lanes < 3
    bool host_store;
    int64_t a_store_lo() const { return store_lo + R; }  // allocated plane of store index 0
    int64_t store_planes() const { return store_hi - store_lo; }
    int nb() const { return b_hi - b_lo; }
};

oocs_status make_geometry(const oocs_config *cfg, Geometry *geo, std::string *err);
// g0 = global chunk counter of the run's first chunk (runs continue each other's numbering when chainable)
void lower_schedule(const Geometry &geo, int64_t sweeps, std::vector<oocs_op> &ops, int64_t g0 = 0);
// runs of this plan may be issued back to back without draining in between (oocs_run_async): host store,
// codec modes, Algorithm 1, one rank
bool chainable(const Geometry &geo);

// kernels.cu
// n_arr (<= N_ARRAYS) arrays of the same geometry; BlockQuant does them in one launch
cudaError_t launch_decode(const void *const *src, float *const *dst, int n_arr, int64_t ax, int64_t ay,
                          int64_t planes, int64_t pitch, int codec, int q, cudaStream_t st);
cudaError_t launch_encode(const float *const *src, void *const *dst, int n_arr, int64_t ax, int64_t ay,
                          int64_t planes, int64_t pitch, int codec, int q, int *err, cudaStream_t st);
// BlockQuant: decode only the x/y ring blocks of every slab (the rest of the array is the fused step's)
cudaError_t launch_decode_ring(const void *src, float *dst, int64_t ax, int64_t ay, int64_t planes, int64_t pitch, int q,
                               cudaStream_t st);
// the decode -> first step fusion (OOCS_FLAG_FUSE_DECODE): p_prev read from its BlockQuant records
// (rec_pprev = the records of the working buffer's plane 0, 16-byte aligned; z_lo a multiple of 4)
bool step_fused_ok(int q);
cudaError_t launch_step_fused(const float *vel, float *pprev, const float *pcurr, const void *rec_pprev, int64_t ax,
                              int64_t ay, int64_t pitch, int64_t planes, int64_t z_lo, int64_t z_hi, float dt, int q,
                              cudaStream_t st);
cudaError_t launch_step(const float *vel, float *pprev, const float *pcurr, int64_t ax, int64_t ay, int64_t pitch,
                        int64_t planes, int64_t z_lo, int64_t z_hi, float dt, int stencil, cudaStream_t st);
// max |x| over `rows` rows of `n` floats (row stride `pitch` floats) folded into *out (float bits as u32,
// atomicMax; NaN compares above +Inf); *out must be initialised by the caller
cudaError_t launch_absmax(const float *src, int64_t rows, int64_t n, int64_t pitch, uint32_t *out, cudaStream_t st);

// SM copy of one or two equal-length byte ranges (8-byte multiples), dst possibly peer memory: the multi-GPU
// halo send, and the carry of region sharing (a copy-engine D2D of ~0.8 GB took 5.5 ms at c3)
cudaError_t launch_peer_copy(const void *src0, void *dst0, const void *src1, void *dst1, uint64_t bytes,
                             cudaStream_t st, int ranges = 2);

void set_error(const std::string &msg);

}  // namespace oocs
