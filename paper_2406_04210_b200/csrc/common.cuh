// Shared helpers for the libb2md kernels (sm_100a only).
#pragma once

#include <cuda_runtime.h>
#include <stdint.h>
#include <stdio.h>
#include <stdlib.h>

#include "../../include/b2md.h"

#define B2MD_EXPORT extern "C" __attribute__((visibility("default")))

namespace b2md {

constexpr int kNumSM = 148;  // B200: 2 dies x 74 SMs

void set_error(const char *fmt, ...);

inline int check_cuda(cudaError_t err, const char *what) {
    if (err != cudaSuccess) {
        set_error("%s: %s", what, cudaGetErrorString(err));
        return (int)err;
    }
    return 0;
}

#define B2MD_CHECK_LAUNCH(name)                                        \
    do {                                                               \
        int rc_ = b2md::check_cuda(cudaPeekAtLastError(), name);       \
        if (rc_) return rc_;                                           \
    } while (0)

// Integer A/B knob from the environment, read per call (no cached state in the library).
inline int env_choice(const char *name, int fallback) {
    const char *v = getenv(name);
    return (v && *v) ? atoi(v) : fallback;
}

inline cudaStream_t as_stream(void *s) { return reinterpret_cast<cudaStream_t>(s); }

inline unsigned blocks_for(int64_t n, int threads) {
    return (unsigned)((n + threads - 1) / threads);
}

// Scratch (in int32 units) exclusive_scan_i32 needs for n elements: one 64-bit state word
// per 4096-element tile plus a ticket, with slack for 8-byte alignment (cells.cu).
inline int64_t scan_scratch_ints(int64_t n) {
    return 2 * (((n < 1 ? 1 : n) + 4095) / 4096) + 8;
}
// ... and the kernels it launches: one up to kFusedScanTiles tiles, else three.
constexpr int kFusedScanTiles = 1024;
inline int scan_launches(int64_t n) { return (n + 4095) / 4096 <= kFusedScanTiles ? 1 : 3; }

// Box constants the fp64 (bit-exact) kernels need: L and 1.0/L formed on the
// host in fp64 exactly like the reference (neighbor.py:213-214, core.py:44).
struct BoxD {
    double L[3];
    double invL[3];
};

inline BoxD make_box_d(const b2md_box *box) {
    BoxD b;
    for (int c = 0; c < 3; ++c) {
        b.L[c] = box->edge[c];
        b.invL[c] = 1.0 / box->edge[c];
    }
    return b;
}

// fp32 view of the box for the pair kernels: L = L_hi + L_lo (double-single),
// so that shifting a coordinate by a box length loses nothing.
struct BoxF {
    float L_hi[3];
    float L_lo[3];
    float invL[3];
    float half[3];
};

inline BoxF make_box_f(const b2md_box *box) {
    BoxF b;
    for (int c = 0; c < 3; ++c) {
        b.L_hi[c] = (float)box->edge[c];
        b.L_lo[c] = (float)(box->edge[c] - (double)b.L_hi[c]);
        b.invL[c] = (float)(1.0 / box->edge[c]);
        b.half[c] = (float)(0.5 * box->edge[c]);
    }
    return b;
}

// ---------------------------------------------------------------- device side
__device__ __forceinline__ double ds_to_double(float hi, float lo) {
    // exact: a double-single value has <= 48 significant bits
    return __dadd_rn((double)hi, (double)lo);
}

__device__ __forceinline__ void double_to_ds(double x, float &hi, float &lo) {
    hi = __double2float_rn(x);
    lo = __double2float_rn(__dsub_rn(x, (double)hi));
}

// Error-free a + b -> (s, e) (Knuth two-sum); must not be reassociated.
__device__ __forceinline__ void two_sum(float a, float b, float &s, float &e) {
    s = __fadd_rn(a, b);
    float bb = __fsub_rn(s, a);
    e = __fadd_rn(__fsub_rn(a, __fsub_rn(s, bb)), __fsub_rn(b, bb));
}

// Requires |a| >= |b|.
__device__ __forceinline__ void quick_two_sum(float a, float b, float &s, float &e) {
    s = __fadd_rn(a, b);
    e = __fsub_rn(b, __fsub_rn(s, a));
}

// (hi, lo) += (b_hi, b_lo), renormalised.
__device__ __forceinline__ void ds_add(float &hi, float &lo, float b_hi, float b_lo) {
    float s, e;
    two_sum(hi, b_hi, s, e);
    e = __fadd_rn(e, __fadd_rn(lo, b_lo));
    quick_two_sum(s, e, hi, lo);
}

// Reference minimum image in fp64 without contraction:
// d - L * rint(d * (1/L))   (neighbor.py:140-142)
__device__ __forceinline__ double min_image_f64(double d, double L, double invL) {
    return __dsub_rn(d, __dmul_rn(L, rint(__dmul_rn(d, invL))));
}

__device__ __forceinline__ float warp_max(float v) {
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) v = fmaxf(v, __shfl_xor_sync(0xffffffffu, v, o));
    return v;
}

__device__ __forceinline__ int warp_sum_i(int v) {
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
    return v;
}

}  // namespace b2md
