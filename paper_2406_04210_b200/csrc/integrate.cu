// Velocity Verlet: reference vv_integrate (integrate.py:58-70), wrap_position
// (core.py:72-93), vv_finalize (integrate.py:73-79), plus the in-loop form of
// needs_rebuild (neighbor.py:243-254).
//
// Positions are double-single (hi + lo, ~48 significant bits) as in the paper's
// CUDA code, so the drift r += v*dt does not lose the small increment against a
// coordinate of order L; velocities and forces are fp32.  One pass over the
// state: reads pos_hi, pos_lo, vel, force (+ the list's reference positions),
// writes pos_hi, pos_lo, vel.  Images and the reference copy are touched only for
// the few particles that cross a periodic face in this step.
#include <math.h>

#include "common.cuh"

namespace b2md {

constexpr int kThreads = 256;

struct StepConst {
    float L_hi[3], L_lo[3], invL[3];
    float dt_hi, dt_lo, half_dt;
    float half_skin2;
};

// x (double-single) into [0, L): k = floor(x/L) with the reference's nudges
// (core.py:81-93); returns k.
__device__ __forceinline__ int wrap_ds(float &hi, float &lo, float L_hi, float L_lo, float invL) {
    if (hi >= 0.0f && hi < L_hi) return 0;          // common case (hi == L_hi handled below)
    float kf = floorf(hi * invL);
    if (kf != 0.0f) {
        // (hi, lo) -= k * (L_hi + L_lo), product formed error-free
        const float ph = kf * L_hi;
        const float pl = fmaf(kf, L_hi, -ph) + kf * L_lo;
        ds_add(hi, lo, -ph, -pl);
    }
    // value < 0 ?
    if (hi < 0.0f || (hi == 0.0f && lo < 0.0f)) {
        ds_add(hi, lo, L_hi, L_lo);
        kf -= 1.0f;
    }
    // value >= L ?
    if (hi > L_hi || (hi == L_hi && lo >= L_lo)) {
        ds_add(hi, lo, -L_hi, -L_lo);
        kf += 1.0f;
    }
    return (int)kf;
}

__device__ __forceinline__ void kick(float4 &v, const float4 f, float half_dt) {
    // v += (f / m) * (0.5*dt): divide, then multiply (integrate.py:64,79)
    const float m = v.w;
    v.x = __fadd_rn(v.x, __fmul_rn(__fdiv_rn(f.x, m), half_dt));
    v.y = __fadd_rn(v.y, __fmul_rn(__fdiv_rn(f.y, m), half_dt));
    v.z = __fadd_rn(v.z, __fmul_rn(__fdiv_rn(f.z, m), half_dt));
}

__device__ __forceinline__ void drift(float &hi, float &lo, float v, float dt_hi, float dt_lo) {
    const float ph = v * dt_hi;
    const float pl = fmaf(v, dt_lo, fmaf(v, dt_hi, -ph));   // exact product tail
    ds_add(hi, lo, ph, pl);
}

template <int KICKS, bool GATED>
__global__ void __launch_bounds__(kThreads)
k_integrate(float4 *__restrict__ pos_hi, float4 *__restrict__ pos_lo, float4 *__restrict__ vel,
            const float4 *__restrict__ force, int4 *__restrict__ image, int64_t n,
            const StepConst c, float4 *__restrict__ ref_pos, b2md_status *status) {
    __shared__ float s_max[kThreads / 32];
    // step-graph batches stop advancing once an in-graph list build overflowed
    if (GATED && *(volatile int *)&status->frozen) return;
    const int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
    float d2 = 0.0f;
    if (i < n) {
        float4 v = vel[i];
        const float4 f = force[i];
#pragma unroll
        for (int k = 0; k < KICKS; ++k) kick(v, f, c.half_dt);
        vel[i] = v;
        float4 h = pos_hi[i], l = pos_lo[i];
        drift(h.x, l.x, v.x, c.dt_hi, c.dt_lo);
        drift(h.y, l.y, v.y, c.dt_hi, c.dt_lo);
        drift(h.z, l.z, v.z, c.dt_hi, c.dt_lo);
        const int kx = wrap_ds(h.x, l.x, c.L_hi[0], c.L_lo[0], c.invL[0]);
        const int ky = wrap_ds(h.y, l.y, c.L_hi[1], c.L_lo[1], c.invL[1]);
        const int kz = wrap_ds(h.z, l.z, c.L_hi[2], c.L_lo[2], c.invL[2]);
        pos_hi[i] = h;
        pos_lo[i] = l;
        const bool wrapped = (kx | ky | kz) != 0;
        if (wrapped) {
            int4 im = image[i];
            im.x += kx; im.y += ky; im.z += kz;
            image[i] = im;
        }
        if (ref_pos) {
            float4 r = ref_pos[i];
            if (wrapped) {
                // keep (hi - ref) equal to the unwrapped displacement
                r.x = fmaf(-(float)kx, c.L_hi[0], r.x);
                r.y = fmaf(-(float)ky, c.L_hi[1], r.y);
                r.z = fmaf(-(float)kz, c.L_hi[2], r.z);
                ref_pos[i] = r;
            }
            const float dx = h.x - r.x, dy = h.y - r.y, dz = h.z - r.z;
            d2 = fmaf(dz, dz, fmaf(dy, dy, dx * dx));
        }
    }
    if (ref_pos) {
        d2 = warp_max(d2);
        if ((threadIdx.x & 31) == 0) s_max[threadIdx.x >> 5] = d2;
        __syncthreads();
        if (threadIdx.x < 32) {
            float m = threadIdx.x < kThreads / 32 ? s_max[threadIdx.x] : 0.0f;
            m = warp_max(m);
            if (threadIdx.x == 0 && m > 0.0f) {
                // non-negative floats order like their bit patterns
                atomicMax(&status->max_disp2_bits, __float_as_uint(m));
                if (m > c.half_skin2) status->rebuild_flag = 1;
            }
        }
    }
}

__global__ void __launch_bounds__(kThreads)
k_finalize(float4 *__restrict__ vel, const float4 *__restrict__ force, int64_t n, float half_dt) {
    const int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
    if (i >= n) return;
    float4 v = vel[i];
    kick(v, force[i], half_dt);
    vel[i] = v;
}

static StepConst make_step(const b2md_box *box, double dt, double half_skin2) {
    StepConst c;
    for (int a = 0; a < 3; ++a) {
        c.L_hi[a] = (float)box->edge[a];
        c.L_lo[a] = (float)(box->edge[a] - (double)c.L_hi[a]);
        c.invL[a] = (float)(1.0 / box->edge[a]);
    }
    c.dt_hi = (float)dt;
    c.dt_lo = (float)(dt - (double)c.dt_hi);
    c.half_dt = (float)(0.5 * dt);
    // never fire later than the exact fp64 test: shave the fp32 rounding of the
    // snapshot and of the squared norm off the threshold
    c.half_skin2 = (float)(half_skin2 * (1.0 - 1e-5));
    return c;
}

template <int KICKS, bool GATED = false>
static int launch_integrate(void *d_pos_hi, void *d_pos_lo, void *d_vel, const void *d_force,
                            void *d_image, int64_t n, const b2md_box *box, double dt,
                            void *d_ref_pos, double half_skin2, b2md_status *d_status,
                            void *stream, const char *name) {
    if (n <= 0 || !box || !(dt > 0.0)) { set_error("%s: bad arguments", name); return -1; }
    if (d_ref_pos && !d_status) { set_error("%s: displacement check needs a status block", name); return -2; }
    if (GATED && !d_status) { set_error("%s: gated launch needs a status block", name); return -3; }
    k_integrate<KICKS, GATED><<<blocks_for(n, kThreads), kThreads, 0, as_stream(stream)>>>(
        (float4 *)d_pos_hi, (float4 *)d_pos_lo, (float4 *)d_vel, (const float4 *)d_force,
        (int4 *)d_image, n, make_step(box, dt, half_skin2), (float4 *)d_ref_pos, d_status);
    B2MD_CHECK_LAUNCH(name);
    return 0;
}

}  // namespace b2md

using namespace b2md;

B2MD_EXPORT int b2md_vv_integrate(void *d_pos_hi, void *d_pos_lo, void *d_vel,
                                  const void *d_force_f4, void *d_image_i4, int64_t n,
                                  const b2md_box *box, double dt, void *d_ref_pos_f4,
                                  double half_skin2, b2md_status *d_status, void *stream) {
    return launch_integrate<1>(d_pos_hi, d_pos_lo, d_vel, d_force_f4, d_image_i4, n, box, dt,
                               d_ref_pos_f4, half_skin2, d_status, stream, "b2md_vv_integrate");
}

B2MD_EXPORT int b2md_vv_finalize_integrate(void *d_pos_hi, void *d_pos_lo, void *d_vel,
                                           const void *d_force_f4, void *d_image_i4, int64_t n,
                                           const b2md_box *box, double dt, void *d_ref_pos_f4,
                                           double half_skin2, b2md_status *d_status,
                                           void *stream) {
    return launch_integrate<2>(d_pos_hi, d_pos_lo, d_vel, d_force_f4, d_image_i4, n, box, dt,
                               d_ref_pos_f4, half_skin2, d_status, stream,
                               "b2md_vv_finalize_integrate");
}

B2MD_EXPORT int b2md_vv_integrate_gated(void *d_pos_hi, void *d_pos_lo, void *d_vel,
                                        const void *d_force_f4, void *d_image_i4, int64_t n,
                                        const b2md_box *box, double dt, void *d_ref_pos_f4,
                                        double half_skin2, b2md_status *d_status, int32_t kicks,
                                        void *stream) {
    if (kicks == 2)
        return launch_integrate<2, true>(d_pos_hi, d_pos_lo, d_vel, d_force_f4, d_image_i4, n, box,
                                         dt, d_ref_pos_f4, half_skin2, d_status, stream,
                                         "b2md_vv_integrate_gated");
    return launch_integrate<1, true>(d_pos_hi, d_pos_lo, d_vel, d_force_f4, d_image_i4, n, box, dt,
                                     d_ref_pos_f4, half_skin2, d_status, stream,
                                     "b2md_vv_integrate_gated");
}

B2MD_EXPORT int b2md_vv_finalize(void *d_vel, const void *d_force_f4, int64_t n, double dt,
                                 void *stream) {
    if (n <= 0 || !(dt > 0.0)) { set_error("b2md_vv_finalize: bad arguments"); return -1; }
    k_finalize<<<blocks_for(n, kThreads), kThreads, 0, as_stream(stream)>>>(
        (float4 *)d_vel, (const float4 *)d_force_f4, n, (float)(0.5 * dt));
    B2MD_CHECK_LAUNCH("b2md_vv_finalize");
    return 0;
}
