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
#include "integrate.cuh"

namespace b2md {

constexpr int kThreads = 256;

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
        float4 h = pos_hi[i];
        d2 = advance_particle<KICKS>(i, h, force[i], pos_lo, vel, image, c, ref_pos);
        pos_hi[i] = h;
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
