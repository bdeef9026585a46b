// Andersen thermostat with counter-based random streams: reference
// andersen_thermostat (integrate.py:82-107) on top of rng.py:40-66.
//
// Every random number is addressed by (seed, stream, step, word): raw 64-bit
// words are Philox4x64-10 with key (seed, 0) and counter (b + 1, 0, stream, step)
// for block b = word / 4 (numpy's Philox increments the counter before producing
// its first block), word % 4 selects the lane; u = ((raw >> 11) + 0.5) * 2^-53;
// normals are the inverse normal CDF of u (Cephes ndtri, the algorithm behind
// scipy.special.ndtri, evaluated in fp64).  At step s the thermostat stream
// supplies n uniforms (word i decides particle i) followed by 3n normals (word
// n + 3 i + c is component c of particle i), all indexed by the LOGICAL particle
// id, so the outcome does not depend on the device row order.
#include <math.h>

#include "common.cuh"
#include "integrate.cuh"

namespace b2md {

struct Words4 { uint64_t w[4]; };

__device__ __forceinline__ Words4 philox4x64_10(uint64_t c0, uint64_t c1, uint64_t c2, uint64_t c3,
                                                uint64_t k0, uint64_t k1) {
    const uint64_t M0 = 0xD2E7470EE14C6C93ull, M1 = 0xCA5A826395121157ull;
    const uint64_t W0 = 0x9E3779B97F4A7C15ull, W1 = 0xBB67AE8584CAA73Bull;
#pragma unroll
    for (int r = 0; r < 10; ++r) {
        const uint64_t hi0 = __umul64hi(M0, c0), lo0 = M0 * c0;
        const uint64_t hi1 = __umul64hi(M1, c2), lo1 = M1 * c2;
        const uint64_t n0 = hi1 ^ c1 ^ k0, n2 = hi0 ^ c3 ^ k1;
        c0 = n0; c1 = lo1; c2 = n2; c3 = lo0;
        k0 += W0; k1 += W1;
    }
    Words4 out;
    out.w[0] = c0; out.w[1] = c1; out.w[2] = c2; out.w[3] = c3;
    return out;
}

__device__ __forceinline__ uint64_t stream_word(uint64_t seed, uint64_t stream, uint64_t step,
                                                uint64_t word) {
    const Words4 b = philox4x64_10(word / 4 + 1, 0, stream, step, seed, 0);
    return b.w[word & 3];
}

__device__ __forceinline__ double word_to_uniform(uint64_t raw) {
    // ((raw >> 11) + 0.5) * 2^-53, exact in fp64 (rng.py:57)
    return __dmul_rn(__dadd_rn((double)(raw >> 11), 0.5), 1.1102230246251565e-16);
}

__device__ __forceinline__ double polevl(double x, const double *c, int n) {
    double a = c[0];
    for (int k = 1; k <= n; ++k) a = __dadd_rn(__dmul_rn(a, x), c[k]);
    return a;
}

__device__ __forceinline__ double p1evl(double x, const double *c, int n) {
    double a = __dadd_rn(x, c[0]);
    for (int k = 1; k < n; ++k) a = __dadd_rn(__dmul_rn(a, x), c[k]);
    return a;
}

// Inverse of the standard normal CDF, Cephes ndtri (Moshier), fp64, no FMA.
__device__ double ndtri_f64(double y0) {
    const double P0[5] = {-5.99633501014107895267E1, 9.80010754185999661536E1,
                          -5.66762857469070293439E1, 1.39312609387279679503E1,
                          -1.23916583867381258016E0};
    const double Q0[8] = {1.95448858338141759834E0, 4.67627912898881538453E0,
                          8.63602421390890590575E1, -2.25462687854119370527E2,
                          2.00260212380060660359E2, -8.20372256168333339912E1,
                          1.59056225126211695515E1, -1.18331621121330003142E0};
    const double P1[9] = {4.05544892305962419923E0, 3.15251094599893866154E1,
                          5.71628192246421288162E1, 4.40805073893200834700E1,
                          1.46849561928858024014E1, 2.18663306850790267539E0,
                          -1.40256079171354495875E-1, -3.50424626827848203418E-2,
                          -8.57456785154685413611E-4};
    const double Q1[8] = {1.57799883256466749731E1, 4.53907635128879210584E1,
                          4.13172038254672030440E1, 1.50425385692907503408E1,
                          2.50464946208309415979E0, -1.42182922854787788574E-1,
                          -3.80806407691578277194E-2, -9.33259480895457427372E-4};
    const double P2[9] = {3.23774891776946035970E0, 6.91522889068984211695E0,
                          3.93881025292474443415E0, 1.33303460815807542389E0,
                          2.01485389549179081538E-1, 1.23716634817820021358E-2,
                          3.01581553508235416007E-4, 2.65806974686737550832E-6,
                          6.23974539184983293730E-9};
    const double Q2[8] = {6.02427039364742014255E0, 3.67983563856160859403E0,
                          1.37702099489081330271E0, 2.16236993594496635890E-1,
                          1.34204006088543189037E-2, 3.28014464682127739104E-4,
                          2.89247864745380683936E-6, 6.79019408009981274425E-9};
    const double s2pi = 2.50662827463100050242E0, expm2 = 0.13533528323661269189;
    bool negate = true;
    double y = y0;
    if (y > __dsub_rn(1.0, expm2)) { y = __dsub_rn(1.0, y); negate = false; }
    if (y > expm2) {
        y = __dsub_rn(y, 0.5);
        const double y2 = __dmul_rn(y, y);
        const double x = __dadd_rn(y, __dmul_rn(y, __ddiv_rn(__dmul_rn(y2, polevl(y2, P0, 4)),
                                                             p1evl(y2, Q0, 8))));
        return __dmul_rn(x, s2pi);
    }
    double x = sqrt(__dmul_rn(-2.0, log(y)));
    const double x0 = __dsub_rn(x, __ddiv_rn(log(x), x));
    const double z = __ddiv_rn(1.0, x);
    const double x1 = x < 8.0 ? __ddiv_rn(__dmul_rn(z, polevl(z, P1, 8)), p1evl(z, Q1, 8))
                              : __ddiv_rn(__dmul_rn(z, polevl(z, P2, 8)), p1evl(z, Q2, 8));
    x = __dsub_rn(x0, x1);
    return negate ? -x : x;
}

// The thermostat's decision and draw for logical particle i (integrate.py:96-104): true if
// the velocity v (w = mass) was redrawn.
__device__ __forceinline__ bool andersen_redraw(float4 &v, uint64_t i, int64_t n, uint64_t seed,
                                                uint64_t step, double p, double temperature) {
    const double u = word_to_uniform(stream_word(seed, 0, step, i));
    if (!(u < p)) return false;                       // integrate.py:96 `redraw = u < p`
    const double scale = sqrt(__ddiv_rn(temperature, (double)v.w));   // sqrt(T / m)
    const uint64_t base = (uint64_t)n + 3 * i;
    v.x = (float)__dmul_rn(ndtri_f64(word_to_uniform(stream_word(seed, 0, step, base))), scale);
    v.y = (float)__dmul_rn(ndtri_f64(word_to_uniform(stream_word(seed, 0, step, base + 1))), scale);
    v.z = (float)__dmul_rn(ndtri_f64(word_to_uniform(stream_word(seed, 0, step, base + 2))), scale);
    return true;
}

__global__ void k_andersen(float4 *__restrict__ vel, const float4 *__restrict__ ids, int64_t n,
                           uint64_t seed, uint64_t step, double p, double temperature,
                           int32_t *__restrict__ redrawn) {
    const int64_t r = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
    int hit = 0;
    if (r < n) {
        const uint64_t i = ids ? (uint64_t)(uint32_t)__float_as_int(ids[r].w) : (uint64_t)r;
        float4 v = vel[r];
        if (andersen_redraw(v, i, n, seed, step, p, temperature)) {
            hit = 1;
            vel[r] = v;
        }
    }
    hit = warp_sum_i(hit);
    if ((threadIdx.x & 31) == 0 && hit && redrawn) atomicAdd(redrawn, hit);
}

// The finalize slots of a thermostatted step in one pass over the velocities (sim.py:86-87):
// vv_finalize (second half-kick with the new forces, integrate.py:73-79), then the thermostat;
// with INTEGRATE also vv_integrate of the NEXT step (first half-kick with the same forces,
// drift, wrap, image counters, displacement check -- the body of k_integrate<1>).  Per particle
// the operations and their order are those of the separate launches: bit-identical.
constexpr int kFusedThreads = 256;

template <bool INTEGRATE>
__global__ void __launch_bounds__(kFusedThreads)
k_finalize_andersen(float4 *__restrict__ pos_hi, float4 *__restrict__ pos_lo,
                    float4 *__restrict__ vel, const float4 *__restrict__ force,
                    int4 *__restrict__ image, int64_t n, const StepConst c,
                    float4 *__restrict__ ref_pos, b2md_status *status, uint64_t seed,
                    uint64_t step, double p, double temperature) {
    __shared__ float s_max[kFusedThreads / 32];
    const int64_t r = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
    float d2 = 0.0f;
    if (r < n) {
        float4 v = vel[r];
        const float4 f = force[r];
        kick(v, f, c.half_dt);                                        // vv_finalize
        float4 l = pos_lo[r];                                         // (w = logical id)
        const uint64_t i = (uint64_t)(uint32_t)__float_as_int(l.w);
        andersen_redraw(v, i, n, seed, step, p, temperature);
        if (INTEGRATE) {
            float4 h = pos_hi[r];
            float4 ref = ref_pos ? ref_pos[r] : make_float4(0.f, 0.f, 0.f, 0.f);
            const float4 ref0 = ref;
            d2 = advance_regs<1>(r, h, l, v, ref, ref_pos != nullptr, f, image, c);
            pos_hi[r] = h;
            pos_lo[r] = l;
            if (ref_pos && (ref.x != ref0.x || ref.y != ref0.y || ref.z != ref0.z)) ref_pos[r] = ref;
        }
        vel[r] = v;
    }
    if (INTEGRATE && ref_pos) {
        d2 = warp_max(d2);
        if ((threadIdx.x & 31) == 0) s_max[threadIdx.x >> 5] = d2;
        __syncthreads();
        if (threadIdx.x < 32) {
            float m = threadIdx.x < kFusedThreads / 32 ? s_max[threadIdx.x] : 0.0f;
            m = warp_max(m);
            if (threadIdx.x == 0 && m > 0.0f) {
                atomicMax(&status->max_disp2_bits, __float_as_uint(m));
                if (m > c.half_skin2) status->rebuild_flag = 1;
            }
        }
    }
}

__global__ void k_stream_words(uint64_t seed, uint64_t stream, uint64_t step, int64_t offset,
                               int64_t count, uint64_t *__restrict__ raw,
                               double *__restrict__ uniform, double *__restrict__ normal) {
    const int64_t k = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
    if (k >= count) return;
    const uint64_t w = stream_word(seed, stream, step, (uint64_t)(offset + k));
    if (raw) raw[k] = w;
    const double u = word_to_uniform(w);
    if (uniform) uniform[k] = u;
    if (normal) normal[k] = ndtri_f64(u);
}

}  // namespace b2md

using namespace b2md;

B2MD_EXPORT int b2md_andersen(void *d_vel, const void *d_ids_pos_lo, int64_t n, uint64_t seed,
                              uint64_t step, double probability, double temperature,
                              int32_t *d_redrawn, void *stream) {
    if (n <= 0 || !(temperature > 0.0) || !(probability >= 0.0)) {
        set_error("b2md_andersen: bad arguments");
        return -1;
    }
    cudaStream_t s = as_stream(stream);
    if (d_redrawn) {
        int rc = check_cuda(cudaMemsetAsync(d_redrawn, 0, sizeof(int32_t), s), "andersen memset");
        if (rc) return rc;
    }
    if (probability <= 0.0) return 0;
    k_andersen<<<blocks_for(n, 128), 128, 0, s>>>((float4 *)d_vel, (const float4 *)d_ids_pos_lo, n,
                                                  seed, step, probability, temperature, d_redrawn);
    B2MD_CHECK_LAUNCH("b2md_andersen");
    return 0;
}

B2MD_EXPORT int b2md_vv_finalize_andersen(void *d_pos_hi, void *d_pos_lo, void *d_vel,
                                          const void *d_force_f4, void *d_image_i4, int64_t n,
                                          const b2md_box *box, double dt, uint64_t seed,
                                          uint64_t step, double probability, double temperature,
                                          int32_t integrate_next, void *d_ref_pos_f4,
                                          double half_skin2, b2md_status *d_status, void *stream) {
    if (n <= 0 || !box || !(dt > 0.0) || !d_pos_lo || !d_vel || !d_force_f4 ||
        !(temperature > 0.0) || !(probability >= 0.0) ||
        (integrate_next && (!d_pos_hi || !d_image_i4)) || (d_ref_pos_f4 && !d_status)) {
        set_error("b2md_vv_finalize_andersen: bad arguments");
        return -1;
    }
    const StepConst c = make_step(box, dt, half_skin2);
    cudaStream_t s = as_stream(stream);
    const unsigned blocks = blocks_for(n, kFusedThreads);
    if (integrate_next)
        k_finalize_andersen<true><<<blocks, kFusedThreads, 0, s>>>(
            (float4 *)d_pos_hi, (float4 *)d_pos_lo, (float4 *)d_vel, (const float4 *)d_force_f4,
            (int4 *)d_image_i4, n, c, (float4 *)d_ref_pos_f4, d_status, seed, step, probability,
            temperature);
    else
        k_finalize_andersen<false><<<blocks, kFusedThreads, 0, s>>>(
            (float4 *)d_pos_hi, (float4 *)d_pos_lo, (float4 *)d_vel, (const float4 *)d_force_f4,
            (int4 *)d_image_i4, n, c, nullptr, d_status, seed, step, probability, temperature);
    B2MD_CHECK_LAUNCH("b2md_vv_finalize_andersen");
    return 0;
}

B2MD_EXPORT int b2md_stream_words(uint64_t seed, uint64_t stream_id, uint64_t step,
                                  int64_t word_offset, int64_t count, uint64_t *d_raw,
                                  double *d_uniform, double *d_normal, void *stream) {
    if (count < 0 || word_offset < 0) { set_error("b2md_stream_words: bad arguments"); return -1; }
    if (count == 0) return 0;
    k_stream_words<<<blocks_for(count, 128), 128, 0, as_stream(stream)>>>(
        seed, stream_id, step, word_offset, count, d_raw, d_uniform, d_normal);
    B2MD_CHECK_LAUNCH("b2md_stream_words");
    return 0;
}
