// Thermodynamic reductions: reference reduce_sum (observables.py:28-74) and the
// observables built on it (observables.py:77-98, sim.py:159-174).
//
// The reference fixes the summation tree: blocks of 4096 values, inside a block
// and across the block partials adjacent pairs are added level by level and an
// odd leftover is carried unchanged.  That tree is position-aligned, so it equals
// a padded power-of-two tree in which a missing right operand leaves the left one
// untouched; and because 4096 is a power of two, the tree over the partials can
// itself be evaluated in 4096-wide blocks, level after level.  Every level here is
// one launch of one CTA per 4096 inputs: 4 consecutive values per thread, then
// shuffle-down by 1,2,4,8,16 lanes, then the 32 warp results by one warp -- the
// same pairing, in fp64, hence bit-identical to the reference for fp64 inputs.
//
// b2md_thermo evaluates the per-particle terms on the fly (fp64 from the fp32
// state, no FMA) and pushes the 8 sums through the tree in one pass over vel,
// force and virial.
#include "common.cuh"

namespace b2md {

constexpr int kTreeThreads = 1024;
constexpr int kTreeItems = 4;
constexpr int kTreeBlock = kTreeThreads * kTreeItems;  // 4096 (observables.py:26)

// x (+) y where y may be absent.
__device__ __forceinline__ double tree_add(double x, double y, bool y_present) {
    return y_present ? __dadd_rn(x, y) : x;
}

// Reduce one 4096-block.  v[q][k] = value k (of 4) of quantity q held by this
// thread, covering block-local elements 4*tid+k; `m` = number of valid elements
// in the block.  Result for every q is returned on thread 0.
template <int NQ>
__device__ __forceinline__ void block_tree(double (&v)[NQ][kTreeItems], int m,
                                           double (&out)[NQ], double *smem /* NQ*32 */) {
    const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
    const int e0 = tid * kTreeItems;
#pragma unroll
    for (int q = 0; q < NQ; ++q) {
        double a = tree_add(v[q][0], v[q][1], e0 + 1 < m);
        double b = tree_add(v[q][2], v[q][3], e0 + 3 < m);
        double s = tree_add(a, b, e0 + 2 < m);
#pragma unroll
        for (int o = 1; o < 32; o <<= 1) {
            const double t = __shfl_down_sync(0xffffffffu, s, o);
            s = tree_add(s, t, (lane + o < 32) && (e0 + o * kTreeItems < m));
        }
        if (lane == 0) smem[q * 32 + warp] = s;
    }
    __syncthreads();
    if (warp == 0) {
#pragma unroll
        for (int q = 0; q < NQ; ++q) {
            double s = smem[q * 32 + lane];
#pragma unroll
            for (int o = 1; o < 32; o <<= 1) {
                const double t = __shfl_down_sync(0xffffffffu, s, o);
                s = tree_add(s, t, (lane + o < 32) && ((lane + o) * 32 * kTreeItems < m));
            }
            out[q] = s;
        }
    }
}

// Generic level: NQ interleaved-by-array inputs in[q * in_stride + e] -> out[q * out_stride + block].
template <int NQ>
__global__ void __launch_bounds__(kTreeThreads)
k_tree_level(const double *__restrict__ in, int64_t n, int64_t in_stride, double *__restrict__ out,
             int64_t out_stride) {
    __shared__ double smem[NQ * 32];
    const int64_t base = (int64_t)blockIdx.x * kTreeBlock;
    const int m = (int)min((int64_t)kTreeBlock, n - base);
    double v[NQ][kTreeItems];
#pragma unroll
    for (int q = 0; q < NQ; ++q)
#pragma unroll
        for (int k = 0; k < kTreeItems; ++k) {
            const int e = threadIdx.x * kTreeItems + k;
            v[q][k] = e < m ? in[q * in_stride + base + e] : 0.0;
        }
    double r[NQ];
    block_tree<NQ>(v, m, r, smem);
    if (threadIdx.x == 0)
#pragma unroll
        for (int q = 0; q < NQ; ++q) out[q * out_stride + blockIdx.x] = r[q];
}

constexpr int kThermoQ = 7;  // e_pot, e_kin, p_x, p_y, p_z, virial, mass

// Level 0 of measure(): per-particle terms from the packed state.
__global__ void __launch_bounds__(kTreeThreads)
k_thermo_level0(const float4 *__restrict__ vel, const float4 *__restrict__ force,
                const float *__restrict__ virial, int64_t n, double *__restrict__ out,
                int64_t out_stride) {
    __shared__ double smem[kThermoQ * 32];
    const int64_t base = (int64_t)blockIdx.x * kTreeBlock;
    const int m = (int)min((int64_t)kTreeBlock, n - base);
    double v[kThermoQ][kTreeItems];
#pragma unroll
    for (int k = 0; k < kTreeItems; ++k) {
        const int e = threadIdx.x * kTreeItems + k;
        if (e < m) {
            const float4 vv = vel[base + e];
            const float4 ff = force[base + e];
            const double mass = (double)vv.w;
            const double vx = vv.x, vy = vv.y, vz = vv.z;
            // 0.5 * m * ((vx*vx + vy*vy) + vz*vz)   (observables.py:82)
            const double v2 = __dadd_rn(__dadd_rn(__dmul_rn(vx, vx), __dmul_rn(vy, vy)),
                                        __dmul_rn(vz, vz));
            v[0][k] = (double)ff.w;
            v[1][k] = __dmul_rn(__dmul_rn(0.5, mass), v2);
            v[2][k] = __dmul_rn(mass, vx);
            v[3][k] = __dmul_rn(mass, vy);
            v[4][k] = __dmul_rn(mass, vz);
            v[5][k] = virial ? (double)virial[base + e] : 0.0;
            v[6][k] = mass;
        } else {
#pragma unroll
            for (int q = 0; q < kThermoQ; ++q) v[q][k] = 0.0;
        }
    }
    double r[kThermoQ];
    block_tree<kThermoQ>(v, m, r, smem);
    if (threadIdx.x == 0)
#pragma unroll
        for (int q = 0; q < kThermoQ; ++q) out[q * out_stride + blockIdx.x] = r[q];
}

__global__ void k_thermo_finish(const double *__restrict__ sums, int64_t stride, int64_t n,
                                double *__restrict__ out8) {
    if (threadIdx.x < kThermoQ) out8[threadIdx.x] = sums[threadIdx.x * stride];
    if (threadIdx.x == kThermoQ) out8[kThermoQ] = (double)n;
}

static inline int64_t n_blocks(int64_t n) { return (n + kTreeBlock - 1) / kTreeBlock; }

// Collapse `nq` arrays of length n (stride in_stride) held in `buf` down to one
// value each, ping-ponging inside scratch.  Returns pointer/stride of the result.
template <int NQ>
static int collapse(const double *in, int64_t n, int64_t in_stride, double *scratch,
                    const double **result, int64_t *result_stride, cudaStream_t s) {
    const double *cur = in;
    int64_t cur_n = n, cur_stride = in_stride;
    double *dst = scratch;
    while (cur_n > 1 || cur == in) {
        const int64_t nb = n_blocks(cur_n);
        k_tree_level<NQ><<<(unsigned)nb, kTreeThreads, 0, s>>>(cur, cur_n, cur_stride, dst, nb);
        cur = dst;
        cur_n = nb;
        cur_stride = nb;
        dst += NQ * nb;
    }
    *result = cur;
    *result_stride = cur_stride;
    B2MD_CHECK_LAUNCH("tree reduce");
    return 0;
}

static int64_t levels_doubles(int64_t n, int nq) {
    int64_t total = 0, cur = n;
    do {
        cur = n_blocks(cur);
        total += nq * cur;
    } while (cur > 1);
    return total + nq;
}

}  // namespace b2md

using namespace b2md;

B2MD_EXPORT int64_t b2md_reduce_scratch_bytes(int64_t n) {
    return (int64_t)sizeof(double) * levels_doubles(n < 1 ? 1 : n, 1);
}

B2MD_EXPORT int b2md_reduce_sum_f64(const double *d_values, int64_t n, double *d_scratch,
                                    double *d_out, void *stream) {
    if (n < 0 || !d_out) { set_error("b2md_reduce_sum_f64: bad arguments"); return -1; }
    cudaStream_t s = as_stream(stream);
    if (n == 0)  // empty input sums to exactly 0.0 (observables.py:51-52)
        return check_cuda(cudaMemsetAsync(d_out, 0, sizeof(double), s), "b2md_reduce_sum_f64");
    const double *res;
    int64_t stride;
    int rc = collapse<1>(d_values, n, n, d_scratch, &res, &stride, s);
    if (rc) return rc;
    return check_cuda(cudaMemcpyAsync(d_out, res, sizeof(double), cudaMemcpyDeviceToDevice, s),
                      "b2md_reduce_sum_f64 copy");
}

B2MD_EXPORT int64_t b2md_thermo_scratch_bytes(int64_t n) {
    return (int64_t)sizeof(double) * levels_doubles(n < 1 ? 1 : n, kThermoQ);
}

B2MD_EXPORT int b2md_thermo(const void *d_vel, const void *d_force_f4, const float *d_virial,
                            int64_t n, double *d_scratch, double *d_out8, void *stream) {
    if (n <= 0 || !d_scratch || !d_out8) { set_error("b2md_thermo: bad arguments"); return -1; }
    cudaStream_t s = as_stream(stream);
    const int64_t nb = n_blocks(n);
    k_thermo_level0<<<(unsigned)nb, kTreeThreads, 0, s>>>(
        (const float4 *)d_vel, (const float4 *)d_force_f4, d_virial, n, d_scratch, nb);
    const double *res = d_scratch;
    int64_t stride = nb;
    if (nb > 1) {
        int rc = collapse<kThermoQ>(d_scratch, nb, nb, d_scratch + kThermoQ * nb, &res, &stride, s);
        if (rc) return rc;
    }
    k_thermo_finish<<<1, 32, 0, s>>>(res, stride, n, d_out8);
    B2MD_CHECK_LAUNCH("b2md_thermo");
    return 0;
}
