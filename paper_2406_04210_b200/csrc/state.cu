// HOST <-> COMPUTE format conversion (replaces TrackedBuffer's np.copyto,
// reference core.py:131-137), status block handling, error reporting.
#include <stdarg.h>

#include "common.cuh"

namespace b2md {

static thread_local char g_error[512] = "no error";

void set_error(const char *fmt, ...) {
    va_list ap;
    va_start(ap, fmt);
    vsnprintf(g_error, sizeof(g_error), fmt, ap);
    va_end(ap);
}

constexpr int kThreads = 256;

__device__ __forceinline__ int64_t logical_row(const float4 *ids, int64_t r) {
    return ids ? (int64_t)__float_as_int(ids[r].w) : r;
}

__global__ void k_status_reset(b2md_status *st, bool keep_singular) {
    st->overflow = 0;
    st->max_count = 0;
    if (!keep_singular) st->singular = ~0ull;
    st->max_disp2_bits = 0u;
    st->rebuild_flag = 0;
    st->max_disp2_f64_bits = 0ull;
    st->n_boundary = 0;
    // graph_steps / graph_rebuilds / frozen belong to the step-graph batch and are
    // reset by the runner, not here
    for (int k = 0; k < 4; ++k) st->reserved[k] = 0;
}

__global__ void k_pack_positions(const double *__restrict__ src, int64_t n,
                                 const float4 *__restrict__ ids, float4 *hi, float4 *lo) {
    int64_t r = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
    if (r >= n) return;
    int64_t s = logical_row(ids, r);
    float4 h = hi[r], l = lo[r];
    double_to_ds(src[3 * s + 0], h.x, l.x);
    double_to_ds(src[3 * s + 1], h.y, l.y);
    double_to_ds(src[3 * s + 2], h.z, l.z);
    hi[r] = h;
    lo[r] = l;
}

__global__ void k_unpack_positions(const float4 *__restrict__ hi, const float4 *__restrict__ lo,
                                   int64_t n, const float4 *__restrict__ ids, double *dst) {
    int64_t r = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
    if (r >= n) return;
    int64_t s = logical_row(ids, r);
    float4 h = hi[r], l = lo[r];
    dst[3 * s + 0] = ds_to_double(h.x, l.x);
    dst[3 * s + 1] = ds_to_double(h.y, l.y);
    dst[3 * s + 2] = ds_to_double(h.z, l.z);
}

__global__ void k_pack_vec3(const double *__restrict__ src, int64_t n,
                            const float4 *__restrict__ ids, float4 *dst) {
    int64_t r = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
    if (r >= n) return;
    int64_t s = logical_row(ids, r);
    float4 v = dst[r];
    v.x = (float)src[3 * s + 0];
    v.y = (float)src[3 * s + 1];
    v.z = (float)src[3 * s + 2];
    dst[r] = v;
}

__global__ void k_unpack_vec3(const float4 *__restrict__ src, int64_t n,
                              const float4 *__restrict__ ids, double *dst) {
    int64_t r = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
    if (r >= n) return;
    int64_t s = logical_row(ids, r);
    float4 v = src[r];
    dst[3 * s + 0] = (double)v.x;
    dst[3 * s + 1] = (double)v.y;
    dst[3 * s + 2] = (double)v.z;
}

__global__ void k_pack_w_f64(const double *__restrict__ src, int64_t n,
                             const float4 *__restrict__ ids, float4 *dst) {
    int64_t r = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
    if (r >= n) return;
    dst[r].w = (float)src[logical_row(ids, r)];
}

__global__ void k_unpack_w_f64(const float4 *__restrict__ src, int64_t n,
                               const float4 *__restrict__ ids, double *dst) {
    int64_t r = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
    if (r >= n) return;
    dst[logical_row(ids, r)] = (double)src[r].w;
}

__global__ void k_pack_w_i32(const int32_t *__restrict__ src, int64_t n,
                             const float4 *__restrict__ ids, float4 *dst) {
    int64_t r = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
    if (r >= n) return;
    dst[r].w = __int_as_float(src[logical_row(ids, r)]);
}

__global__ void k_unpack_w_i32(const float4 *__restrict__ src, int64_t n,
                               const float4 *__restrict__ ids, int32_t *dst) {
    int64_t r = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
    if (r >= n) return;
    dst[logical_row(ids, r)] = __float_as_int(src[r].w);
}

__global__ void k_pack_images(const int64_t *__restrict__ src, int64_t n,
                              const float4 *__restrict__ ids, int4 *dst) {
    int64_t r = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
    if (r >= n) return;
    int64_t s = logical_row(ids, r);
    dst[r] = make_int4((int)src[3 * s], (int)src[3 * s + 1], (int)src[3 * s + 2], 0);
}

__global__ void k_unpack_images(const int4 *__restrict__ src, int64_t n,
                                const float4 *__restrict__ ids, int64_t *dst) {
    int64_t r = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
    if (r >= n) return;
    int64_t s = logical_row(ids, r);
    int4 v = src[r];
    dst[3 * s] = v.x;
    dst[3 * s + 1] = v.y;
    dst[3 * s + 2] = v.z;
}

__global__ void k_pack_scalar(const double *__restrict__ src, int64_t n,
                              const float4 *__restrict__ ids, float *dst) {
    int64_t r = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
    if (r >= n) return;
    dst[r] = (float)src[logical_row(ids, r)];
}

__global__ void k_unpack_scalar(const float *__restrict__ src, int64_t n,
                                const float4 *__restrict__ ids, double *dst) {
    int64_t r = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
    if (r >= n) return;
    dst[logical_row(ids, r)] = (double)src[r];
}

__global__ void k_set_ids(float4 *lo, int64_t n) {
    int64_t r = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
    if (r >= n) return;
    lo[r].w = __int_as_float((int)r);
}

__global__ void k_get_ids(const float4 *__restrict__ lo, int64_t n, int32_t *ids) {
    int64_t r = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
    if (r >= n) return;
    ids[r] = __float_as_int(lo[r].w);
}

}  // namespace b2md

using namespace b2md;

B2MD_EXPORT int b2md_version(void) { return B2MD_VERSION; }

B2MD_EXPORT const char *b2md_last_error_string(void) { return g_error; }

B2MD_EXPORT int b2md_status_reset(b2md_status *d_status, void *stream) {
    if (!d_status) { set_error("b2md_status_reset: null status"); return -1; }
    k_status_reset<<<1, 1, 0, as_stream(stream)>>>(d_status, false);
    B2MD_CHECK_LAUNCH("b2md_status_reset");
    return 0;
}

B2MD_EXPORT int b2md_status_reset_list(b2md_status *d_status, void *stream) {
    if (!d_status) { set_error("b2md_status_reset_list: null status"); return -1; }
    k_status_reset<<<1, 1, 0, as_stream(stream)>>>(d_status, true);
    B2MD_CHECK_LAUNCH("b2md_status_reset_list");
    return 0;
}

#define B2MD_ROWWISE(fn, kernel, ...)                                              \
    do {                                                                           \
        if (n < 0) { set_error(fn ": negative n"); return -1; }                    \
        if (n == 0) return 0;                                                      \
        kernel<<<blocks_for(n, kThreads), kThreads, 0, as_stream(stream)>>>(__VA_ARGS__); \
        B2MD_CHECK_LAUNCH(fn);                                                     \
        return 0;                                                                  \
    } while (0)

B2MD_EXPORT int b2md_pack_positions(const double *d_pos_f64, int64_t n, const void *d_ids,
                                    void *d_pos_hi, void *d_pos_lo, void *stream) {
    B2MD_ROWWISE("b2md_pack_positions", k_pack_positions, d_pos_f64, n, (const float4 *)d_ids,
                 (float4 *)d_pos_hi, (float4 *)d_pos_lo);
}

B2MD_EXPORT int b2md_unpack_positions(const void *d_pos_hi, const void *d_pos_lo, int64_t n,
                                      const void *d_ids, double *d_pos_f64, void *stream) {
    B2MD_ROWWISE("b2md_unpack_positions", k_unpack_positions, (const float4 *)d_pos_hi,
                 (const float4 *)d_pos_lo, n, (const float4 *)d_ids, d_pos_f64);
}

B2MD_EXPORT int b2md_pack_vec3(const double *d_src, int64_t n, const void *d_ids, void *d_dst,
                               void *stream) {
    B2MD_ROWWISE("b2md_pack_vec3", k_pack_vec3, d_src, n, (const float4 *)d_ids, (float4 *)d_dst);
}

B2MD_EXPORT int b2md_unpack_vec3(const void *d_src, int64_t n, const void *d_ids, double *d_dst,
                                 void *stream) {
    B2MD_ROWWISE("b2md_unpack_vec3", k_unpack_vec3, (const float4 *)d_src, n,
                 (const float4 *)d_ids, d_dst);
}

B2MD_EXPORT int b2md_pack_w_f64(const double *d_src, int64_t n, const void *d_ids, void *d_dst,
                                void *stream) {
    B2MD_ROWWISE("b2md_pack_w_f64", k_pack_w_f64, d_src, n, (const float4 *)d_ids, (float4 *)d_dst);
}

B2MD_EXPORT int b2md_unpack_w_f64(const void *d_src, int64_t n, const void *d_ids, double *d_dst,
                                  void *stream) {
    B2MD_ROWWISE("b2md_unpack_w_f64", k_unpack_w_f64, (const float4 *)d_src, n,
                 (const float4 *)d_ids, d_dst);
}

B2MD_EXPORT int b2md_pack_w_i32(const int32_t *d_src, int64_t n, const void *d_ids, void *d_dst,
                                void *stream) {
    B2MD_ROWWISE("b2md_pack_w_i32", k_pack_w_i32, d_src, n, (const float4 *)d_ids, (float4 *)d_dst);
}

B2MD_EXPORT int b2md_unpack_w_i32(const void *d_src, int64_t n, const void *d_ids,
                                  int32_t *d_dst, void *stream) {
    B2MD_ROWWISE("b2md_unpack_w_i32", k_unpack_w_i32, (const float4 *)d_src, n,
                 (const float4 *)d_ids, d_dst);
}

B2MD_EXPORT int b2md_pack_images(const int64_t *d_src, int64_t n, const void *d_ids,
                                 void *d_image, void *stream) {
    B2MD_ROWWISE("b2md_pack_images", k_pack_images, d_src, n, (const float4 *)d_ids,
                 (int4 *)d_image);
}

B2MD_EXPORT int b2md_unpack_images(const void *d_image, int64_t n, const void *d_ids,
                                   int64_t *d_dst, void *stream) {
    B2MD_ROWWISE("b2md_unpack_images", k_unpack_images, (const int4 *)d_image, n,
                 (const float4 *)d_ids, d_dst);
}

B2MD_EXPORT int b2md_pack_scalar_f32(const double *d_src, int64_t n, const void *d_ids,
                                     float *d_dst, void *stream) {
    B2MD_ROWWISE("b2md_pack_scalar_f32", k_pack_scalar, d_src, n, (const float4 *)d_ids, d_dst);
}

B2MD_EXPORT int b2md_unpack_scalar_f32(const float *d_src, int64_t n, const void *d_ids,
                                       double *d_dst, void *stream) {
    B2MD_ROWWISE("b2md_unpack_scalar_f32", k_unpack_scalar, d_src, n, (const float4 *)d_ids,
                 d_dst);
}

B2MD_EXPORT int b2md_set_ids(void *d_pos_lo, int64_t n, void *stream) {
    B2MD_ROWWISE("b2md_set_ids", k_set_ids, (float4 *)d_pos_lo, n);
}

B2MD_EXPORT int b2md_get_ids(const void *d_pos_lo, int64_t n, int32_t *d_ids, void *stream) {
    B2MD_ROWWISE("b2md_get_ids", k_get_ids, (const float4 *)d_pos_lo, n, d_ids);
}
