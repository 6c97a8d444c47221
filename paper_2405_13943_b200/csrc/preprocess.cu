// K1 preprocess_fwd: per-Gaussian EWA projection, SH colour, footprint rect
// and tile count. Replaces project_gaussian / project_cloud / footprint /
// covariance_from_params / sh_color (renderer.cpp:14-40,63-91,121-134;
// cloud.cpp:162-193).
//
// The arithmetic that decides integers (culling, footprint rect, depth order)
// is FP64 and written in the reference's evaluation order; this file is
// compiled with --fmad=false so no multiply-add is contracted, which makes the
// rects and depth keys bit-identical to the FP64 CPU path given the same
// (FP32-stored) parameters. Outputs consumed by the FP32 blend are rounded
// once at the end. Bound: HBM (56 B read + 48 B record + 12 B key/count per
// row) with ~300 FP64 flops per row.
#include "bsg_internal.cuh"

namespace bsg {
namespace {

__device__ __forceinline__ int to_int_clamped(double v) {
    // renderer.cpp:35-38 casts with static_cast<int>; out-of-range values are
    // pinned to +-2^30 first (identical for every in-range value; see oracle).
    if (v < -1073741824.0) return -1073741824;
    if (v > 1073741824.0) return 1073741824;
    return static_cast<int>(v);
}

__device__ __forceinline__ float rcp_approx(float x) {
    float r;
    asm("rcp.approx.ftz.f32 %0, %1;" : "=f"(r) : "f"(x));
    return r;
}
__device__ __forceinline__ float exp2f_approx(float x) {
    float r;
    asm("ex2.approx.ftz.f32 %0, %1;" : "=f"(r) : "f"(x));
    return r;
}
__device__ __forceinline__ float sqrt_approx(float x) {
    float r;
    asm("sqrt.approx.ftz.f32 %0, %1;" : "=f"(r) : "f"(x));
    return r;
}

// 128-thread CTAs, 6 per SM: a CTA's barriers (between the cull, the replays
// and the projection) stall 4 warps instead of 8 (cfg 3: 256 x 3 rows per
// thread-batch 214 us, 128: 208 us, 64 x 12 CTAs: 208 us).
constexpr int kPreThreads = 128;
constexpr int kPreRowsPerThread = 4;
// Phase 1 in batches of kPreRowsPerThread rows per thread, 1536 rows per CTA:
// larger chunks give phase 2 (replays, exact projection) more candidates per
// CTA to spread over its warps (measured at cfg 3 with 256 threads: 1024 /
// 2048 / 4096 / 6144 rows per CTA -> 248 / 240 / 229 / 246 us; later 3072 /
// 4096 / 5120 -> 214 / 220 / 224 us; with 128 threads 1024 / 1536 / 2048 ->
// 218 / 208 / 215 us).
constexpr int kPreSubBatches = 3;
constexpr int kPreChunk = kPreThreads * kPreRowsPerThread * kPreSubBatches;

// Two phases per CTA over a chunk of kPreChunk rows. Phase 1 (FP32, every row):
// a conservative reject -- lambda_max(cov2d) <= |J|_F^2 max(s)^2 + dilation
// (A = J W with W orthonormal, |Sigma|_2 = max(s)^2), so a centre farther
// outside the image than sigma_extent sqrt(bound) (+1% and 2 px slack for
// FP32 rounding) or behind the near plane (with slack) can only be culled.
// Survivors are queued in shared memory. Phase 2 runs the exact FP64 path on
// the queue with every lane busy (rows are in id order, i.e. spatially random,
// so doing this per thread would leave most lanes of a warp idle). The
// visible set and every rect are exactly those of the exact path.
__global__ __launch_bounds__(kPreThreads, 6) void preprocess_kernel(float* __restrict__ x, float* __restrict__ m,
                                                                 float* __restrict__ v, LazyAdam la, uint32_t n,
                                                                 int fd, DevCam cam, DevRender rc,
                                                                 float4* __restrict__ rec,
                                                                 uint64_t* __restrict__ depth_key,
                                                                 uint32_t* __restrict__ tiles,
                                                                 float4* __restrict__ g2d,
                                                                 double* __restrict__ g2d_wide,
                                                                 StepCounters* __restrict__ counters,
                                                                 StepScalars* __restrict__ scalars,
                                                                 uint32_t* __restrict__ tile_cnt,
                                                                 uint32_t* __restrict__ vis_mask, uint32_t mask_words) {
    pdl_prologue();
    __shared__ uint32_t s_rows[kPreChunk];
    __shared__ uint8_t s_stale[kPreChunk];     // Adam steps each queued row is behind (lazy Adam)
    __shared__ uint16_t s_by_stale[kPreChunk];  // queue positions of the stale rows, most stale first
    __shared__ uint32_t s_bin[kAdamRing];
    __shared__ uint32_t s_count, s_nstale;
    __shared__ unsigned long long s_zmin_inv, s_zmax;
    __shared__ uint32_t s_visible;
    __shared__ uint32_t s_vis[kPreChunk / 32];  // this chunk's visibility mask words
    if (threadIdx.x < kPreChunk / 32) s_vis[threadIdx.x] = 0;
    if (threadIdx.x == 0) {
        s_count = 0;
        s_visible = 0;
        s_zmin_inv = 0;
        s_zmax = 0;
    }
    // the step's loss / penalty sums start from zero (accumulated by later kernels)
    if (blockIdx.x == 0 && threadIdx.x < sizeof(StepScalars) / sizeof(double))
        reinterpret_cast<double*>(scalars)[threadIdx.x] = 0.0;
    __syncthreads();
    const uint32_t chunk0 = blockIdx.x * kPreChunk;
    const float fxf = static_cast<float>(cam.fx), fyf = static_cast<float>(cam.fy);
    const float cxf = static_cast<float>(cam.cx), cyf = static_cast<float>(cam.cy);
    float Rf[9], tf[3];
#pragma unroll
    for (int k = 0; k < 9; ++k) Rf[k] = static_cast<float>(cam.R[k]);
#pragma unroll
    for (int k = 0; k < 3; ++k) tf[k] = static_cast<float>(cam.t[k]);
    const float nearf = static_cast<float>(rc.near_plane);
    // all loads of the thread's rows first (one DRAM round trip), then the tests
    // position + log-scale: the first 32-byte sector of the row (two float4)
    const int rs = row_stride(fd);
    for (int sb = 0; sb < kPreSubBatches; ++sb) {
    float pp[kPreRowsPerThread][3], ll[kPreRowsPerThread][3];
    uint32_t stale[kPreRowsPerThread];  // Adam steps the row is behind (lazy Adam)
#pragma unroll
    for (int k = 0; k < kPreRowsPerThread; ++k) {
        const uint32_t i = chunk0 + (sb * kPreRowsPerThread + k) * kPreThreads + threadIdx.x;
        const uint32_t j = i < n ? i : 0;
        const float4* r4 = reinterpret_cast<const float4*>(x + static_cast<size_t>(j) * rs);
        const float4 a = r4[0], b = r4[1];
        pp[k][0] = a.x; pp[k][1] = a.y; pp[k][2] = a.z;
        ll[k][0] = a.w; ll[k][1] = b.x; ll[k][2] = b.y;
        stale[k] = la.t - __float_as_uint(b.w);  // the row's step stamp (slot kMetaSlot)
    }
    // The test is FP32 with explicit FMAs (this file is compiled --fmad=false
    // for the exact FP64 path below) and approximate MUFU reciprocals /
    // exponentials / roots: every bound carries 1% + 2 px of slack, far above
    // their few-ulp errors.
    const float lg_rho = __log2f(la.rho), geo_scale = la.rho / (1.f - la.rho);
    const float sig = static_cast<float>(rc.sigma_extent), dil = static_cast<float>(rc.dilation);
#pragma unroll
    for (int k = 0; k < kPreRowsPerThread; ++k) {
        const uint32_t i = chunk0 + (sb * kPreRowsPerThread + k) * kPreThreads + threadIdx.x;
        if (i >= n) break;
        const float p0 = pp[k][0], p1 = pp[k][1], p2 = pp[k][2];
        const float z = fmaf(Rf[8], p2, fmaf(Rf[7], p1, fmaf(Rf[6], p0, tf[2])));
        const float px = fmaf(Rf[2], p2, fmaf(Rf[1], p1, fmaf(Rf[0], p0, tf[0])));
        const float py = fmaf(Rf[5], p2, fmaf(Rf[4], p1, fmaf(Rf[3], p0, tf[1])));
        // A stale row's current position / log-scale lie within the lazy-Adam
        // drift bound of the stored ones (bsg_internal.cuh, make_lazy_adam):
        // per component dpos / dls, so the camera-space centre within
        // delta = sqrt(3) dpos (R orthonormal).
        float dpos = 0.f, dls = 0.f;
        if (stale[k]) {
            const float geo = geo_scale * (1.f - exp2f_approx(static_cast<float>(stale[k]) * lg_rho)) * 1.01f;
            dpos = la.drift_pos * geo;
            dls = la.drift_ls * geo;
        }
        const float delta = 1.7321f * dpos;
        // FP32 z may differ from FP64 z by ~1e-6 |p|: keep anything that could be past the near plane
        bool cand = z + delta > nearf - 1e-3f * (1.0f + fabsf(p0) + fabsf(p1) + fabsf(p2));
        if (cand && z - delta > 0.5f * nearf) {
            const float iz = rcp_approx(z - delta), iz0 = rcp_approx(z);
            const float fxz = fxf * iz, fyz = fyf * iz;
            const float ax = fabsf(px) + delta, ay = fabsf(py) + delta;
            const float jx = fxz * ax * iz, jy = fyz * ay * iz;
            const float jf2 = fmaf(jy, jy, fmaf(jx, jx, fmaf(fyz, fyz, fxz * fxz)));
            const float lmax = fmaxf(fmaxf(ll[k][0], ll[k][1]), ll[k][2]) + dls;
            const float smax = exp2f_approx(lmax * 1.44269504f) * 1.01f;
            const float rb = fmaf(sig * 1.01f, sqrt_approx(fmaf(jf2 * smax, smax, dil)), 2.0f);
            // |d(f X / Z)| <= f delta (Z + |X|) / (Z (Z - delta)) for a centre moved by <= delta
            const float dz = delta * iz0 * iz * 1.01f;
            const float rx = fmaf(fxf * dz, z + fabsf(px), rb), ry = fmaf(fyf * dz, z + fabsf(py), rb);
            const float mxf = fmaf(fxf * iz0, px, cxf), myf = fmaf(fyf * iz0, py, cyf);
            // (the image bounds converted here, not hoisted out of the loop:
            // nvcc 12.9 dropped this whole test when they were)
            if (mxf + rx < 0.f || mxf - rx > static_cast<float>(cam.W - 1) || myf + ry < 0.f ||
                myf - ry > static_cast<float>(cam.H - 1))
                cand = false;
        }
        if (cand) {
            const uint32_t q = atomicAdd(&s_count, 1u);
            s_rows[q] = i;
            s_stale[q] = static_cast<uint8_t>(stale[k]);
        } else {
            tiles[i] = 0;
        }
    }
    }
    if (threadIdx.x < kAdamRing) s_bin[threadIdx.x] = 0;
    __syncthreads();
    const uint32_t count = s_count;
    // Lazy-Adam catch-up of the stale queued rows, before the projection
    // reads them: one (row, 32-byte sector) per thread, the rows ordered by
    // staleness so that the lanes of a warp replay the same number of steps
    // (in queue order the warp ran as long as its stalest row, most lanes
    // idle), and every warp of the CTA takes part.
    for (uint32_t q = threadIdx.x; q < count; q += kPreThreads)
        if (s_stale[q]) atomicAdd(&s_bin[kAdamRing - 1 - s_stale[q]], 1u);
    __syncthreads();
    if (threadIdx.x < 32) {  // exclusive scan of the 64 bins (most stale first), in place
        const uint32_t a = s_bin[2 * threadIdx.x], b = s_bin[2 * threadIdx.x + 1];
        uint32_t inc = a + b;
#pragma unroll
        for (int o = 1; o < 32; o <<= 1) {
            const uint32_t y = __shfl_up_sync(0xffffffffu, inc, o);
            if (threadIdx.x >= o) inc += y;
        }
        s_bin[2 * threadIdx.x] = inc - a - b;
        s_bin[2 * threadIdx.x + 1] = inc - b;
        if (threadIdx.x == 31) s_nstale = inc;
    }
    __syncthreads();
    for (uint32_t q = threadIdx.x; q < count; q += kPreThreads)
        if (s_stale[q]) s_by_stale[atomicAdd(&s_bin[kAdamRing - 1 - s_stale[q]], 1u)] = static_cast<uint16_t>(q);
    __syncthreads();
    {
        const int H = fd >= 12 ? 3 : 2;
        const uint32_t items = s_nstale * H;
        for (uint32_t it = threadIdx.x; it < items; it += kPreThreads) {
            const uint32_t q = s_by_stale[it / H], h = it % H;
            const uint32_t i = s_rows[q], t0 = la.t - s_stale[q];
            if (fd >= 12) {
                if (h == 0) catch_up_sector_mem<12, 0>(x, m, v, i, t0, la);
                else if (h == 1) catch_up_sector_mem<12, 1>(x, m, v, i, t0, la);
                else catch_up_sector_mem<12, 2>(x, m, v, i, t0, la);
            } else {
                if (h == 0) catch_up_sector_mem<3, 0>(x, m, v, i, t0, la);
                else catch_up_sector_mem<3, 1>(x, m, v, i, t0, la);
            }
        }
    }
    __syncthreads();  // (the caught-up rows are read back below by other threads of the CTA)
    unsigned long long zmin_inv = 0, zmax = 0;  // depth range of this thread's visible splats
    uint32_t nvis = 0;
    for (uint32_t q = threadIdx.x; q < count; q += kPreThreads) {
        const uint32_t i = s_rows[q];
        // the whole row up front (contiguous float4s): one dependent DRAM round trip
        float prm[kMaxD];
        const float4* r4 = reinterpret_cast<const float4*>(x + static_cast<size_t>(i) * rs);
        {
            const float4 a = r4[0], b = r4[1], c2 = r4[2], d = r4[3];
            prm[kPos + 0] = a.x; prm[kPos + 1] = a.y; prm[kPos + 2] = a.z;
            prm[kLs + 0] = a.w; prm[kLs + 1] = b.x; prm[kLs + 2] = b.y;
            prm[kRot + 0] = c2.x; prm[kRot + 1] = c2.y; prm[kRot + 2] = c2.z; prm[kRot + 3] = c2.w;
            prm[kFeat + 0] = d.x; prm[kFeat + 1] = d.y; prm[kFeat + 2] = d.z;
            if (fd >= 12) {
                prm[kFeat + 3] = d.w;
                const float4 e = r4[4], f = r4[5];
                prm[kFeat + 4] = e.x; prm[kFeat + 5] = e.y; prm[kFeat + 6] = e.z; prm[kFeat + 7] = e.w;
                prm[kFeat + 8] = f.x; prm[kFeat + 9] = f.y; prm[kFeat + 10] = f.z; prm[kFeat + 11] = f.w;
                prm[kFeat + 12] = b.z;  // op
            } else {
                prm[kFeat + 3] = b.z;  // op
            }
        }
        const double p0 = prm[kPos + 0], p1 = prm[kPos + 1], p2 = prm[kPos + 2];
        // p_cam = R p + t (camera.hpp:28)
        double pc[3];
#pragma unroll
        for (int r = 0; r < 3; ++r) pc[r] = ((cam.R[3 * r] * p0 + cam.R[3 * r + 1] * p1) + cam.R[3 * r + 2] * p2) + cam.t[r];
        uint32_t ntiles = 0;
        if (pc[2] > rc.near_plane) {
            // Sigma = (R S)(R S)^T, R from the normalized quaternion (cloud.cpp:162-167, math.hpp:25-44)
            double qw = prm[kRot + 0], qx = prm[kRot + 1], qy = prm[kRot + 2], qz = prm[kRot + 3];
            const double qn = sqrt(((qw * qw + qx * qx) + qy * qy) + qz * qz);
            if (qn == 0.0) {
                qw = 1.0; qx = 0.0; qy = 0.0; qz = 0.0;
            } else {
                qw = qw / qn; qx = qx / qn; qy = qy / qn; qz = qz / qn;
            }
            double R[3][3];
            R[0][0] = 1 - 2 * (qy * qy + qz * qz); R[0][1] = 2 * (qx * qy - qw * qz); R[0][2] = 2 * (qx * qz + qw * qy);
            R[1][0] = 2 * (qx * qy + qw * qz); R[1][1] = 1 - 2 * (qx * qx + qz * qz); R[1][2] = 2 * (qy * qz - qw * qx);
            R[2][0] = 2 * (qx * qz - qw * qy); R[2][1] = 2 * (qy * qz + qw * qx); R[2][2] = 1 - 2 * (qx * qx + qy * qy);
            const double s[3] = {exp(static_cast<double>(prm[kLs + 0])), exp(static_cast<double>(prm[kLs + 1])),
                                 exp(static_cast<double>(prm[kLs + 2]))};
            double M[3][3];
#pragma unroll
            for (int a = 0; a < 3; ++a)
#pragma unroll
                for (int b = 0; b < 3; ++b) M[a][b] = R[a][b] * s[b];
            double S[3][3];
#pragma unroll
            for (int a = 0; a < 3; ++a)
#pragma unroll
                for (int b = 0; b < 3; ++b) S[a][b] = (M[a][0] * M[b][0] + M[a][1] * M[b][1]) + M[a][2] * M[b][2];

            // mean2d (camera.hpp:34-36); J (renderer.cpp:14-20); A = J W; cov2d = A S A^T + dilation I
            const double z = pc[2];
            const double mx = cam.fx * pc[0] / z + cam.cx;
            const double my = cam.fy * pc[1] / z + cam.cy;
            const double iz = 1.0 / z, iz2 = iz * iz;
            const double J[2][3] = {{cam.fx * iz, 0.0, -cam.fx * pc[0] * iz2}, {0.0, cam.fy * iz, -cam.fy * pc[1] * iz2}};
            double A[2][3], T[2][3], C[2][2];
#pragma unroll
            for (int r = 0; r < 2; ++r)
#pragma unroll
                for (int k = 0; k < 3; ++k)
                    A[r][k] = (J[r][0] * cam.R[k] + J[r][1] * cam.R[3 + k]) + J[r][2] * cam.R[6 + k];
#pragma unroll
            for (int r = 0; r < 2; ++r)
#pragma unroll
                for (int k = 0; k < 3; ++k) T[r][k] = (A[r][0] * S[0][k] + A[r][1] * S[1][k]) + A[r][2] * S[2][k];
#pragma unroll
            for (int r = 0; r < 2; ++r)
#pragma unroll
                for (int q = 0; q < 2; ++q) {
                    const double v = (T[r][0] * A[q][0] + T[r][1] * A[q][1]) + T[r][2] * A[q][2];
                    C[r][q] = v + (r == q ? rc.dilation : rc.dilation * 0.0);
                }
            // max_eigenvalue_2x2 (renderer.cpp:22-26), footprint (renderer.cpp:33-40)
            const double mid = 0.5 * (C[0][0] + C[1][1]);
            const double det = C[0][0] * C[1][1] - C[0][1] * C[1][0];
            const double lam = mid + sqrt(fmax(0.0, mid * mid - det));
            const double radius = rc.sigma_extent * sqrt(lam);
            const int x0 = max(0, to_int_clamped(ceil(mx - radius)));
            const int x1 = min(cam.W - 1, to_int_clamped(floor(mx + radius)));
            const int y0 = max(0, to_int_clamped(ceil(my - radius)));
            const int y1 = min(cam.H - 1, to_int_clamped(floor(my + radius)));
            if (x0 <= x1 && y0 <= y1) {
                // minv (renderer.cpp:76-78), colour (cloud.cpp:180-193), opacity (cloud.hpp:55).
                // These only reach the FP32 record (no integer depends on them): one
                // reciprocal instead of three FP64 divisions (~1 FP64 ulp apart).
                const double idet = 1.0 / det;
                const double m00 = C[1][1] * idet, m01 = -C[0][1] * idet, m11 = C[0][0] * idet;
                double col[3];
#pragma unroll
                for (int ch = 0; ch < 3; ++ch) col[ch] = kSh0 * static_cast<double>(prm[kFeat + ch]);
                if (fd >= 12) {
                    const double u0 = p0 - cam.center[0], u1 = p1 - cam.center[1], u2 = p2 - cam.center[2];
                    const double un = sqrt((u0 * u0 + u1 * u1) + u2 * u2);
                    const double iun = 1.0 / un;  // (record only, as above)
                    const double d0 = u0 * iun, d1 = u1 * iun, d2 = u2 * iun;
                    const double b0 = -kSh1 * d1, b1 = kSh1 * d2, b2 = -kSh1 * d0;
#pragma unroll
                    for (int ch = 0; ch < 3; ++ch)
                        col[ch] += b0 * static_cast<double>(prm[kFeat + 3 + 3 * ch]) +
                                   b1 * static_cast<double>(prm[kFeat + 4 + 3 * ch]) +
                                   b2 * static_cast<double>(prm[kFeat + 5 + 3 * ch]);
                }
                const double o = 1.0 / (1.0 + exp(-static_cast<double>(fd >= 12 ? prm[kFeat + kMaxFd] : prm[kFeat + 3])));  // op_comp(fd)
                const uint32_t r01 = (static_cast<uint32_t>(x0) & 0xffffu) | (static_cast<uint32_t>(x1) << 16);
                const uint32_t r23 = (static_cast<uint32_t>(y0) & 0xffffu) | (static_cast<uint32_t>(y1) << 16);
                // The blend evaluates q = d^T minv d (d = pixel - mean) as |L d|^2 with
                // minv = L^T L, L = [[l11, l12], [0, l22]], in the affine form
                // L d = L (p - o) + k around o = the rect centre, so no FP32 term is
                // ever large: near-plane splats (depth ~0.01, |mean2d| ~1e6 px,
                // minv ~1e-7) cancel terms of ~1e3 into q ~ 0.1 in the conic form,
                // which FP32 cannot hold; here that cancellation happens once, in
                // FP64 (k). L and k carry sqrt(log2(e) / 2), so the blend's
                // exponent is ex2(-|L d|^2) = exp(-q / 2).
                const double l11 = sqrt(m00), l12 = m01 / l11, l22 = sqrt(fmax(0.0, m11 - l12 * l12));
                const double ox = 0.5 * static_cast<double>(x0 + x1), oy = 0.5 * static_cast<double>(y0 + y1);
                const double k1 = -(l11 * (mx - ox) + l12 * (my - oy)), k2 = -(l22 * (my - oy));
                rec[3 * static_cast<size_t>(i) + 0] =
                    make_float4(static_cast<float>(kQScale * l11), static_cast<float>(kQScale * l12),
                                static_cast<float>(kQScale * l22), static_cast<float>(kQScale * k1));
                rec[3 * static_cast<size_t>(i) + 1] =
                    make_float4(static_cast<float>(kQScale * k2), static_cast<float>(o), static_cast<float>(col[0]), static_cast<float>(col[1]));
                // gradient target: the row, or a wide footprint's FP64 slot (see kWideArea)
                uint32_t wslot = i;
                if (static_cast<uint32_t>(x1 - x0 + 1) * static_cast<uint32_t>(y1 - y0 + 1) >= kWideArea) {
                    const uint32_t w = atomicAdd(&counters->wide, 1u);
                    if (w < kWideCap) {
                        wslot = kWideBit | w;
#pragma unroll
                        for (int k = 0; k < 9; ++k) g2d_wide[9 * static_cast<size_t>(w) + k] = 0.0;
                    }
                }
                rec[3 * static_cast<size_t>(i) + 2] =
                    make_float4(static_cast<float>(col[2]), __uint_as_float(r01), __uint_as_float(r23),
                                __uint_as_float(wslot));
                ntiles = static_cast<uint32_t>((x1 / kTile - x0 / kTile + 1) * (y1 / kTile - y0 / kTile + 1));
                // pairs per tile for the per-tile binning
                for (int ty = y0 / kTile; ty <= y1 / kTile; ++ty)
                    for (int tx = x0 / kTile; tx <= x1 / kTile; ++tx)
                        atomicAdd(&tile_cnt[kTileSub * (ty * cam.tiles_x + tx) + (i & (kTileSub - 1))], 1u);
                const unsigned long long zb = static_cast<unsigned long long>(__double_as_longlong(z));
                depth_key[i] = zb;
                zmin_inv = max(zmin_inv, ~zb);
                zmax = max(zmax, zb);
                ++nvis;
                atomicOr(&s_vis[(i - chunk0) >> 5], 1u << (i & 31u));
                const float4 zero = make_float4(0.f, 0.f, 0.f, 0.f);
                g2d[3 * static_cast<size_t>(i) + 0] = zero;
                g2d[3 * static_cast<size_t>(i) + 1] = zero;
                // (float 9, unused by the accumulators: the gradient target, so the
                // fold reads it with the gradients instead of from the splat record)
                g2d[3 * static_cast<size_t>(i) + 2] = make_float4(0.f, __uint_as_float(wslot), 0.f, 0.f);
            }
        }
        tiles[i] = ntiles;
    }
    // visible depth range (keys the 32-bit depth sort); one atomic pair per CTA
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) {
        zmin_inv = max(zmin_inv, __shfl_xor_sync(0xffffffffu, zmin_inv, o));
        zmax = max(zmax, __shfl_xor_sync(0xffffffffu, zmax, o));
    }
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) nvis += __shfl_xor_sync(0xffffffffu, nvis, o);
    if ((threadIdx.x & 31) == 0 && zmax) {
        atomicMax(&s_zmin_inv, zmin_inv);
        atomicMax(&s_zmax, zmax);
        atomicAdd(&s_visible, nvis);
    }
    __syncthreads();
    // the visibility mask (1 bit per row, the compaction's input on the
    // per-tile path and the Adam's visible-row test): whole words per chunk
    if (threadIdx.x < kPreChunk / 32 && (chunk0 >> 5) + threadIdx.x < mask_words)
        vis_mask[(chunk0 >> 5) + threadIdx.x] = s_vis[threadIdx.x];
    if (threadIdx.x == 0 && s_zmax) {
        atomicMax(&counters->zmin_inv, s_zmin_inv);
        atomicMax(&counters->zmax, s_zmax);
        atomicAdd(&counters->visible_pre, s_visible);
    }
}

}  // namespace

DevCam make_cam(const bsg_camera& c) {
    DevCam d{};
    d.fx = c.fx; d.fy = c.fy; d.cx = c.cx; d.cy = c.cy;
    for (int k = 0; k < 9; ++k) d.R[k] = c.R[k];
    for (int k = 0; k < 3; ++k) d.t[k] = c.t[k];
    // center = -(R^T t), camera.hpp:31, same evaluation order as the oracle
    for (int k = 0; k < 3; ++k) d.center[k] = -((c.R[k] * c.t[0] + c.R[3 + k] * c.t[1]) + c.R[6 + k] * c.t[2]);
    d.W = static_cast<int>(c.width);
    d.H = static_cast<int>(c.height);
    d.tiles_x = (d.W + kTile - 1) / kTile;
    d.tiles_y = (d.H + kTile - 1) / kTile;
    return d;
}

DevRender make_render(const bsg_render_config& r) {
    DevRender d{};
    d.near_plane = r.near_plane;
    d.dilation = r.dilation;
    d.alpha_clamp = r.alpha_clamp;
    d.tstop = r.transmittance_stop;
    d.sigma_extent = r.sigma_extent;
    for (int k = 0; k < 3; ++k) d.bg[k] = static_cast<float>(r.background[k]);
    d.lambda = r.lambda;
    return d;
}

void launch_preprocess(Ctx* c, const DevCam& cam, const DevRender& rc) {
    if (c->n == 0) {
        BSG_CUDA(cudaMemsetAsync(c->scalars, 0, sizeof(StepScalars), c->stream));
        return;
    }
    const uint32_t blocks = static_cast<uint32_t>((c->n + kPreChunk - 1) / kPreChunk);
    const LazyAdam la = make_lazy_adam(c);
    launch_pdl(c->stream, blocks, kPreThreads, 0, preprocess_kernel, c->x, c->m, c->v, la, static_cast<uint32_t>(c->n), c->fd, cam, rc, c->rec,
                                                      c->depth_key, c->tiles, c->g2d, c->g2d_wide, c->counters,
                                                      c->scalars, c->tile_cnt, c->vis_mask,
                                                      static_cast<uint32_t>(c->cap / 32));
    BSG_LAUNCHED(c);
}

}  // namespace bsg
