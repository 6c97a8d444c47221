// K9 fold + K10 Adam. The fold of the image-space splat gradients to the
// parameters (renderer.cpp:313-403) runs once per VISIBLE splat over the
// compacted list (FP64 arithmetic, ~1.5k flops) and writes the parameter
// gradient rows it touched; the dense Adam (trainer.cpp:120-131,267-281) with
// the consensus penalty (admm.cpp:11-45, trainer.cpp:257-265) and quaternion
// canonicalisation (cloud.cpp:82-85) then streams every row once. Keeping the
// FP64 fold out of the dense kernel keeps the dense kernel a pure HBM stream:
// per row it reads x, m, v (3 x 4D bytes) and the visible flag, and writes
// x, m, v back; visible rows add a 4D-byte gradient read, shared rows z and u.
#include "bsg_internal.cuh"

#include <algorithm>
#include <cmath>

namespace bsg {
namespace {

// Fold of one visible row; FP64 arithmetic over FP32 inputs. g receives the
// D parameter gradients; returns the screen-space gradient norm.
// The row's parameters in component order, from its row-major x (current:
// the preprocess caught every visible row up and nothing writes x before the
// Adam): whole aligned sectors, 64 bytes at SH degree 0.
template <int fd>
__device__ __forceinline__ void load_row(const float* __restrict__ x, uint32_t i, float (&prm)[11 + fd]) {
    constexpr int D = 11 + fd, NS = fd <= 4 ? 16 : 24;  // slots in use
    const float4* r4 = reinterpret_cast<const float4*>(x + static_cast<size_t>(i) * row_stride(fd));
    float v[NS];
#pragma unroll
    for (int k = 0; k < NS / 4; ++k) {
        const float4 q = r4[k];
        v[4 * k] = q.x; v[4 * k + 1] = q.y; v[4 * k + 2] = q.z; v[4 * k + 3] = q.w;
    }
#pragma unroll
    for (int c = 0; c < D; ++c) prm[c] = v[pslot(c, fd)];
}

// The 9 image-space gradients of row i: FP32 record, or the FP64 slot of a
// wide splat (the gradient target -- rec[3i+2].w -- is also in float 9 of the
// record, see kWideArea). The blend backward
// accumulates the mean path as sum k L'^T L' d and the covariance path as
// sum k (L'^T L' d)(L'^T L' d)^T with the scaled factor L' = kQScale L and
// without the 1/2 (renderer.cpp:298-306); both are rescaled here.
struct Grad2D {
    double v[9];
};
__device__ __forceinline__ void unscale_g2d(Grad2D& g) {
    constexpr double kMean = 1.0 / kQScale2, kCov = 0.5 / (kQScale2 * kQScale2);
    g.v[0] *= kMean;
    g.v[1] *= kMean;
    g.v[2] *= kCov;
    g.v[3] *= kCov;
    g.v[4] *= kCov;
}
__device__ __forceinline__ Grad2D load_g2d(uint32_t i, const float4* __restrict__ rec,
                                           const float4* __restrict__ g2d, const double* __restrict__ g2d_wide) {
    (void)rec;
    Grad2D g;
    const float4 ga = g2d[3 * static_cast<size_t>(i)], gb = g2d[3 * static_cast<size_t>(i) + 1],
                 gc = g2d[3 * static_cast<size_t>(i) + 2];
    const uint32_t target = __float_as_uint(gc.y);  // (written there by the preprocess, preprocess.cu)
    if (target & kWideBit) {
        const uint32_t wslot = target & ~kWideBit;
#pragma unroll
        for (int k = 0; k < 9; ++k) g.v[k] = g2d_wide[9 * static_cast<size_t>(wslot) + k];
    } else {
        g.v[0] = ga.x; g.v[1] = ga.y; g.v[2] = ga.z; g.v[3] = ga.w;
        g.v[4] = gb.x; g.v[5] = gb.y; g.v[6] = gb.z; g.v[7] = gb.w; g.v[8] = gc.x;
    }
    unscale_g2d(g);
    return g;
}

template <int fd>
__device__ __forceinline__ double fold_row(const float (&prm)[11 + fd], const Grad2D& g2, const DevCam& cam,
                                           double* g) {
    const double gm0 = g2.v[0], gm1 = g2.v[1];
    const double gcov[2][2] = {{g2.v[2], g2.v[3]}, {g2.v[3], g2.v[4]}};
    const double gcol[3] = {g2.v[5], g2.v[6], g2.v[7]};
    const double gop = g2.v[8];

    const double pos[3] = {prm[kPos + 0], prm[kPos + 1], prm[kPos + 2]};
    double pc[3];
#pragma unroll
    for (int r = 0; r < 3; ++r) pc[r] = ((cam.R[3 * r] * pos[0] + cam.R[3 * r + 1] * pos[1]) + cam.R[3 * r + 2] * pos[2]) + cam.t[r];
    const double z = pc[2], iz = 1.0 / z, iz2 = iz * iz, iz3 = iz2 * iz;

    // opacity logit (renderer.cpp:325-327)
    const double ol = prm[kFeat + fd];  // op_comp(fd)
    const double o = 1.0 / (1.0 + exp(-ol));
    g[op_comp(fd)] = gop * o * (1.0 - o);

    // features (renderer.cpp:329-352)
#pragma unroll
    for (int ch = 0; ch < 3; ++ch) g[kFeat + ch] = kSh0 * gcol[ch];
    double gpd[3] = {0, 0, 0};
    if constexpr (fd >= 12) {
        const double u0 = pos[0] - cam.center[0], u1 = pos[1] - cam.center[1], u2 = pos[2] - cam.center[2];
        const double un = sqrt(u0 * u0 + u1 * u1 + u2 * u2);
        const double dir[3] = {u0 / un, u1 / un, u2 / un};
        const double b0 = -kSh1 * dir[1], b1 = kSh1 * dir[2], b2 = -kSh1 * dir[0];
        double gd[3] = {0, 0, 0};
#pragma unroll
        for (int ch = 0; ch < 3; ++ch) {
            g[kFeat + 3 + 3 * ch] = b0 * gcol[ch];
            g[kFeat + 4 + 3 * ch] = b1 * gcol[ch];
            g[kFeat + 5 + 3 * ch] = b2 * gcol[ch];
            const double f3 = prm[kFeat + 3 + 3 * ch], f4 = prm[kFeat + 4 + 3 * ch], f5 = prm[kFeat + 5 + 3 * ch];
            gd[0] += gcol[ch] * (f5 * -kSh1);
            gd[1] += gcol[ch] * (f3 * -kSh1);
            gd[2] += gcol[ch] * (f4 * kSh1);
        }
        const double dd = dir[0] * gd[0] + dir[1] * gd[1] + dir[2] * gd[2];
#pragma unroll
        for (int k = 0; k < 3; ++k) gpd[k] = (gd[k] - dir[k] * dd) / un;
    }

    // screen-space norm (renderer.cpp:356-358)
    const double sx = gm0 * cam.W * 0.5, sy = gm1 * cam.H * 0.5;
    const double sgn = sqrt(sx * sx + sy * sy);

    // mean path (renderer.cpp:360-362)
    double gpc[3] = {gm0 * cam.fx * iz, gm1 * cam.fy * iz, -gm0 * cam.fx * pc[0] * iz2 - gm1 * cam.fy * pc[1] * iz2};

    // covariance path (renderer.cpp:364-378)
    const double J[2][3] = {{cam.fx * iz, 0.0, -cam.fx * pc[0] * iz2}, {0.0, cam.fy * iz, -cam.fy * pc[1] * iz2}};
    double A[2][3];
#pragma unroll
    for (int r = 0; r < 2; ++r)
#pragma unroll
        for (int k = 0; k < 3; ++k) A[r][k] = J[r][0] * cam.R[k] + J[r][1] * cam.R[3 + k] + J[r][2] * cam.R[6 + k];

    double qw = prm[kRot + 0], qx = prm[kRot + 1], qy = prm[kRot + 2], qz = prm[kRot + 3];
    const double qn = sqrt(qw * qw + qx * qx + qy * qy + qz * qz);
    double hw, hx, hy, hz;
    if (qn == 0.0) {
        hw = 1; hx = 0; hy = 0; hz = 0;
    } else {
        hw = qw / qn; hx = qx / qn; hy = qy / qn; hz = qz / qn;
    }
    double R[3][3];
    R[0][0] = 1 - 2 * (hy * hy + hz * hz); R[0][1] = 2 * (hx * hy - hw * hz); R[0][2] = 2 * (hx * hz + hw * hy);
    R[1][0] = 2 * (hx * hy + hw * hz); R[1][1] = 1 - 2 * (hx * hx + hz * hz); R[1][2] = 2 * (hy * hz - hw * hx);
    R[2][0] = 2 * (hx * hz - hw * hy); R[2][1] = 2 * (hy * hz + hw * hx); R[2][2] = 1 - 2 * (hx * hx + hy * hy);
    const double sc[3] = {exp(static_cast<double>(prm[kLs + 0])), exp(static_cast<double>(prm[kLs + 1])),
                          exp(static_cast<double>(prm[kLs + 2]))};
    double M[3][3], S[3][3];
#pragma unroll
    for (int a = 0; a < 3; ++a)
#pragma unroll
        for (int b = 0; b < 3; ++b) M[a][b] = R[a][b] * sc[b];
#pragma unroll
    for (int a = 0; a < 3; ++a)
#pragma unroll
        for (int b = 0; b < 3; ++b) S[a][b] = M[a][0] * M[b][0] + M[a][1] * M[b][1] + M[a][2] * M[b][2];

    // g_sigma = A^T gcov A ; g_a = 2 gcov A S ; g_j = g_a W^T
    double atg[3][2], gS[3][3], ga0[2][3], gA[2][3], gJ[2][3];
#pragma unroll
    for (int r = 0; r < 3; ++r)
#pragma unroll
        for (int s = 0; s < 2; ++s) atg[r][s] = A[0][r] * gcov[0][s] + A[1][r] * gcov[1][s];
#pragma unroll
    for (int r = 0; r < 3; ++r)
#pragma unroll
        for (int k = 0; k < 3; ++k) gS[r][k] = atg[r][0] * A[0][k] + atg[r][1] * A[1][k];
#pragma unroll
    for (int r = 0; r < 2; ++r)
#pragma unroll
        for (int k = 0; k < 3; ++k) ga0[r][k] = 2.0 * (gcov[r][0] * A[0][k] + gcov[r][1] * A[1][k]);
#pragma unroll
    for (int r = 0; r < 2; ++r)
#pragma unroll
        for (int k = 0; k < 3; ++k) gA[r][k] = ga0[r][0] * S[0][k] + ga0[r][1] * S[1][k] + ga0[r][2] * S[2][k];
#pragma unroll
    for (int r = 0; r < 2; ++r)
#pragma unroll
        for (int k = 0; k < 3; ++k) gJ[r][k] = gA[r][0] * cam.R[3 * k] + gA[r][1] * cam.R[3 * k + 1] + gA[r][2] * cam.R[3 * k + 2];
    gpc[0] += gJ[0][2] * (-cam.fx * iz2);
    gpc[1] += gJ[1][2] * (-cam.fy * iz2);
    gpc[2] += gJ[0][0] * (-cam.fx * iz2) + gJ[1][1] * (-cam.fy * iz2) + gJ[0][2] * (2.0 * cam.fx * pc[0] * iz3) +
              gJ[1][2] * (2.0 * cam.fy * pc[1] * iz3);
#pragma unroll
    for (int k = 0; k < 3; ++k)
        g[kPos + k] = cam.R[k] * gpc[0] + cam.R[3 + k] * gpc[1] + cam.R[6 + k] * gpc[2] + gpd[k];

    // log-scale and quaternion (renderer.cpp:383-402)
    double gM[3][3], gR[3][3];
#pragma unroll
    for (int a = 0; a < 3; ++a)
#pragma unroll
        for (int b = 0; b < 3; ++b) gM[a][b] = 2.0 * (gS[a][0] * M[0][b] + gS[a][1] * M[1][b] + gS[a][2] * M[2][b]);
#pragma unroll
    for (int a = 0; a < 3; ++a)
#pragma unroll
        for (int b = 0; b < 3; ++b) gR[a][b] = gM[a][b] * sc[b];
#pragma unroll
    for (int k = 0; k < 3; ++k) g[kLs + k] = (R[0][k] * gM[0][k] + R[1][k] * gM[1][k] + R[2][k] * gM[2][k]) * sc[k];
    // dR/dq_hat (renderer.cpp:198-213), contracted with gR
    const double gq0 = 2.0 * (gR[0][1] * -hz + gR[0][2] * hy + gR[1][0] * hz + gR[1][2] * -hx + gR[2][0] * -hy + gR[2][1] * hx);
    const double gq1 = 2.0 * (gR[0][1] * hy + gR[0][2] * hz + gR[1][0] * hy + gR[1][1] * (-2 * hx) + gR[1][2] * -hw +
                              gR[2][0] * hz + gR[2][1] * hw + gR[2][2] * (-2 * hx));
    const double gq2 = 2.0 * (gR[0][0] * (-2 * hy) + gR[0][1] * hx + gR[0][2] * hw + gR[1][0] * hx + gR[1][2] * hz +
                              gR[2][0] * -hw + gR[2][1] * hz + gR[2][2] * (-2 * hy));
    const double gq3 = 2.0 * (gR[0][0] * (-2 * hz) + gR[0][1] * -hw + gR[0][2] * hx + gR[1][0] * hw + gR[1][1] * (-2 * hz) +
                              gR[1][2] * hy + gR[2][0] * hx + gR[2][1] * hy);
    const double qdot = hw * gq0 + hx * gq1 + hy * gq2 + hz * gq3;
    const double inv_qn = qn == 0.0 ? 0.0 : 1.0 / qn;
    g[kRot + 0] = (gq0 - hw * qdot) * inv_qn;
    g[kRot + 1] = (gq1 - hx * qdot) * inv_qn;
    g[kRot + 2] = (gq2 - hy * qdot) * inv_qn;
    g[kRot + 3] = (gq3 - hz * qdot) * inv_qn;
    return sgn;
}

template <int fd>
__global__ __launch_bounds__(256) void fold_grads_kernel(const float* __restrict__ x, size_t cap, uint32_t n,
                                                         DevCam cam, const uint32_t* __restrict__ tiles,
                                                         const float4* __restrict__ rec,
                                                         const float4* __restrict__ g2d,
                                                         const double* __restrict__ g2d_wide, double* __restrict__ gout,
                                                         double* __restrict__ sgn_out, uint8_t* __restrict__ vis) {
    pdl_prologue();
    const uint32_t i = blockIdx.x * blockDim.x + threadIdx.x;
    if (i >= n) return;
    constexpr int D = 11 + fd;
    double g[D];
#pragma unroll
    for (int c = 0; c < D; ++c) g[c] = 0.0;
    double s = 0.0;
    const bool visible = tiles[i] > 0;
    if (visible) {
        float prm[11 + fd];
        load_row<fd>(x, i, prm);
        s = fold_row<fd>(prm, load_g2d(i, rec, g2d, g2d_wide), cam, g);
    }
#pragma unroll
    for (int c = 0; c < D; ++c) gout[static_cast<size_t>(c) * n + i] = g[c];
    sgn_out[i] = s;
    vis[i] = visible ? 1 : 0;
}

// The Adam step (trainer.cpp:267-281) of one row, a sector at a time. The
// parameters and both moments are row-major (row_stride(fd) floats per row,
// bsg_internal.cuh): a sector is 8 slots of x, m and v, two float4 each. The
// rotation sector (slots 8-11) is canonicalised (cloud.cpp:82-85,
// math.hpp:25-34) after its step; shared rows add rho (x - z + u) evaluated at
// the pre-step x (admm.cpp:24-28, trainer.cpp:257-265), their anchor found
// through the shared-row bit mask + per-word prefix. The step itself is
// adam_update_step (bsg_internal.cuh), shared with the lazy replays.
__device__ __forceinline__ float adam_update(float x, float g, float& m, float& v, float lr, const AdamStep& st) {
    return adam_update_step(x, g, m, v, lr, st.b1, st.omb1, st.b2, st.omb2, st.inv_bc1, st.inv_bc2, st.eps);
}

template <int fd, int h>
__device__ __forceinline__ double adam_sector_core(float* __restrict__ x, float* __restrict__ m,
                                                   float* __restrict__ v, uint32_t i, float (&xs)[8], float (&ms)[8],
                                                   float (&vs)[8], float (&g)[8], bool visible, float sgn, int aj,
                                                   const float* __restrict__ z, const float* __restrict__ u, size_t ns,
                                                   const float* __restrict__ rho_dev, const AdamStep& st);

// The rest of a sector's step, its render gradient g given: penalty, Adam,
// canonicalisation, step stamp and densify statistics, stores.
template <int fd, int h>
__device__ __forceinline__ double adam_sector_core(float* __restrict__ x, float* __restrict__ m,
                                                   float* __restrict__ v, uint32_t i, float (&xs)[8], float (&ms)[8],
                                                   float (&vs)[8], float (&g)[8], bool visible, float sgn, int aj,
                                                   const float* __restrict__ z, const float* __restrict__ u, size_t ns,
                                                   const float* __restrict__ rho_dev, const AdamStep& st) {
    constexpr int RS = row_stride(fd);
    const size_t off = static_cast<size_t>(i) * RS + 8 * h;
    double pen = 0.0;
    if (aj >= 0) {
        float zr[8], ur[8];
#pragma unroll
        for (int j = 0; j < 8; ++j) {
            const int c = comp_of_slot(8 * h + j, fd);
            zr[j] = c >= 0 ? z[static_cast<size_t>(c) * ns + aj] : 0.f;
            ur[j] = c >= 0 ? u[static_cast<size_t>(c) * ns + aj] : 0.f;
        }
#pragma unroll
        for (int j = 0; j < 8; ++j) {
            const int c = comp_of_slot(8 * h + j, fd);
            if (c < 0) continue;
            const float rho = rho_dev[c];
            const float d = xs[j] - zr[j] + ur[j];
            pen += 0.5 * static_cast<double>(rho) * static_cast<double>(d) * static_cast<double>(d);
            g[j] += rho * d;
        }
    }
#pragma unroll
    for (int j = 0; j < 8; ++j) {
        const int c = comp_of_slot(8 * h + j, fd);
        if (c >= 0) xs[j] = adam_update(xs[j], g[j], ms[j], vs[j], st.lr[c], st);
    }
    if (h == 1) canonicalize(xs[0], xs[1], xs[2], xs[3]);  // slots 8-11: the rotation
    if (h == 0) {  // row metadata (bsg_internal.cuh): step stamp; densify statistics (trainer.cpp:284-289)
        xs[kMetaSlot] = __uint_as_float(st.t);
        if (visible) {
            ms[kMetaSlot] += sgn;
            vs[kMetaSlot] = __uint_as_float(__float_as_uint(vs[kMetaSlot]) + 1u);
        }
    }
    float4* x4 = reinterpret_cast<float4*>(x + off);
    float4* m4 = reinterpret_cast<float4*>(m + off);
    float4* v4 = reinterpret_cast<float4*>(v + off);
    x4[0] = make_float4(xs[0], xs[1], xs[2], xs[3]);
    x4[1] = make_float4(xs[4], xs[5], xs[6], xs[7]);
    m4[0] = make_float4(ms[0], ms[1], ms[2], ms[3]);
    m4[1] = make_float4(ms[4], ms[5], ms[6], ms[7]);
    v4[0] = make_float4(vs[0], vs[1], vs[2], vs[3]);
    v4[1] = make_float4(vs[4], vs[5], vs[6], vs[7]);
    return pen;
}

// Fold + Adam of the visible rows in one pass (thread = visible row): the
// FP64 fold of fold_visible_kernel, then each sector's step with the
// gradient still in registers (no [D][V] gradient buffer round trip, the
// row's parameters read once). Anchored rows that are not visible: the
// sparse kernel. The first thread files the step's constants in the ring.
template <int fd>
__global__ __launch_bounds__(128) void fold_adam_kernel(float* __restrict__ x, float* __restrict__ m,
                                                        float* __restrict__ v, DevCam cam,
                                                        const uint32_t* __restrict__ vis_rows, uint32_t V,
                                                        const float4* __restrict__ rec,
                                                        const float4* __restrict__ g2d,
                                                        const double* __restrict__ g2d_wide,
                                                        const uint32_t* __restrict__ sh_mask,
                                                        const uint32_t* __restrict__ sh_prefix,
                                                        const float* __restrict__ z, const float* __restrict__ u,
                                                        size_t ns, const float* __restrict__ rho_dev, AdamStep st,
                                                        float4* __restrict__ ring, double* __restrict__ penalty) {
    pdl_prologue();
    __shared__ double s_red[4];
    constexpr int D = 11 + fd, H = fd <= 4 ? 2 : 3, RS = row_stride(fd);
    const uint32_t p = blockIdx.x * blockDim.x + threadIdx.x;
    if (p == 0) ring[st.t % kAdamRing] = make_float4(st.inv_bc1, st.inv_bc2, st.lr[kPos], 0.f);
    double pen = 0.0;
    if (p < V) {
        const uint32_t i = vis_rows[p];
        float gf[D], sgn;
        {
            double g[D];
#pragma unroll
            for (int c = 0; c < D; ++c) g[c] = 0.0;
            float prm[D];
            load_row<fd>(x, i, prm);
            sgn = static_cast<float>(fold_row<fd>(prm, load_g2d(i, rec, g2d, g2d_wide), cam, g));
#pragma unroll
            for (int c = 0; c < D; ++c) gf[c] = static_cast<float>(g[c]);
        }
        int aj = -1;
        if (st.has_anchor) {
            const uint32_t word = i >> 5, bit = i & 31u, sm = sh_mask[word];
            if ((sm >> bit) & 1u) aj = static_cast<int>(sh_prefix[word] + __popc(sm & ((1u << bit) - 1u)));
            BSG_DASSERT(aj < static_cast<int>(ns));
        }
#pragma unroll
        for (int h = 0; h < H; ++h) {
            const size_t off = static_cast<size_t>(i) * RS + 8 * h;
            float xs[8], ms[8], vs[8], gs[8];
            const float4* x4 = reinterpret_cast<const float4*>(x + off);
            const float4* m4 = reinterpret_cast<const float4*>(m + off);
            const float4* v4 = reinterpret_cast<const float4*>(v + off);
            const float4 xa = x4[0], xb = x4[1], ma = m4[0], mb = m4[1], va = v4[0], vb = v4[1];
            xs[0] = xa.x; xs[1] = xa.y; xs[2] = xa.z; xs[3] = xa.w; xs[4] = xb.x; xs[5] = xb.y; xs[6] = xb.z; xs[7] = xb.w;
            ms[0] = ma.x; ms[1] = ma.y; ms[2] = ma.z; ms[3] = ma.w; ms[4] = mb.x; ms[5] = mb.y; ms[6] = mb.z; ms[7] = mb.w;
            vs[0] = va.x; vs[1] = va.y; vs[2] = va.z; vs[3] = va.w; vs[4] = vb.x; vs[5] = vb.y; vs[6] = vb.z; vs[7] = vb.w;
#pragma unroll
            for (int j = 0; j < 8; ++j) {
                const int c = comp_of_slot(8 * h + j, fd);
                gs[j] = c >= 0 ? gf[c < 0 ? 0 : c] : 0.f;
            }
            if (h == 0)
                pen += adam_sector_core<fd, 0>(x, m, v, i, xs, ms, vs, gs, true, sgn, aj, z, u, ns, rho_dev, st);
            else if (h == 1)
                pen += adam_sector_core<fd, 1>(x, m, v, i, xs, ms, vs, gs, true, sgn, aj, z, u, ns, rho_dev, st);
            else if constexpr (H > 2)
                pen += adam_sector_core<fd, 2>(x, m, v, i, xs, ms, vs, gs, true, sgn, aj, z, u, ns, rho_dev, st);
        }
    }
    if (st.has_anchor) {
#pragma unroll
        for (int o = 16; o > 0; o >>= 1) pen += __shfl_xor_sync(0xffffffffu, pen, o);
        if ((threadIdx.x & 31) == 0) s_red[threadIdx.x >> 5] = pen;
        __syncthreads();
        if (threadIdx.x == 0) {
            const double tt = (s_red[0] + s_red[1]) + (s_red[2] + s_red[3]);
            if (tt != 0.0) atomicAdd(penalty, tt);
        }
    }
}

// Sparse Adam of the anchored rows that are not visible (penalty gradient
// rho (x - z + u) only; the visible rows' steps run in fold_adam_kernel).
// Thread = one sector of one such row; the row's step stamp becomes the
// step's count. The first thread also files the step's constants in the ring
// (the kernel always runs, at least one CTA).
template <int fd>
__global__ __launch_bounds__(256, 4) void adam_sparse_kernel(float* __restrict__ x, float* __restrict__ m,
                                                          float* __restrict__ v,
                                                          const uint32_t* __restrict__ sh_rows, uint32_t n_sh,
                                                          const uint32_t* __restrict__ vis_mask,
                                                          const uint32_t* __restrict__ sh_mask,
                                                          const uint32_t* __restrict__ sh_prefix,
                                                          const float* __restrict__ z, const float* __restrict__ u,
                                                          size_t ns, const float* __restrict__ rho_dev, AdamStep st,
                                                          float4* __restrict__ ring, double* __restrict__ penalty) {
    pdl_prologue();
    __shared__ double s_red[8];
    constexpr int H = fd <= 4 ? 2 : 3, RS = row_stride(fd);
    const size_t t = static_cast<size_t>(blockIdx.x) * blockDim.x + threadIdx.x;
    if (t == 0) ring[st.t % kAdamRing] = make_float4(st.inv_bc1, st.inv_bc2, st.lr[kPos], 0.f);
    const size_t idx = t / H;
    const int h = static_cast<int>(t % H);
    double pen = 0.0;
    uint32_t i = 0;
    bool live = false;
    if (idx < n_sh && st.has_anchor) {
        i = sh_rows[idx];
        live = !((vis_mask[i >> 5] >> (i & 31u)) & 1u);  // visible anchored rows: fold_adam_kernel
    }
    if (live) {
        const uint32_t word = i >> 5, bit = i & 31u, sm = sh_mask[word];
        const int aj = ((sm >> bit) & 1u) ? static_cast<int>(sh_prefix[word] + __popc(sm & ((1u << bit) - 1u))) : -1;
        BSG_DASSERT(aj < static_cast<int>(ns));
        const size_t off = static_cast<size_t>(i) * RS + 8 * h;
        float xs[8], ms[8], vs[8], g[8] = {0.f, 0.f, 0.f, 0.f, 0.f, 0.f, 0.f, 0.f};
        const float4* x4 = reinterpret_cast<const float4*>(x + off);
        const float4* m4 = reinterpret_cast<const float4*>(m + off);
        const float4* v4 = reinterpret_cast<const float4*>(v + off);
        const float4 xa = x4[0], xb = x4[1], ma = m4[0], mb = m4[1], va = v4[0], vb = v4[1];
        xs[0] = xa.x; xs[1] = xa.y; xs[2] = xa.z; xs[3] = xa.w; xs[4] = xb.x; xs[5] = xb.y; xs[6] = xb.z; xs[7] = xb.w;
        ms[0] = ma.x; ms[1] = ma.y; ms[2] = ma.z; ms[3] = ma.w; ms[4] = mb.x; ms[5] = mb.y; ms[6] = mb.z; ms[7] = mb.w;
        vs[0] = va.x; vs[1] = va.y; vs[2] = va.z; vs[3] = va.w; vs[4] = vb.x; vs[5] = vb.y; vs[6] = vb.z; vs[7] = vb.w;
        if (h == 0)
            pen = adam_sector_core<fd, 0>(x, m, v, i, xs, ms, vs, g, false, 0.f, aj, z, u, ns, rho_dev, st);
        else if (h == 1)
            pen = adam_sector_core<fd, 1>(x, m, v, i, xs, ms, vs, g, false, 0.f, aj, z, u, ns, rho_dev, st);
        else if constexpr (H > 2)
            pen = adam_sector_core<fd, 2>(x, m, v, i, xs, ms, vs, g, false, 0.f, aj, z, u, ns, rho_dev, st);
    }
    if (st.has_anchor) {
#pragma unroll
        for (int o = 16; o > 0; o >>= 1) pen += __shfl_xor_sync(0xffffffffu, pen, o);
        if ((threadIdx.x & 31) == 0) s_red[threadIdx.x >> 5] = pen;
        __syncthreads();
        if (threadIdx.x == 0) {
            double tt = 0;
            for (int w = 0; w < 8; ++w) tt += s_red[w];
            if (tt != 0.0) atomicAdd(penalty, tt);
        }
    }
}

// Every stale row caught up to la.t (one thread per row, sector by sector).
template <int fd>
__global__ __launch_bounds__(256) void materialize_kernel(float* __restrict__ x, float* __restrict__ m,
                                                          float* __restrict__ v, uint32_t n, LazyAdam la) {
    const uint32_t i = blockIdx.x * blockDim.x + threadIdx.x;
    if (i >= n) return;
    const uint32_t t0 = __float_as_uint(x[static_cast<size_t>(i) * row_stride(fd) + kMetaSlot]);
    if (t0 >= la.t) return;
    BSG_DASSERT(la.t - t0 <= kAdamRing);
    catch_up_row<fd>(x, m, v, i, t0, la);  // (writes the new stamp)
}

__global__ void reset_row_meta_kernel(float* __restrict__ x, float* __restrict__ m, float* __restrict__ v, size_t cap,
                                      int rs, uint32_t stamp, int reset_stats) {
    for (size_t i = blockIdx.x * static_cast<size_t>(blockDim.x) + threadIdx.x; i < cap;
         i += static_cast<size_t>(gridDim.x) * blockDim.x) {
        x[i * rs + kMetaSlot] = __uint_as_float(stamp);
        if (reset_stats) {
            m[i * rs + kMetaSlot] = 0.f;
            v[i * rs + kMetaSlot] = 0.f;
        }
    }
}

}  // namespace

void launch_fold_grads(Ctx* c, const DevCam& cam, double* g_out, double* sgn, uint8_t* vis) {
    if (c->n == 0) return;
    const uint32_t blocks = static_cast<uint32_t>((c->n + 255) / 256);
    if (c->fd == 3)
        launch_pdl(c->stream, blocks, 256, 0, fold_grads_kernel<3>, c->x, c->cap, static_cast<uint32_t>(c->n), cam, c->tiles,
                                                            c->rec, c->g2d, c->g2d_wide, g_out, sgn, vis);
    else
        launch_pdl(c->stream, blocks, 256, 0, fold_grads_kernel<12>, c->x, c->cap, static_cast<uint32_t>(c->n), cam, c->tiles,
                                                             c->rec, c->g2d, c->g2d_wide, g_out, sgn, vis);
    BSG_LAUNCHED(c);
}

void launch_adam(Ctx* c, const DevCam& cam, const AdamStep& st, double* loss_out, int step_index) {
    (void)loss_out;
    (void)step_index;
    if (c->n == 0) return;
    const uint32_t Vf = c->last_counters.visible;
    if (Vf) {
        if (c->fd == 3)
            launch_pdl(PdlAlways{}, c->stream, (Vf + 127) / 128, 128, 0, fold_adam_kernel<3>, c->x, c->m, c->v, cam,
                       c->vis_rows, Vf, c->rec, c->g2d, c->g2d_wide, c->sh_mask, c->sh_prefix, c->z, c->u,
                       c->n_shared, c->rho_dev, st, c->adam_ring, &c->scalars->penalty);
        else
            launch_pdl(PdlAlways{}, c->stream, (Vf + 127) / 128, 128, 0, fold_adam_kernel<12>, c->x, c->m, c->v, cam,
                       c->vis_rows, Vf, c->rec, c->g2d, c->g2d_wide, c->sh_mask, c->sh_prefix, c->z, c->u,
                       c->n_shared, c->rho_dev, st, c->adam_ring, &c->scalars->penalty);
        BSG_LAUNCHED(c);
    }
    const uint32_t n_sh = st.has_anchor ? static_cast<uint32_t>(c->n_shared) : 0u;
    const size_t threads = static_cast<size_t>(n_sh) * (c->fd <= 4 ? 2 : 3);
    const uint32_t grid = static_cast<uint32_t>(std::max<size_t>(1, (threads + 255) / 256));
    if (n_sh == 0 && Vf > 0) {  // (the fused kernel filed the ring entry)
        if (st.t % c->adam_sync == 0) materialize(c);
        return;
    }
    if (c->fd == 3)
        launch_pdl(PdlAlways{}, c->stream, grid, 256, 0, adam_sparse_kernel<3>, c->x, c->m, c->v, c->sh_rows, n_sh,
                   c->vis_mask, c->sh_mask, c->sh_prefix, c->z, c->u, c->n_shared, c->rho_dev, st, c->adam_ring,
                   &c->scalars->penalty);
    else
        launch_pdl(PdlAlways{}, c->stream, grid, 256, 0, adam_sparse_kernel<12>, c->x, c->m, c->v, c->sh_rows, n_sh,
                   c->vis_mask, c->sh_mask, c->sh_prefix, c->z, c->u, c->n_shared, c->rho_dev, st, c->adam_ring,
                   &c->scalars->penalty);
    BSG_LAUNCHED(c);
    // every adam_sync (<= kAdamRing / 2) steps all rows catch up: a stale row
    // never needs a step the ring no longer holds
    if (st.t % c->adam_sync == 0) materialize(c);
}

LazyAdam make_lazy_adam(const Ctx* c) {
    LazyAdam la{};
    const bsg_trainer_config& t = c->tcfg;
    la.b1 = static_cast<float>(t.beta1);
    la.b2 = static_cast<float>(t.beta2);
    la.omb1 = static_cast<float>(1.0 - t.beta1);
    la.omb2 = static_cast<float>(1.0 - t.beta2);
    la.eps = static_cast<float>(t.eps);
    for (int k = 0; k < c->D; ++k) {
        double lr = t.lr_features;
        if (k < kRot) lr = t.lr_position;  // (the ring carries the decayed rate per step)
        else if (k < kLs) lr = t.lr_rotation;
        else if (k < kFeat) lr = t.lr_log_scale;
        else if (k == op_comp(c->fd)) lr = t.lr_opacity;
        la.lr[k] = static_cast<float>(lr);
    }
    la.ring = c->adam_ring;
    la.t = static_cast<uint32_t>(c->adam_t);
    // |m_hat / (sqrt(v_hat) + eps)| <= (1 - b1) sqrt(1 / (1 - b1^2 / b2)) / sqrt(1 - b2) (Cauchy-Schwarz on
    // the moment sums; the bias corrections only shrink it), and a zero-gradient step scales it by
    // rho = b1 / sqrt(b2): after k such steps a component has moved by at most
    // bound * lr * rho (1 - rho^k) / (1 - rho). drift_* = bound * lr (with 1% slack);
    // the preprocess multiplies by the geometric factor of the row's staleness.
    const double b1 = t.beta1, b2 = t.beta2;
    const double bound = (1.0 - b1) * std::sqrt(1.0 / (1.0 - b1 * b1 / b2)) / std::sqrt(1.0 - b2);
    la.rho = static_cast<float>(b1 / std::sqrt(b2) * (1.0 + 1e-6));
    la.drift_pos = static_cast<float>(1.01 * bound * std::max(t.lr_position, t.lr_position * t.lr_position_decay));
    la.drift_ls = static_cast<float>(1.01 * bound * t.lr_log_scale);
    return la;
}

void materialize(Ctx* c) {
    if (c->n == 0 || c->adam_t == 0) return;
    const LazyAdam la = make_lazy_adam(c);
    const uint32_t n = static_cast<uint32_t>(c->n);
    if (c->fd == 3)
        materialize_kernel<3><<<(n + 255) / 256, 256, 0, c->stream>>>(c->x, c->m, c->v, n, la);
    else
        materialize_kernel<12><<<(n + 255) / 256, 256, 0, c->stream>>>(c->x, c->m, c->v, n, la);
    BSG_LAUNCHED(c);
}

void reset_row_meta(Ctx* c, uint32_t stamp, bool reset_stats) {
    if (c->cap == 0) return;
    reset_row_meta_kernel<<<148 * 4, 256, 0, c->stream>>>(c->x, c->m, c->v, c->cap, row_stride(c->fd), stamp,
                                                                   reset_stats ? 1 : 0);
    BSG_LAUNCHED(c);
}

}  // namespace bsg
