// K7 loss: L1 + lambda (1 - SSIM) and its image gradient dL/dC, replacing
// loss_value / ssim_with_gradient / the L1 gradient loop
// (renderer.cpp:185-192,259-272; ssim.cpp:34-185).
//
// Pass A (per valid 11x11 window, tiles of 32x8 windows): separable Gaussian
// blur of x, y, x^2, y^2, xy from a shared-memory patch, per-window SSIM and
// the three partial maps f1 = A - 2 mu_x B - mu_y C, f2 = 2B, f3 = C
// (ssim.cpp:153-172). Pass B (per pixel, tiles of 32x8): the adjoint
// ("spread", full correlation with zero padding) of f1..f3 from a patch, then
// dL/dC = sign(x - y)/(3HW) - lambda (g1 + x g2 + y g3)/count. Both passes are
// HBM/L2 streaming stencils. Reductions of the loss terms go to FP64.
#include "bsg_internal.cuh"

namespace bsg {
namespace {

constexpr int kW = 11, kHalf = 5;
constexpr int kTx = 32, kTy = 8;
constexpr int kPx = kTx + 2 * kHalf, kPy = kTy + 2 * kHalf;  // 42 x 18 patch
__constant__ float c_win[kW];

__device__ __forceinline__ double block_sum_d(double v, double* s_red) {
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    if (lane == 0) s_red[warp] = v;
    __syncthreads();
    double t = 0;
    if (threadIdx.x == 0)
        for (int w = 0; w < (blockDim.x >> 5); ++w) t += s_red[w];
    __syncthreads();
    return t;
}

// x, y: HxWx3 FP32. f: [3 channels][3 maps][Hv][Wv].
__global__ __launch_bounds__(256) void ssim_windows_kernel(const float* __restrict__ x, const float* __restrict__ y,
                                                           int W, int H, float* __restrict__ f,
                                                           double* __restrict__ ssim_sum) {
    __shared__ float s_x[kPy][kPx], s_y[kPy][kPx];
    __shared__ float s_h[5][kPy][kTx];
    __shared__ double s_red[8];
    const int Wv = W - 2 * kHalf, Hv = H - 2 * kHalf;
    const int wx0 = blockIdx.x * kTx, wy0 = blockIdx.y * kTy;
    const int tx = threadIdx.x % kTx, ty = threadIdx.x / kTx;
    const float C1 = 1e-4f, C2 = 9e-4f;
    double local = 0.0;
    for (int ch = 0; ch < 3; ++ch) {
        // window (wx, wy) covers pixels [wx, wx+10] x [wy, wy+10]
        for (int k = threadIdx.x; k < kPx * kPy; k += 256) {
            const int lx = k % kPx, ly = k / kPx;
            const int gx = wx0 + lx, gy = wy0 + ly;
            float a = 0.f, b = 0.f;
            if (gx < W && gy < H) {
                const size_t p = 3 * (static_cast<size_t>(gy) * W + gx) + ch;
                a = x[p];
                b = y[p];
            }
            s_x[ly][lx] = a;
            s_y[ly][lx] = b;
        }
        __syncthreads();
        for (int k = threadIdx.x; k < kPy * kTx; k += 256) {
            const int lx = k % kTx, ly = k / kTx;
            float sx = 0, sy = 0, sxx = 0, syy = 0, sxy = 0;
#pragma unroll
            for (int t = 0; t < kW; ++t) {
                const float w = c_win[t], a = s_x[ly][lx + t], b = s_y[ly][lx + t];
                sx += w * a;
                sy += w * b;
                sxx += w * (a * a);
                syy += w * (b * b);
                sxy += w * (a * b);
            }
            s_h[0][ly][lx] = sx; s_h[1][ly][lx] = sy; s_h[2][ly][lx] = sxx; s_h[3][ly][lx] = syy; s_h[4][ly][lx] = sxy;
        }
        __syncthreads();
        const int wx = wx0 + tx, wy = wy0 + ty;
        if (wx < Wv && wy < Hv) {
            float mx = 0, my = 0, ex2 = 0, ey2 = 0, exy = 0;
#pragma unroll
            for (int t = 0; t < kW; ++t) {
                const float w = c_win[t];
                mx += w * s_h[0][ty + t][tx];
                my += w * s_h[1][ty + t][tx];
                ex2 += w * s_h[2][ty + t][tx];
                ey2 += w * s_h[3][ty + t][tx];
                exy += w * s_h[4][ty + t][tx];
            }
            const float vx = ex2 - mx * mx, vy = ey2 - my * my, cxy = exy - mx * my;
            const float n1 = 2.f * mx * my + C1, n2 = 2.f * cxy + C2;
            const float d1 = mx * mx + my * my + C1, d2 = vx + vy + C2;
            const float denom = d1 * d2;
            const float sv = (n1 * n2) / denom;
            const float A = 2.f * my * n2 / denom - sv * 2.f * mx / d1;
            const float B = -sv / d2;
            const float Cc = 2.f * n1 / denom;
            const size_t plane = static_cast<size_t>(Wv) * Hv;
            const size_t o = static_cast<size_t>(wy) * Wv + wx;
            f[(3 * ch + 0) * plane + o] = A - 2.f * mx * B - my * Cc;
            f[(3 * ch + 1) * plane + o] = 2.f * B;
            f[(3 * ch + 2) * plane + o] = Cc;
            local += static_cast<double>(sv);
        }
        __syncthreads();
    }
    const double t = block_sum_d(local, s_red);
    if (threadIdx.x == 0) atomicAdd(ssim_sum, t);
}

// Per pixel: spread f1..f3 (adjoint of the valid blur) and form dL/dC.
__global__ __launch_bounds__(256) void ssim_pixels_kernel(const float* __restrict__ x, const float* __restrict__ y,
                                                          int W, int H, const float* __restrict__ f, int has_ssim,
                                                          float lam_over_count, float inv_count3,
                                                          float* __restrict__ dl_dc, double* __restrict__ l1_sum) {
    __shared__ float s_f[3][kPy][kPx];
    __shared__ float s_v[3][kTy][kPx];
    __shared__ double s_red[8];
    const int Wv = W - 2 * kHalf, Hv = H - 2 * kHalf;
    const int px0 = blockIdx.x * kTx, py0 = blockIdx.y * kTy;
    const int tx = threadIdx.x % kTx, ty = threadIdx.x / kTx;
    const int px = px0 + tx, py = py0 + ty;
    const bool inside = px < W && py < H;
    double local = 0.0;
    for (int ch = 0; ch < 3; ++ch) {
        float g1 = 0.f, g2 = 0.f, g3 = 0.f;
        if (has_ssim) {
            // windows [px0-10, px0+31] x [py0-10, py0+7]
            const size_t plane = static_cast<size_t>(Wv) * Hv;
            for (int k = threadIdx.x; k < kPx * kPy; k += 256) {
                const int lx = k % kPx, ly = k / kPx;
                const int wx = px0 - 2 * kHalf + lx, wy = py0 - 2 * kHalf + ly;
                const bool ok = wx >= 0 && wy >= 0 && wx < Wv && wy < Hv;
                const size_t o = ok ? static_cast<size_t>(wy) * Wv + wx : 0;
#pragma unroll
                for (int m = 0; m < 3; ++m) s_f[m][ly][lx] = ok ? f[(3 * ch + m) * plane + o] : 0.f;
            }
            __syncthreads();
            // vertical: v(wx, py) = sum_t k[t] f(wx, py - t)
            for (int k = threadIdx.x; k < kTy * kPx; k += 256) {
                const int lx = k % kPx, ly = k / kPx;
                float a = 0, b = 0, c = 0;
#pragma unroll
                for (int t = 0; t < kW; ++t) {
                    const float w = c_win[t];
                    a += w * s_f[0][ly + 2 * kHalf - t][lx];
                    b += w * s_f[1][ly + 2 * kHalf - t][lx];
                    c += w * s_f[2][ly + 2 * kHalf - t][lx];
                }
                s_v[0][ly][lx] = a; s_v[1][ly][lx] = b; s_v[2][ly][lx] = c;
            }
            __syncthreads();
#pragma unroll
            for (int t = 0; t < kW; ++t) {
                const float w = c_win[t];
                g1 += w * s_v[0][ty][tx + 2 * kHalf - t];
                g2 += w * s_v[1][ty][tx + 2 * kHalf - t];
                g3 += w * s_v[2][ty][tx + 2 * kHalf - t];
            }
            __syncthreads();
        }
        if (inside) {
            const size_t p = 3 * (static_cast<size_t>(py) * W + px) + ch;
            const float a = x[p], b = y[p];
            const float diff = a - b;
            const float sgn = diff > 0.f ? 1.f : (diff < 0.f ? -1.f : 0.f);
            local += fabs(static_cast<double>(diff));
            dl_dc[p] = sgn * inv_count3 - lam_over_count * (g1 + a * g2 + b * g3);
        }
    }
    const double t = block_sum_d(local, s_red);
    if (threadIdx.x == 0) atomicAdd(l1_sum, t);
}

__global__ void finalize_kernel(const StepScalars* s, double inv_count3, double inv_count, int has_ssim, double lambda,
                                int add_penalty, double* out) {
    const double l1 = s->l1_sum * inv_count3;
    const double ss = has_ssim ? s->ssim_sum * inv_count : 1.0;
    double loss = l1 + lambda * (1.0 - ss);
    if (add_penalty) loss += s->penalty;
    out[0] = loss;
    out[1] = l1;
    out[2] = ss;
}

bool g_win_ready[64] = {};

}  // namespace

void launch_loss(Ctx* c, const DevCam& cam, const DevRender& rc, const float* gt) {
    if (!g_win_ready[c->device]) {
        // ssim_window_1d (ssim.cpp:112-122), computed in FP64 then rounded.
        float w[kW];
        double k[kW], sum = 0;
        for (int i = 0; i < kW; ++i) {
            const double d = i - kHalf;
            k[i] = std::exp(-d * d / (2.0 * 1.5 * 1.5));
            sum += k[i];
        }
        for (int i = 0; i < kW; ++i) w[i] = static_cast<float>(k[i] / sum);
        BSG_CUDA(cudaMemcpyToSymbol(c_win, w, sizeof(w)));
        g_win_ready[c->device] = true;
    }
    const int W = cam.W, H = cam.H;
    const bool has_ssim = W >= kW && H >= kW;
    const int Wv = W - 2 * kHalf, Hv = H - 2 * kHalf;
    const double count = has_ssim ? 3.0 * Wv * Hv : 1.0;
    if (has_ssim) {
        dim3 grid((Wv + kTx - 1) / kTx, (Hv + kTy - 1) / kTy);
        ssim_windows_kernel<<<grid, 256, 0, c->stream>>>(c->out_rgb, gt, W, H, c->ssim_f, &c->scalars->ssim_sum);
        BSG_LAUNCHED(c);
    }
    dim3 grid2((W + kTx - 1) / kTx, (H + kTy - 1) / kTy);
    ssim_pixels_kernel<<<grid2, 256, 0, c->stream>>>(c->out_rgb, gt, W, H, c->ssim_f, has_ssim ? 1 : 0,
                                                     static_cast<float>(rc.lambda / count),
                                                     static_cast<float>(1.0 / (3.0 * W * H)), c->dl_dc,
                                                     &c->scalars->l1_sum);
    BSG_LAUNCHED(c);
}

void launch_finalize_loss(Ctx* c, const DevCam& cam, const DevRender& rc, double* out, bool add_penalty) {
    const int W = cam.W, H = cam.H;
    const bool has_ssim = W >= kW && H >= kW;
    const double count = has_ssim ? 3.0 * (W - 2 * kHalf) * (H - 2 * kHalf) : 1.0;
    finalize_kernel<<<1, 1, 0, c->stream>>>(c->scalars, 1.0 / (3.0 * W * H), 1.0 / count, has_ssim ? 1 : 0, rc.lambda,
                                            add_penalty ? 1 : 0, out);
    BSG_LAUNCHED(c);
}

}  // namespace bsg
