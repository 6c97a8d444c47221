// K8 loss: L1 + lambda (1 - SSIM) and its image gradient dL/dC, replacing
// loss_value / ssim_with_gradient / the L1 gradient loop
// (renderer.cpp:185-192,259-272; ssim.cpp:34-185).
//
// Pass A (windows): per 64x16 tile of valid 11x11 windows and per channel,
// the five blurred moments (x, y, x^2, y^2, xy) by a separable pass over a
// shared-memory patch, then SSIM and the three partial maps
// f1 = A - 2 mu_x B - mu_y C, f2 = 2B, f3 = C (ssim.cpp:153-172).
// Pass B (pixels): per 64x16 pixel tile, the adjoint of the valid blur
// ("spread", full correlation with zero padding == valid correlation of the
// zero-padded maps with the symmetric window) of f1..f3, then
// dL/dC = sign(x - y)/(3HW) - lambda (g1 + x g2 + y g3)/count.
// Each thread produces 4 adjacent outputs per pass so a row of inputs is read
// with 128-bit shared loads and reused across 4 outputs (register blocking).
// Loss partials are reduced to FP64.
#include <type_traits>

#include "bsg_internal.cuh"

namespace bsg {
namespace {

constexpr int kW = 11, kHalf = 5;
constexpr int kTX = 64, kTY = 16;                 // outputs per tile
constexpr int kPX = kTX + 2 * kHalf;              // 74 patch columns
constexpr int kPY = kTY + 2 * kHalf;              // 26 patch rows
constexpr int kPS = 76;                           // padded row stride (16 B aligned)
constexpr int kThreads = 256;
// ssim_window_1d (ssim.cpp:112-122): exp(-d^2 / (2 1.5^2)) normalised in FP64,
// rounded to FP32. Compile-time immediates so every tap is an FFMA with an
// immediate operand (half the FMA-pipe occupancy of a register/constant
// operand); launch_loss re-derives them on the host and refuses to run on a
// mismatch.
__device__ constexpr float kWin[kW] = {0x1.0d956cp-10f, 0x1.f1fe02p-8f, 0x1.26eb18p-5f, 0x1.bff0fep-4f,
                                       0x1.b43c40p-3f,  0x1.106560p-2f, 0x1.b43c40p-3f, 0x1.bff0fep-4f,
                                       0x1.26eb18p-5f,  0x1.f1fe02p-8f, 0x1.0d956cp-10f};
constexpr float kWinHost[kW] = {0x1.0d956cp-10f, 0x1.f1fe02p-8f, 0x1.26eb18p-5f, 0x1.bff0fep-4f,
                                0x1.b43c40p-3f,  0x1.106560p-2f, 0x1.b43c40p-3f, 0x1.bff0fep-4f,
                                0x1.26eb18p-5f,  0x1.f1fe02p-8f, 0x1.0d956cp-10f};

__device__ __forceinline__ double block_sum_d(double v, double* s_red) {
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    if (lane == 0) s_red[warp] = v;
    __syncthreads();
    double t = 0;
    if (threadIdx.x == 0)
        for (int w = 0; w < (kThreads >> 5); ++w) t += s_red[w];
    __syncthreads();
    return t;
}

// 16 consecutive floats of a patch row (16 B aligned).
__device__ __forceinline__ void load16(const float* p, float (&v)[16]) {
#pragma unroll
    for (int k = 0; k < 4; ++k) {
        const float4 q = reinterpret_cast<const float4*>(p)[k];
        v[4 * k] = q.x; v[4 * k + 1] = q.y; v[4 * k + 2] = q.z; v[4 * k + 3] = q.w;
    }
}

// Four adjacent 11-tap correlations of a 14-wide window of v.
__device__ __forceinline__ void corr4(const float (&v)[16], float (&o)[4]) {
#pragma unroll
    for (int j = 0; j < 4; ++j) {
        float s = 0.f;
#pragma unroll
        for (int t = 0; t < kW; ++t) s += kWin[t] * v[j + t];
        o[j] = s;
    }
}

// Ground truth as FP32, or as the 8-bit values of the reference's PPM images
// (bsg_train_steps_host_u8): the reference's dequantisation v / 255 in FP64
// rounded to FP32 (image.cpp:21-27), here as q = v r (r = 1/255 rounded)
// refined by one FMA residual step -- the correctly rounded FP32 quotient,
// equal to the FP64 one rounded, for every v in 0..255 (checked exhaustively;
// three FMA-pipe ops instead of an IEEE division).
__device__ __forceinline__ float gt_val(const float* __restrict__ y, size_t p) { return y[p]; }
__device__ __forceinline__ float gt_val(const uint8_t* __restrict__ y, size_t p) {
    constexpr float r = 1.0f / 255.0f;
    const float v = static_cast<float>(y[p]);
    const float q = __fmul_rn(v, r);
    return __fmaf_rn(__fmaf_rn(-q, 255.f, v), r, q);
}

struct WinSmem {
    float x[2][kPY][kPS], y[2][kPY][kPS];
    float h[5][kPY][kTX];
};

__device__ __forceinline__ void cp_async4(float* dst, const float* src, bool ok) {
    const unsigned d = static_cast<unsigned>(__cvta_generic_to_shared(dst));
    asm volatile("cp.async.ca.shared.global [%0], [%1], 4, %2;\n" ::"r"(d), "l"(src), "r"(ok ? 4 : 0));
}

// x, y: HxWx3 FP32 (y: FP32 or 8-bit). f: [3 channels][3 maps][Hv][Wv].
// Double-buffered patches: channel ch+1's loads are in flight (cp.async; for
// 8-bit ground truth the y patch is converted through registers) while
// channel ch is blurred.
template <typename G>
__global__ __launch_bounds__(kThreads) void ssim_windows_kernel(const float* __restrict__ x,
                                                                const G* __restrict__ y, int W, int H,
                                                                float* __restrict__ f, double* __restrict__ ssim_sum) {
    pdl_prologue();
    extern __shared__ __align__(16) unsigned char smem_raw[];
    WinSmem& S = *reinterpret_cast<WinSmem*>(smem_raw);
    __shared__ double s_red[kThreads / 32];
    const int Wv = W - 2 * kHalf, Hv = H - 2 * kHalf;
    const int wx0 = blockIdx.x * kTX, wy0 = blockIdx.y * kTY;
    const float C1 = 1e-4f, C2 = 9e-4f;
    const size_t plane = static_cast<size_t>(Wv) * Hv;
    // window (wx, wy) covers pixels [wx, wx+10] x [wy, wy+10]; patch rows per
    // warp, columns per lane, consecutive lanes on consecutive pixels
    auto fetch = [&](int ch, int buf) {
        for (int ly = threadIdx.x >> 5; ly < kPY; ly += kThreads / 32) {
            const int gy = wy0 + ly, lane = threadIdx.x & 31;
#pragma unroll
            for (int cc = 0; cc < 3; ++cc) {
                const int lx = lane + 32 * cc, gx = wx0 + lx;
                if (lx < kPX) {
                    const bool ok = gx < W && gy < H;
                    const size_t p = ok ? 3 * (static_cast<size_t>(gy) * W + gx) + ch : 0;
                    cp_async4(&S.x[buf][ly][lx], x + p, ok);
                    if constexpr (std::is_same<G, float>::value) {
                        cp_async4(&S.y[buf][ly][lx], y + p, ok);
                    } else {
                        S.y[buf][ly][lx] = ok ? gt_val(y, p) : 0.f;
                    }
                }
            }
        }
        asm volatile("cp.async.commit_group;\n" ::);
    };
    fetch(0, 0);
    double local = 0.0;
    for (int ch = 0; ch < 3; ++ch) {
        const int buf = ch & 1;
        if (ch < 2) {
            fetch(ch + 1, buf ^ 1);
            asm volatile("cp.async.wait_group 1;\n" ::);
        } else {
            asm volatile("cp.async.wait_group 0;\n" ::);
        }
        __syncthreads();
        // horizontal: 26 rows x 16 groups of 4 outputs, five moments
        for (int it = threadIdx.x; it < kPY * (kTX / 4); it += kThreads) {
            const int r = it / (kTX / 4), g4 = 4 * (it % (kTX / 4));
            float a[16], b[16], t[16], o[4];
            load16(&S.x[buf][r][g4], a);
            load16(&S.y[buf][r][g4], b);
            corr4(a, o);
            *reinterpret_cast<float4*>(&S.h[0][r][g4]) = make_float4(o[0], o[1], o[2], o[3]);
            corr4(b, o);
            *reinterpret_cast<float4*>(&S.h[1][r][g4]) = make_float4(o[0], o[1], o[2], o[3]);
#pragma unroll
            for (int k = 0; k < 16; ++k) t[k] = a[k] * a[k];
            corr4(t, o);
            *reinterpret_cast<float4*>(&S.h[2][r][g4]) = make_float4(o[0], o[1], o[2], o[3]);
#pragma unroll
            for (int k = 0; k < 16; ++k) t[k] = b[k] * b[k];
            corr4(t, o);
            *reinterpret_cast<float4*>(&S.h[3][r][g4]) = make_float4(o[0], o[1], o[2], o[3]);
#pragma unroll
            for (int k = 0; k < 16; ++k) t[k] = a[k] * b[k];
            corr4(t, o);
            *reinterpret_cast<float4*>(&S.h[4][r][g4]) = make_float4(o[0], o[1], o[2], o[3]);
        }
        __syncthreads();
        // vertical: thread = one column, four consecutive window rows
        {
            const int col = threadIdx.x % kTX, r0 = 4 * (threadIdx.x / kTX);
            float m[5][4];
#pragma unroll
            for (int q = 0; q < 5; ++q) {
                float v[16];
#pragma unroll
                for (int k = 0; k < 14; ++k) v[k] = S.h[q][r0 + k][col];
                v[14] = v[15] = 0.f;
                corr4(v, m[q]);
            }
            const int wx = wx0 + col;
#pragma unroll
            for (int j = 0; j < 4; ++j) {
                const int wy = wy0 + r0 + j;
                if (wx < Wv && wy < Hv) {
                    const float mx = m[0][j], my = m[1][j];
                    const float vx = m[2][j] - mx * mx, vy = m[3][j] - my * my, cxy = m[4][j] - mx * my;
                    const float n1 = 2.f * mx * my + C1, n2 = 2.f * cxy + C2;
                    const float d1 = mx * mx + my * my + C1, d2 = vx + vy + C2;
                    // d1 >= C1, d2 >= C2 - O(ulp): two approximate reciprocals
                    // (~1 ulp) instead of five IEEE divisions (ssim.cpp:153-172)
                    float rd1, rd2;
                    asm("rcp.approx.ftz.f32 %0, %1;" : "=f"(rd1) : "f"(d1));
                    asm("rcp.approx.ftz.f32 %0, %1;" : "=f"(rd2) : "f"(d2));
                    const float rden = rd1 * rd2;
                    const float sv = (n1 * n2) * rden;
                    const float A = 2.f * my * n2 * rden - sv * 2.f * mx * rd1;
                    const float B = -sv * rd2;
                    const float Cc = 2.f * n1 * rden;
                    const size_t o = static_cast<size_t>(wy) * Wv + wx;
                    f[(3 * ch + 0) * plane + o] = A - 2.f * mx * B - my * Cc;
                    f[(3 * ch + 1) * plane + o] = 2.f * B;
                    f[(3 * ch + 2) * plane + o] = Cc;
                    local += static_cast<double>(sv);
                }
            }
        }
        // (no barrier: the next channel's barrier after its fetch orders the
        // S.h reads above before its horizontal pass overwrites them)
    }
    const double t = block_sum_d(local, s_red);
    if (threadIdx.x == 0) atomicAdd(ssim_sum, t);
}

// Double-buffered f patches filled by cp.async: channel ch+1's patch loads
// are in flight while channel ch is spread (the loads were the kernel's
// stall: long scoreboard); 54 KB and <= 64 registers, 4 CTAs per SM
// (cfg 3 loss stage 136 -> 128 us against the single-buffered 6-CTA form).
struct PixSmem {
    float f[2][3][kPY][kPS];
    float h[kPY][kTX];
};

// Per pixel: spread f1..f3 (adjoint of the valid blur) and form dL/dC.
template <typename G>
__global__ __launch_bounds__(kThreads, 4) void ssim_pixels_kernel(const float* __restrict__ x, const G* __restrict__ y,
                                                               int W, int H, const float* __restrict__ f, int has_ssim,
                                                               float lam_over_count, float inv_count3,
                                                               float* __restrict__ dl_dc, double* __restrict__ l1_sum) {
    pdl_prologue();
    extern __shared__ __align__(16) unsigned char smem_raw[];
    PixSmem& S = *reinterpret_cast<PixSmem*>(smem_raw);
    __shared__ double s_red[kThreads / 32];
    const int Wv = W - 2 * kHalf, Hv = H - 2 * kHalf;
    const int px0 = blockIdx.x * kTX, py0 = blockIdx.y * kTY;
    const size_t plane = static_cast<size_t>(Wv) * Hv;
    const int col = threadIdx.x % kTX, r0 = 4 * (threadIdx.x / kTX);
    // windows [px0-10, px0+63] x [py0-10, py0+15], zero outside the valid grid;
    // patch rows per warp, columns per lane
    auto fetch = [&](int ch, int buf) {
        for (int ly = threadIdx.x >> 5; ly < kPY; ly += kThreads / 32) {
            const int wy = py0 - 2 * kHalf + ly, lane = threadIdx.x & 31;
#pragma unroll
            for (int cc = 0; cc < 3; ++cc) {
                const int lx = lane + 32 * cc, wx = px0 - 2 * kHalf + lx;
                if (lx < kPX) {
                    const bool ok = wx >= 0 && wy >= 0 && wx < Wv && wy < Hv;
                    const size_t o = ok ? static_cast<size_t>(wy) * Wv + wx : 0;
#pragma unroll
                    for (int m = 0; m < 3; ++m) cp_async4(&S.f[buf][m][ly][lx], f + (3 * ch + m) * plane + o, ok);
                }
            }
        }
        asm volatile("cp.async.commit_group;\n" ::);
    };
    if (has_ssim) fetch(0, 0);
    double local = 0.0;
    for (int ch = 0; ch < 3; ++ch) {
        float g[3][4] = {{0.f, 0.f, 0.f, 0.f}, {0.f, 0.f, 0.f, 0.f}, {0.f, 0.f, 0.f, 0.f}};
        const int px = px0 + col;
        float xa[4], yb[4];
#pragma unroll
        for (int j = 0; j < 4; ++j) {
            const int py = py0 + r0 + j;
            xa[j] = yb[j] = 0.f;
            if (px < W && py < H) {
                const size_t p = 3 * (static_cast<size_t>(py) * W + px) + ch;
                xa[j] = x[p];
                yb[j] = gt_val(y, p);
            }
        }
        if (has_ssim) {
            const int buf = ch & 1;
            if (ch < 2) {
                fetch(ch + 1, buf ^ 1);
                asm volatile("cp.async.wait_group 1;\n" ::);
            } else {
                asm volatile("cp.async.wait_group 0;\n" ::);
            }
            __syncthreads();
#pragma unroll
            for (int m = 0; m < 3; ++m) {
                for (int it = threadIdx.x; it < kPY * (kTX / 4); it += kThreads) {
                    const int r = it / (kTX / 4), g4 = 4 * (it % (kTX / 4));
                    float a[16], o[4];
                    load16(&S.f[buf][m][r][g4], a);
                    corr4(a, o);  // symmetric window: full correlation of the padded map
                    *reinterpret_cast<float4*>(&S.h[r][g4]) = make_float4(o[0], o[1], o[2], o[3]);
                }
                __syncthreads();
                float v[16];
#pragma unroll
                for (int k = 0; k < 14; ++k) v[k] = S.h[r0 + k][col];
                v[14] = v[15] = 0.f;
                corr4(v, g[m]);
                __syncthreads();
            }
        }
#pragma unroll
        for (int j = 0; j < 4; ++j) {
            const int py = py0 + r0 + j;
            if (px < W && py < H) {
                const size_t p = 3 * (static_cast<size_t>(py) * W + px) + ch;
                const float a = xa[j], b = yb[j];
                const float diff = a - b;
                const float sgn = diff > 0.f ? 1.f : (diff < 0.f ? -1.f : 0.f);
                local += fabs(static_cast<double>(diff));
                dl_dc[p] = sgn * inv_count3 - lam_over_count * (g[0][j] + a * g[1][j] + b * g[2][j]);
            }
        }
    }
    const double t = block_sum_d(local, s_red);
    if (threadIdx.x == 0) atomicAdd(l1_sum, t);
}

__global__ void finalize_kernel(const StepScalars* s, double inv_count3, double inv_count, int has_ssim, double lambda,
                                int add_penalty, double* out) {
    pdl_prologue();
    const double l1 = s->l1_sum * inv_count3;
    const double ss = has_ssim ? s->ssim_sum * inv_count : 1.0;
    double loss = l1 + lambda * (1.0 - ss);
    if (add_penalty) loss += s->penalty;
    out[0] = loss;
    out[1] = l1;
    out[2] = ss;
}

bool g_ready[64] = {};

}  // namespace

void ensure_ssim_ready(Ctx* c) {
    if (!g_ready[c->device]) {
        // ssim_window_1d (ssim.cpp:112-122), computed in FP64 then rounded: must
        // equal the compiled-in taps.
        double k[kW], sum = 0;
        for (int i = 0; i < kW; ++i) {
            const double d = i - kHalf;
            k[i] = std::exp(-d * d / (2.0 * 1.5 * 1.5));
            sum += k[i];
        }
        for (int i = 0; i < kW; ++i)
            if (static_cast<float>(k[i] / sum) != kWinHost[i])
                throw Error{BSG_ERR_CUDA, "SSIM window taps differ from ssim_window_1d"};
        BSG_CUDA(cudaFuncSetAttribute(ssim_windows_kernel<float>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                      static_cast<int>(sizeof(WinSmem))));
        BSG_CUDA(cudaFuncSetAttribute(ssim_windows_kernel<uint8_t>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                      static_cast<int>(sizeof(WinSmem))));
        BSG_CUDA(cudaFuncSetAttribute(ssim_pixels_kernel<float>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                      static_cast<int>(sizeof(PixSmem))));
        BSG_CUDA(cudaFuncSetAttribute(ssim_pixels_kernel<uint8_t>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                      static_cast<int>(sizeof(PixSmem))));
        g_ready[c->device] = true;
    }
}

namespace {

template <typename G>
void launch_loss_t(Ctx* c, const DevCam& cam, const DevRender& rc, const G* gt) {
    ensure_ssim_ready(c);
    const int W = cam.W, H = cam.H;
    const bool has_ssim = W >= kW && H >= kW;
    const int Wv = W - 2 * kHalf, Hv = H - 2 * kHalf;
    const double count = has_ssim ? 3.0 * Wv * Hv : 1.0;
    if (has_ssim) {
        dim3 grid((Wv + kTX - 1) / kTX, (Hv + kTY - 1) / kTY);
        launch_pdl(c->stream, grid, kThreads, sizeof(WinSmem), ssim_windows_kernel<G>, c->out_rgb, gt, W, H, c->ssim_f,
                   &c->scalars->ssim_sum);
        BSG_LAUNCHED(c);
    }
    dim3 grid2((W + kTX - 1) / kTX, (H + kTY - 1) / kTY);
    launch_pdl(c->stream, grid2, kThreads, sizeof(PixSmem), ssim_pixels_kernel<G>, c->out_rgb, gt, W, H, c->ssim_f,
               has_ssim ? 1 : 0, static_cast<float>(rc.lambda / count), static_cast<float>(1.0 / (3.0 * W * H)),
               c->dl_dc, &c->scalars->l1_sum);
    BSG_LAUNCHED(c);
}

}  // namespace

void launch_loss(Ctx* c, const DevCam& cam, const DevRender& rc, const float* gt) { launch_loss_t(c, cam, rc, gt); }
void launch_loss(Ctx* c, const DevCam& cam, const DevRender& rc, const uint8_t* gt) { launch_loss_t(c, cam, rc, gt); }

// Windows pass only (mean SSIM into scalars->ssim_sum); false when the image
// is smaller than the window (ssim.cpp:12-14: SSIM = 1).
bool launch_ssim_windows(Ctx* c, const DevCam& cam, const float* gt) {
    const int W = cam.W, H = cam.H;
    if (W < kW || H < kW) return false;
    ensure_ssim_ready(c);
    const int Wv = W - 2 * kHalf, Hv = H - 2 * kHalf;
    dim3 grid((Wv + kTX - 1) / kTX, (Hv + kTY - 1) / kTY);
    launch_pdl(c->stream, grid, kThreads, sizeof(WinSmem), ssim_windows_kernel<float>, c->out_rgb, gt, W, H, c->ssim_f,
               &c->scalars->ssim_sum);
    BSG_LAUNCHED(c);
    return true;
}

void launch_finalize_loss(Ctx* c, const DevCam& cam, const DevRender& rc, double* out, bool add_penalty) {
    const int W = cam.W, H = cam.H;
    const bool has_ssim = W >= kW && H >= kW;
    const double count = has_ssim ? 3.0 * (W - 2 * kHalf) * (H - 2 * kHalf) : 1.0;
    launch_pdl(c->stream, 1, 1, 0, finalize_kernel, c->scalars, 1.0 / (3.0 * W * H), 1.0 / count, has_ssim ? 1 : 0, rc.lambda,
                                            add_penalty ? 1 : 0, out);
    BSG_LAUNCHED(c);
}

}  // namespace bsg
