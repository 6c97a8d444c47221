// GPU evaluation path: evaluate (metrics.cpp:28-51) of the
// block's cloud over holdout views -- render (K1-K7), PSNR (metrics.cpp:14-26)
// from an FP64 sum of squared differences against the FP64 ground truth, and
// mean SSIM (ssim.cpp) from the windows pass of the loss kernels.
#include <cmath>
#include <vector>

#include "bsg_internal.cuh"

namespace bsg {
namespace {

__global__ __launch_bounds__(256) void sqdiff_kernel(const float* __restrict__ rgb, const double* __restrict__ gt,
                                                     size_t n, double* __restrict__ out) {
    __shared__ double s_red[8];
    double acc = 0.0;
    for (size_t i = blockIdx.x * static_cast<size_t>(blockDim.x) + threadIdx.x; i < n;
         i += static_cast<size_t>(gridDim.x) * blockDim.x) {
        const double d = static_cast<double>(rgb[i]) - gt[i];
        acc += d * d;
    }
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) acc += __shfl_xor_sync(0xffffffffu, acc, o);
    if ((threadIdx.x & 31) == 0) s_red[threadIdx.x >> 5] = acc;
    __syncthreads();
    if (threadIdx.x == 0) {
        double t = 0;
        for (int w = 0; w < 8; ++w) t += s_red[w];
        atomicAdd(out, t);
    }
}

__global__ void narrow_kernel(const double* __restrict__ in, float* __restrict__ out, size_t n) {
    for (size_t i = blockIdx.x * static_cast<size_t>(blockDim.x) + threadIdx.x; i < n;
         i += static_cast<size_t>(gridDim.x) * blockDim.x)
        out[i] = static_cast<float>(in[i]);
}

}  // namespace

// One holdout view: render with rc, then squared error and SSIM against gt
// (device FP64, 3HW). Returns {psnr, ssim} (metrics.cpp:14-26, ssim.cpp).
void eval_view(Ctx* c, const DevCam& cam, const DevRender& rc, const double* gt_dev, double* scratch, double out[2]) {
    project_and_bin_public(c, cam, rc);
    launch_blend_fwd(c, cam, rc);
    const size_t n = 3 * static_cast<size_t>(cam.W) * cam.H;
    BSG_CUDA(cudaMemsetAsync(scratch, 0, sizeof(double), c->stream));
    BSG_CUDA(cudaMemsetAsync(c->scalars, 0, sizeof(StepScalars), c->stream));
    const unsigned grid = static_cast<unsigned>(std::min<size_t>((n + 255) / 256, 148 * 8));
    sqdiff_kernel<<<grid, 256, 0, c->stream>>>(c->out_rgb, gt_dev, n, scratch);
    BSG_LAUNCHED(c);
    narrow_kernel<<<grid, 256, 0, c->stream>>>(gt_dev, c->gt_stage, n);
    BSG_LAUNCHED(c);
    const bool has_ssim = launch_ssim_windows(c, cam, c->gt_stage);
    double h[2] = {0, 0};
    BSG_CUDA(cudaMemcpyAsync(&h[0], scratch, sizeof(double), cudaMemcpyDeviceToHost, c->stream));
    BSG_CUDA(cudaMemcpyAsync(&h[1], &c->scalars->ssim_sum, sizeof(double), cudaMemcpyDeviceToHost, c->stream));
    BSG_CUDA(cudaStreamSynchronize(c->stream));
    const double mse = h[0] / static_cast<double>(n);
    out[0] = mse <= 0 ? 99.0 : std::min(99.0, 10.0 * std::log10(1.0 / mse));
    const double windows = 3.0 * (cam.W - 10) * (cam.H - 10);
    out[1] = has_ssim ? h[1] / windows : 1.0;
}

}  // namespace bsg
