// K11-K14: consensus round on the shared Gaussians over a compact global
// slot index. Replaces consensus_average / dual_update / residuals
// (admm.cpp:71-198), the worker half of apply_broadcast (trainer.cpp:168-223)
// and the master's gather/broadcast (runtime.cpp:482-570).
//
// Sum over owners is a reduction (NCCL AllReduce over NVLink, or an in-order
// sum for a single-process group), so every block ends the round holding z
// for every slot: there is no master hop. The quaternion sign alignment to the
// lowest-id owner (admm.cpp:100-106) needs that owner's q first, so a 4-float
// pre-reduction publishes it. HBM-bound element-wise kernels.
#include <cfloat>

#include "bsg_internal.cuh"

namespace bsg {
namespace {

__device__ __forceinline__ float relaxed(float x, float zp, float alpha, bool blend) {
    // admm.hpp:38-41: alpha == 1 returns x bitwise.
    if (!blend || alpha == 1.0f) return x;
    return alpha * x + (1.0f - alpha) * zp;
}

__global__ void pack_q_kernel(const float* __restrict__ x, int fd, const uint32_t* __restrict__ rows,
                              const uint32_t* __restrict__ slots, const uint8_t* __restrict__ first, size_t ns,
                              size_t S, float* __restrict__ qref) {
    const size_t j = blockIdx.x * static_cast<size_t>(blockDim.x) + threadIdx.x;
    if (j >= ns || !first[j]) return;
    const uint32_t r = rows[j], s = slots[j];
#pragma unroll
    for (int c = 0; c < 4; ++c) qref[c * S + s] = x[pidx(r, kRot + c, fd)];
}

template <int D>
__global__ __launch_bounds__(256) void pack_main_kernel(const float* __restrict__ x, size_t cap,
                                                        const uint32_t* __restrict__ rows,
                                                        const uint32_t* __restrict__ slots,
                                                        const uint8_t* __restrict__ first, size_t ns, size_t S,
                                                        const float* __restrict__ qref,
                                                        const float* __restrict__ zprev,
                                                        const uint8_t* __restrict__ in_zprev, float alpha, int relax,
                                                        float* __restrict__ pack) {
    const size_t j = blockIdx.x * static_cast<size_t>(blockDim.x) + threadIdx.x;
    if (j >= ns) return;
    const uint32_t r = rows[j], s = slots[j];
    const bool blend = relax && in_zprev[s];
    float v[D], zp[D];
#pragma unroll
    for (int c = 0; c < D; ++c) {
        v[c] = x[pidx(r, c, D - 11)];
        zp[c] = blend ? zprev[c * S + s] : 0.f;
    }
    float flip = 0.f;
    if (!first[j]) {
        const float dot = ((v[kRot] * qref[s] + v[kRot + 1] * qref[S + s]) + v[kRot + 2] * qref[2 * S + s]) +
                          v[kRot + 3] * qref[3 * S + s];
        if (dot < 0.f) {
#pragma unroll
            for (int c = kRot; c < kRot + 4; ++c) v[c] = -v[c];
            flip = 1.f;
        }
    }
#pragma unroll
    for (int c = 0; c < D; ++c) pack[c * S + s] = relaxed(v[c], zp[c], alpha, blend);
    pack[static_cast<size_t>(D) * S + s] = flip;
}

__device__ __forceinline__ void block_add(double v, double* dst, double* s_red) {
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
    if ((threadIdx.x & 31) == 0) s_red[threadIdx.x >> 5] = v;
    __syncthreads();
    if (threadIdx.x == 0) {
        double t = 0;
        for (int w = 0; w < static_cast<int>(blockDim.x >> 5); ++w) t += s_red[w];
        if (t != 0.0) atomicAdd(dst, t);
    }
}

// Worker half (trainer.cpp:186-222): x_hat = relaxed(x, anchor) WITHOUT the
// sign flip, u += x_hat - z, reset flipped / listed slots, anchor := z; plus
// this block's share of the primal residual (raw x, admm.cpp:151-165).
__global__ __launch_bounds__(256) void dual_update_kernel(const float* __restrict__ x, size_t cap, int D,
                                                          const uint32_t* __restrict__ rows,
                                                          const uint32_t* __restrict__ slots, size_t ns, size_t S,
                                                          const float* __restrict__ pack,
                                                          const float* __restrict__ zslot,
                                                          const uint8_t* __restrict__ slot_reset, float alpha,
                                                          int relax, float* __restrict__ z, float* __restrict__ u,
                                                          double* __restrict__ scal) {
    __shared__ double s_red[8];
    const size_t j = blockIdx.x * static_cast<size_t>(blockDim.x) + threadIdx.x;
    double p2 = 0.0;
    if (j < ns) {
        const uint32_t r = rows[j], s = slots[j];
        const bool reset = pack[static_cast<size_t>(D) * S + s] > 0.f || (slot_reset && slot_reset[s]);
        for (int c = 0; c < D; ++c) {
            const float xv = x[pidx(r, c, D - 11)];
            const float zn = zslot[c * S + s];
            const float xh = relaxed(xv, z[c * ns + j], alpha, relax != 0);
            const double dr = static_cast<double>(xv) - zn;
            p2 += dr * dr;
            u[c * ns + j] = reset ? 0.f : u[c * ns + j] + (xh - zn);
            z[c * ns + j] = zn;
        }
    }
    block_add(p2, &scal[0], s_red);
}

// One pass over this block's shared rows after the reduction of `pack`
// (replaces a pass over every global slot): z = sum / owners for the block's
// own slots, this block's share of the dual residual (admm.cpp:183-198; each
// slot counted by its lowest owner only, summed across ranks with the primal
// partials) and of the flip count, z_prev := z, and the worker half of
// apply_broadcast (trainer.cpp:186-222): x_hat = relaxed(x, anchor) WITHOUT the
// sign flip, u += x_hat - z, reset flipped / listed slots, anchor := z, plus
// the primal residual partial on the raw x (admm.cpp:151-165).
template <int D>
__global__ __launch_bounds__(256, 2) void unpack_own_kernel(const float* __restrict__ x, size_t cap,
                                                         const uint32_t* __restrict__ rows,
                                                         const uint32_t* __restrict__ slots,
                                                         const uint8_t* __restrict__ first, size_t ns, size_t S,
                                                         const float* __restrict__ pack,
                                                         const uint32_t* __restrict__ owners,
                                                         float* __restrict__ zprev, uint8_t* __restrict__ in_zprev,
                                                         const float* __restrict__ rho,
                                                         const uint8_t* __restrict__ slot_reset, float alpha, int relax,
                                                         float* __restrict__ z, float* __restrict__ u,
                                                         double* __restrict__ scal) {
    __shared__ double s_red[8];
    const size_t j = blockIdx.x * static_cast<size_t>(blockDim.x) + threadIdx.x;
    double p2 = 0.0, d2 = 0.0, flips = 0.0;
    if (j < ns) {
        const uint32_t r = rows[j], s = slots[j];
        // every load of the row first (one round trip; the loop below then has no
        // load-after-store ordering to respect)
        float pk[D], zp[D], xv[D], za[D], uv[D];
#pragma unroll
        for (int c = 0; c < D; ++c) {
            pk[c] = pack[c * S + s];
            zp[c] = zprev[c * S + s];
            xv[c] = x[pidx(r, c, D - 11)];
            za[c] = z[c * ns + j];
            uv[c] = u[c * ns + j];
        }
        const bool lead = first[j] != 0;
        const float inv = 1.0f / static_cast<float>(owners[s]);
        const bool had = in_zprev[s] != 0;
        const bool flipped = pack[static_cast<size_t>(D) * S + s] > 0.f;
        const bool reset = flipped || (slot_reset && slot_reset[s]);
#pragma unroll
        for (int c = 0; c < D; ++c) {
            const float zv = pk[c] * inv;
            if (lead && had) {
                const double dv = static_cast<double>(rho[c]) * (static_cast<double>(zv) - zp[c]);
                d2 += dv * dv;
            }
            const float xh = relaxed(xv[c], za[c], alpha, relax != 0);
            const double dr = static_cast<double>(xv[c]) - zv;
            p2 += dr * dr;
            uv[c] = reset ? 0.f : uv[c] + (xh - zv);
            zp[c] = zv;
        }
#pragma unroll
        for (int c = 0; c < D; ++c) {
            zprev[c * S + s] = zp[c];
            z[c * ns + j] = zp[c];
            u[c * ns + j] = uv[c];
        }
        in_zprev[s] = 1;
        flips = lead && flipped ? 1.0 : 0.0;
    }
    block_add(p2, &scal[0], s_red);
    __syncthreads();
    block_add(d2, &scal[1], s_red);
    __syncthreads();
    block_add(flips, &scal[2], s_red);
}

// z for every slot from the reduced sums (consensus download, diagnostics).
__global__ void slots_from_sums_kernel(const float* __restrict__ pack, int D, size_t S,
                                       const uint32_t* __restrict__ owners, float* __restrict__ zslot) {
    const size_t s = blockIdx.x * static_cast<size_t>(blockDim.x) + threadIdx.x;
    if (s >= S) return;
    const float inv = 1.0f / static_cast<float>(owners[s]);
    for (int c = 0; c < D; ++c) zslot[c * S + s] = pack[c * S + s] * inv;
}

// Diagnostics: duals packed by slot for the dual-mean check (runtime.cpp:572-606),
// and +x / -x packed for max_disagreement (admm.cpp:219-243) under a MAX reduction.
__global__ void pack_duals_kernel(const float* __restrict__ u, int D, const uint32_t* __restrict__ slots, size_t ns,
                                  size_t S, float* __restrict__ pack) {
    const size_t j = blockIdx.x * static_cast<size_t>(blockDim.x) + threadIdx.x;
    if (j >= ns) return;
    const uint32_t s = slots[j];
    for (int c = 0; c < D; ++c) pack[c * S + s] = u[c * ns + j];
}

__global__ void pack_minmax_kernel(const float* __restrict__ x, size_t cap, int D, const uint32_t* __restrict__ rows,
                                   const uint32_t* __restrict__ slots, size_t ns, size_t S, float* __restrict__ pack) {
    const size_t j = blockIdx.x * static_cast<size_t>(blockDim.x) + threadIdx.x;
    if (j >= ns) return;
    const uint32_t r = rows[j], s = slots[j];
    for (int c = 0; c < D; ++c) {
        const float v = x[pidx(r, c, D - 11)];
        pack[c * S + s] = v;
        pack[(D + c) * S + s] = -v;
    }
}

__global__ void fill_kernel(float* p, size_t n, float v) {
    const size_t i = blockIdx.x * static_cast<size_t>(blockDim.x) + threadIdx.x;
    if (i < n) p[i] = v;
}

__global__ __launch_bounds__(256) void dual_linf_kernel(const float* __restrict__ pack, int D, size_t S,
                                                        const uint32_t* __restrict__ owners,
                                                        unsigned long long* __restrict__ out_bits) {
    const size_t s = blockIdx.x * static_cast<size_t>(blockDim.x) + threadIdx.x;
    double m = 0.0;
    if (s < S) {
        const double inv = 1.0 / owners[s];
        for (int c = 0; c < D; ++c) m = fmax(m, fabs(pack[c * S + s] * inv));
    }
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) m = fmax(m, __shfl_xor_sync(0xffffffffu, m, o));
    if ((threadIdx.x & 31) == 0 && m > 0) atomicMax(out_bits, static_cast<unsigned long long>(__double_as_longlong(m)));
}

__global__ __launch_bounds__(256) void spread_kernel(const float* __restrict__ pack, int D, size_t S,
                                                     const uint32_t* __restrict__ owners,
                                                     unsigned long long* __restrict__ out_bits) {
    const size_t s = blockIdx.x * static_cast<size_t>(blockDim.x) + threadIdx.x;
    double m = 0.0;
    if (s < S && owners[s] >= 2) {
        for (int c = 0; c < D; ++c) m = fmax(m, static_cast<double>(pack[c * S + s]) + pack[(D + c) * S + s]);
    }
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) m = fmax(m, __shfl_xor_sync(0xffffffffu, m, o));
    if ((threadIdx.x & 31) == 0 && m > 0) atomicMax(out_bits, static_cast<unsigned long long>(__double_as_longlong(m)));
}

inline unsigned grid_for(size_t n) { return static_cast<unsigned>((n + 255) / 256); }

__device__ __forceinline__ void rho_to_components(const double* rs, int fd, float* rho_dev) {
    const int D = 11 + fd;
    for (int k = 0; k < D; ++k) {
        double r = rs[3];                       // features
        if (k < kRot) r = rs[0];
        else if (k < kLs) r = rs[1];
        else if (k < kFeat) r = rs[2];
        else if (k == kFeat + fd) r = rs[4];    // opacity
        rho_dev[k] = static_cast<float>(r);
    }
}

// adapt_penalties (admm.cpp:200-217) from the reduced residuals: primal^2 in
// scal[0], dual^2 in scal[1] (identical on every rank after the reduction).
__global__ void adapt_kernel(const double* __restrict__ scal, double* __restrict__ rs, int fd,
                             float* __restrict__ rho_dev, bsg_adapt_args a) {
    if (threadIdx.x != 0 || blockIdx.x != 0) return;
    if (a.adaptive && a.iteration <= a.freeze_iteration) {
        const double primal = sqrt(scal[0]), dual = sqrt(scal[1]);
        double f = 1.0;
        if (primal > a.mu * dual)
            f = a.tau_inc;
        else if (dual > a.mu * primal)
            f = 1.0 / a.tau_dec;
        if (f != 1.0)
            for (int k = 0; k < 5; ++k) rs[k] *= f;
    }
    rho_to_components(rs, fd, rho_dev);
}

__global__ void rho_components_kernel(const double* __restrict__ rs, int fd, float* __restrict__ rho_dev) {
    if (threadIdx.x == 0 && blockIdx.x == 0) rho_to_components(rs, fd, rho_dev);
}

}  // namespace

void round_pack_q(Ctx* c) {
    BSG_CUDA(cudaMemsetAsync(c->qref, 0, 4 * c->n_slots * sizeof(float), c->stream));
    if (c->n_shared == 0) return;
    pack_q_kernel<<<grid_for(c->n_shared), 256, 0, c->stream>>>(c->x, c->fd, c->sh_rows, c->sh_slots, c->sh_first,
                                                                 c->n_shared, c->n_slots, c->qref);
    BSG_LAUNCHED(c);
}

void round_pack_main(Ctx* c, double alpha, bool relax) {
    BSG_CUDA(cudaMemsetAsync(c->pack, 0, (c->D + 1) * c->n_slots * sizeof(float), c->stream));
    if (c->n_shared == 0) return;
    auto kern = c->fd == 3 ? pack_main_kernel<14> : pack_main_kernel<23>;
    kern<<<grid_for(c->n_shared), 256, 0, c->stream>>>(c->x, c->cap, c->sh_rows, c->sh_slots, c->sh_first,
                                                       c->n_shared, c->n_slots, c->qref, c->zprev, c->in_zprev,
                                                       static_cast<float>(alpha), relax ? 1 : 0, c->pack);
    BSG_LAUNCHED(c);
}

// After the reduction of `pack`: z of the own slots, dual update, residual partials.
void round_unpack(Ctx* c, double alpha, bool relax, const uint8_t* reset_slots_dev, size_t n_reset, bool diag) {
    (void)n_reset;
    BSG_CUDA(cudaMemsetAsync(c->round_scalars, 0, 8 * sizeof(double), c->stream));
    if (c->n_shared > 0) {
        auto kern = c->fd == 3 ? unpack_own_kernel<14> : unpack_own_kernel<23>;
        kern<<<grid_for(c->n_shared), 256, 0, c->stream>>>(
            c->x, c->cap, c->sh_rows, c->sh_slots, c->sh_first, c->n_shared, c->n_slots, c->pack, c->slot_owners,
            c->zprev, c->in_zprev, c->rho_dev, reset_slots_dev ? c->slot_reset : nullptr, static_cast<float>(alpha),
            relax ? 1 : 0, c->z, c->u, c->round_scalars);
        BSG_LAUNCHED(c);
    }
    c->zslot_from_pack = true;
    if (diag) round_slots_from_sums(c);  // diagnostics reuse `pack`
}

// zslot (z of every slot) from the reduced sums still held in `pack`.
void round_slots_from_sums(Ctx* c) {
    if (!c->zslot_from_pack) return;
    if (c->n_slots > 0) {
        slots_from_sums_kernel<<<grid_for(c->n_slots), 256, 0, c->stream>>>(c->pack, c->D, c->n_slots, c->slot_owners,
                                                                            c->zslot);
        BSG_LAUNCHED(c);
    }
    c->zslot_from_pack = false;
}

// apply_broadcast with a host-provided z (trainer.cpp:168-223): zslot holds
// z for every slot; no flips, resets from slot_reset.
void round_apply_broadcast(Ctx* c, double alpha, bool relax, bool has_resets) {
    BSG_CUDA(cudaMemsetAsync(c->round_scalars, 0, 8 * sizeof(double), c->stream));
    BSG_CUDA(cudaMemsetAsync(c->pack + static_cast<size_t>(c->D) * c->n_slots, 0, c->n_slots * sizeof(float), c->stream));
    if (c->n_shared == 0) return;
    dual_update_kernel<<<grid_for(c->n_shared), 256, 0, c->stream>>>(
        c->x, c->cap, c->D, c->sh_rows, c->sh_slots, c->n_shared, c->n_slots, c->pack, c->zslot,
        has_resets ? c->slot_reset : nullptr, static_cast<float>(alpha), relax ? 1 : 0, c->z, c->u, c->round_scalars);
    BSG_LAUNCHED(c);
}

void round_pack_duals(Ctx* c) {
    BSG_CUDA(cudaMemsetAsync(c->pack, 0, c->D * c->n_slots * sizeof(float), c->stream));
    if (c->n_shared == 0) return;
    pack_duals_kernel<<<grid_for(c->n_shared), 256, 0, c->stream>>>(c->u, c->D, c->sh_slots, c->n_shared, c->n_slots,
                                                                     c->pack);
    BSG_LAUNCHED(c);
}

void round_dual_linf(Ctx* c) {
    if (c->n_slots == 0) return;
    dual_linf_kernel<<<grid_for(c->n_slots), 256, 0, c->stream>>>(
        c->pack, c->D, c->n_slots, c->slot_owners, reinterpret_cast<unsigned long long*>(&c->round_scalars[3]));
    BSG_LAUNCHED(c);
}

void round_pack_minmax(Ctx* c) {
    const size_t n = 2 * c->D * c->n_slots;
    if (n == 0) return;
    fill_kernel<<<grid_for(n), 256, 0, c->stream>>>(c->pack, n, -FLT_MAX);
    BSG_LAUNCHED(c);
    if (c->n_shared == 0) return;
    pack_minmax_kernel<<<grid_for(c->n_shared), 256, 0, c->stream>>>(c->x, c->cap, c->D, c->sh_rows, c->sh_slots,
                                                                      c->n_shared, c->n_slots, c->pack);
    BSG_LAUNCHED(c);
}

void round_spread(Ctx* c) {
    if (c->n_slots == 0) return;
    spread_kernel<<<grid_for(c->n_slots), 256, 0, c->stream>>>(
        c->pack, c->D, c->n_slots, c->slot_owners, reinterpret_cast<unsigned long long*>(&c->round_scalars[4]));
    BSG_LAUNCHED(c);
}

void round_adapt(Ctx* c, const bsg_adapt_args& a) {
    adapt_kernel<<<1, 32, 0, c->stream>>>(c->round_scalars, c->rho_state, c->fd, c->rho_dev, a);
    BSG_LAUNCHED(c);
}

void upload_rho(Ctx* c) {
    const double h[5] = {c->rho.rho_p, c->rho.rho_q, c->rho.rho_s, c->rho.rho_f, c->rho.rho_o};
    BSG_CUDA(cudaMemcpyAsync(c->rho_state, h, sizeof(h), cudaMemcpyHostToDevice, c->stream));
    rho_components_kernel<<<1, 32, 0, c->stream>>>(c->rho_state, c->fd, c->rho_dev);
    BSG_LAUNCHED(c);
    BSG_CUDA(cudaStreamSynchronize(c->stream));  // h lives on this stack frame
}

}  // namespace bsg
