// K17 densification: maybe_densify (trainer.cpp:301-385) and
// OptimizerState::remove_and_append (trainer.cpp:39-53) on the device.
//
// One classification pass decides every row in FP64 (compiled with
// --fmad=false, in the oracle's operation order): prune (opacity below the
// threshold), or for rows whose mean screen-space gradient reaches the
// threshold: clone (largest scale below split_scale), split in two (non-shared)
// or bud one child (shared: the id must stay alive across blocks). Two scans
// give every survivor its new row and every parent its first child slot; one
// scatter pass writes the compacted parameters and Adam moments (survivors in
// order, then the children in parent order, moments zero) into fresh row-major
// buffers. Ids, the removed / new id lists and the shared-row bookkeeping are
// updated on the host from the 1-byte action per row (one download per
// densification, every `interval` iterations).
#include <cmath>

#include "bsg_internal.cuh"

namespace bsg {
namespace {

enum : uint8_t { kActKeep = 0, kActPrune = 1, kActClone = 2, kActSplit = 3, kActBud = 4 };

struct DensifyParams {
    double grad_threshold, prune_opacity, split_scale, log_shrink;
};

// Offset of the children along the longest axis (trainer.cpp:327-331) and that
// axis' scale; quat_normalized / quat_to_rotation as math.hpp:25-44.
__device__ __forceinline__ double split_offset(const float* __restrict__ x, int fd, uint32_t i, double off[3]) {
    const double s[3] = {exp(static_cast<double>(x[pidx(i, kLs + 0, fd)])), exp(static_cast<double>(x[pidx(i, kLs + 1, fd)])),
                         exp(static_cast<double>(x[pidx(i, kLs + 2, fd)]))};
    int axis = 0;
    for (int a = 1; a < 3; ++a)
        if (s[a] > s[axis]) axis = a;  // Eigen maxCoeff: first maximum
    double w = x[pidx(i, kRot + 0, fd)], qx = x[pidx(i, kRot + 1, fd)], qy = x[pidx(i, kRot + 2, fd)],
           qz = x[pidx(i, kRot + 3, fd)];
    const double n = sqrt(((w * w + qx * qx) + qy * qy) + qz * qz);
    if (n == 0.0) {
        w = 1.0; qx = 0.0; qy = 0.0; qz = 0.0;
    } else {
        w = w / n; qx = qx / n; qy = qy / n; qz = qz / n;
    }
    double col[3];
    if (axis == 0) {
        col[0] = 1 - 2 * (qy * qy + qz * qz); col[1] = 2 * (qx * qy + w * qz); col[2] = 2 * (qx * qz - w * qy);
    } else if (axis == 1) {
        col[0] = 2 * (qx * qy - w * qz); col[1] = 1 - 2 * (qx * qx + qz * qz); col[2] = 2 * (qy * qz + w * qx);
    } else {
        col[0] = 2 * (qx * qz + w * qy); col[1] = 2 * (qy * qz - w * qx); col[2] = 1 - 2 * (qx * qx + qy * qy);
    }
    const double h = 0.5 * s[axis];
    for (int k = 0; k < 3; ++k) off[k] = col[k] * h;
    return s[axis];
}

__global__ __launch_bounds__(256) void densify_classify_kernel(const float* __restrict__ x, size_t cap, uint32_t n,
                                                               int fd, const float* __restrict__ m,
                                                               const float* __restrict__ v,
                                                               const uint32_t* __restrict__ sh_mask, DensifyParams p,
                                                               uint8_t* __restrict__ action,
                                                               uint32_t* __restrict__ keep,
                                                               uint32_t* __restrict__ nchild) {
    const uint32_t i = blockIdx.x * blockDim.x + threadIdx.x;
    if (i >= n) return;
    uint8_t act = kActKeep;
    const double o = 1.0 / (1.0 + exp(-static_cast<double>(x[pidx(i, kFeat + fd, fd)])));  // cloud.hpp:55
    if (o < p.prune_opacity) {
        act = kActPrune;
    } else if (const uint32_t seen = __float_as_uint(v[static_cast<size_t>(i) * row_stride(fd) + kMetaSlot])) {
        // densify statistics in the rows' metadata slot (bsg_internal.cuh)
        const double mean_grad = static_cast<double>(m[static_cast<size_t>(i) * row_stride(fd) + kMetaSlot]) / seen;
        if (!(mean_grad < p.grad_threshold)) {
            double off[3];
            const double smax = split_offset(x, fd, i, off);
            const bool shared = (sh_mask[i >> 5] >> (i & 31)) & 1u;
            act = smax >= p.split_scale ? (shared ? kActBud : kActSplit) : kActClone;
        }
    }
    action[i] = act;
    keep[i] = (act == kActPrune || act == kActSplit) ? 0u : 1u;
    nchild[i] = act == kActSplit ? 2u : ((act == kActClone || act == kActBud) ? 1u : 0u);
}

template <int D>
__global__ __launch_bounds__(256) void densify_scatter_kernel(const float* __restrict__ x, const float* __restrict__ m,
                                                              const float* __restrict__ v, size_t cap, uint32_t n,
                                                              const uint8_t* __restrict__ action,
                                                              const uint32_t* __restrict__ keep_pos,
                                                              const uint32_t* __restrict__ child_pos, uint32_t n_keep,
                                                              double log_shrink, float* __restrict__ nx,
                                                              float* __restrict__ nm, float* __restrict__ nv,
                                                              size_t ncap) {
    const uint32_t i = blockIdx.x * blockDim.x + threadIdx.x;
    if (i >= n) return;
    const uint8_t act = action[i];
    if (act != kActPrune && act != kActSplit) {
        const size_t r = keep_pos[i];
        constexpr int RS = row_stride(D - 11);
#pragma unroll
        for (int k = 0; k < RS; ++k) {  // whole rows (padding included)
            nx[r * RS + k] = x[static_cast<size_t>(i) * RS + k];
            nm[r * RS + k] = m[static_cast<size_t>(i) * RS + k];
            nv[r * RS + k] = v[static_cast<size_t>(i) * RS + k];
        }
    }
    if (act == kActKeep || act == kActPrune) return;
    double off[3] = {0.0, 0.0, 0.0};
    if (act != kActClone) split_offset(x, D - 11, i, off);
    const int count = act == kActSplit ? 2 : 1;
    for (int s = 0; s < count; ++s) {
        const size_t r = static_cast<size_t>(n_keep) + child_pos[i] + s;
        constexpr int fd = D - 11;
#pragma unroll
        for (int c = 0; c < D; ++c) {
            float val = x[pidx(i, c, fd)];
            if (act != kActClone) {
                if (c >= kPos && c < kPos + 3) {
                    const double o = s == 0 ? off[c - kPos] : -off[c - kPos];
                    val = static_cast<float>(static_cast<double>(val) + o);
                } else if (c >= kLs && c < kLs + 3) {
                    val = static_cast<float>(static_cast<double>(val) - log_shrink);
                }
            }
            nx[pidx(r, c, fd)] = val;
            nm[pidx(r, c, fd)] = 0.f;  // remove_and_append appends zero moments
            nv[pidx(r, c, fd)] = 0.f;
        }
    }
}

// z / u of the shared rows that survive: new[j'] = old[src[j']], D components.
__global__ void gather_cols_kernel(const float* __restrict__ in, size_t n_in, const uint32_t* __restrict__ src,
                                   size_t n_out, int D, float* __restrict__ out) {
    const size_t j = blockIdx.x * static_cast<size_t>(blockDim.x) + threadIdx.x;
    if (j >= n_out) return;
    const uint32_t s = src[j];
    for (int c = 0; c < D; ++c) out[c * n_out + j] = in[c * n_in + s];
}

template <typename T>
void realloc_dev(T** p, size_t count) {
    if (*p) cudaFree(*p);
    *p = nullptr;
    BSG_CUDA(cudaMalloc(p, std::max<size_t>(count, 1) * sizeof(T)));
}

}  // namespace

void maybe_densify(Ctx* c) {
    const bsg_densify_config& d = c->tcfg.densify;
    const uint64_t it = c->iteration;
    if (!d.enabled || it == 0) return;
    if (it % d.interval != 0 || it > d.stop_iteration) return;  // trainer.cpp:303-304
    const uint32_t n = static_cast<uint32_t>(c->n);
    if (n == 0) return;
    // an asynchronous round still in flight (bsg_consensus_round_async, then
    // bsg_train_steps across a densification iteration): densification
    // rewrites the anchor / dual rows the round writes, so it waits for the
    // round here; the round's result stays pending for bsg_consensus_wait
    if (c->round_pending) BSG_CUDA(cudaEventSynchronize(c->round_done));
    DensifyParams p;
    p.grad_threshold = d.grad_threshold;
    p.prune_opacity = d.prune_opacity;
    p.split_scale = d.split_scale_fraction * c->scene_extent;
    p.log_shrink = std::log(d.split_shrink);
    // per-row scratch of the step is free here: tiles (as bytes) holds the
    // actions, vrow[0/1] the flags, poff / vis_rows their exclusive scans
    uint8_t* action = reinterpret_cast<uint8_t*>(c->tiles);
    uint32_t* keep = c->vrow[0];
    uint32_t* nchild = c->vrow[1];
    uint32_t* keep_pos = c->poff;
    uint32_t* child_pos = c->vis_rows;
    materialize(c);
    densify_classify_kernel<<<(n + 255) / 256, 256, 0, c->stream>>>(c->x, c->cap, n, c->fd, c->m, c->v,
                                                                    c->sh_mask, p, action, keep, nchild);
    BSG_LAUNCHED(c);
    scan_exclusive_u32(c, keep, nullptr, keep_pos, n, &c->counters->dens_keep);
    scan_exclusive_u32(c, nchild, nullptr, child_pos, n, &c->counters->dens_children);
    std::vector<uint8_t> act(n);
    BSG_CUDA(cudaMemcpyAsync(act.data(), action, n, cudaMemcpyDeviceToHost, c->stream));
    BSG_CUDA(cudaMemcpyAsync(c->counters_host, c->counters, sizeof(StepCounters), cudaMemcpyDeviceToHost, c->stream));
    BSG_CUDA(cudaStreamSynchronize(c->stream));
    const uint32_t n_keep = c->counters_host->dens_keep, n_child = c->counters_host->dens_children;
    if (n_keep == n && n_child == 0) {
        reset_row_meta(c, static_cast<uint32_t>(c->adam_t), true);  // (every row is current: materialized above)
        return;
    }
    // ids (trainer.cpp:315-355): removal order is row order; children take
    // consecutive ids from the block's allocator in parent order
    if (c->alloc_next + n_child > c->alloc_end) throw Error{BSG_ERR_CAPACITY, "id allocator exhausted"};
    std::vector<uint64_t> ids;
    ids.reserve(static_cast<size_t>(n_keep) + n_child);
    std::vector<uint32_t> new_row(n, UINT32_MAX);
    for (uint32_t i = 0; i < n; ++i) {
        if (act[i] == kActPrune || act[i] == kActSplit) {
            c->removed_ids.push_back(c->ids[i]);
        } else {
            new_row[i] = static_cast<uint32_t>(ids.size());
            ids.push_back(c->ids[i]);
        }
    }
    for (uint32_t k = 0; k < n_child; ++k) {
        ids.push_back(c->alloc_next + k);
        c->new_ids.push_back(c->alloc_next + k);
    }
    c->alloc_next += n_child;
    // parameters and moments into fresh buffers (grown when needed)
    const size_t n_new = static_cast<size_t>(n_keep) + n_child;
    const size_t ncap = n_new <= c->cap ? c->cap : ((n_new + n_new / 4) + 31) / 32 * 32;
    float *nx = nullptr, *nm = nullptr, *nv = nullptr;
    BSG_CUDA(cudaMalloc(&nx, row_stride(c->fd) * ncap * sizeof(float)));
    BSG_CUDA(cudaMalloc(&nm, row_stride(c->fd) * ncap * sizeof(float)));
    BSG_CUDA(cudaMalloc(&nv, row_stride(c->fd) * ncap * sizeof(float)));
    // children rows are written slot by slot: their padding starts zeroed
    BSG_CUDA(cudaMemsetAsync(nx, 0, row_stride(c->fd) * ncap * sizeof(float), c->stream));
    BSG_CUDA(cudaMemsetAsync(nm, 0, row_stride(c->fd) * ncap * sizeof(float), c->stream));
    BSG_CUDA(cudaMemsetAsync(nv, 0, row_stride(c->fd) * ncap * sizeof(float), c->stream));
    if (c->fd == 3)
        densify_scatter_kernel<14><<<(n + 255) / 256, 256, 0, c->stream>>>(
            c->x, c->m, c->v, c->cap, n, action, keep_pos, child_pos, n_keep, p.log_shrink, nx, nm, nv, ncap);
    else
        densify_scatter_kernel<23><<<(n + 255) / 256, 256, 0, c->stream>>>(
            c->x, c->m, c->v, c->cap, n, action, keep_pos, child_pos, n_keep, p.log_shrink, nx, nm, nv, ncap);
    BSG_LAUNCHED(c);
    BSG_CUDA(cudaStreamSynchronize(c->stream));
    cudaFree(c->x);
    cudaFree(c->m);
    cudaFree(c->v);
    c->x = nx;
    c->m = nm;
    c->v = nv;
    if (ncap != c->cap) alloc_row_scratch(c, ncap);
    c->n = n_new;
    c->ids = std::move(ids);
    reset_row_meta(c, static_cast<uint32_t>(c->adam_t), true);  // every row current (materialized above; children new)
    // shared rows (trainer.cpp:360-371): pruned shared ids leave the consensus;
    // survivors move to their new rows (split never applies to shared rows)
    if (c->n_shared) {
        std::vector<uint32_t> src, rows, slots;
        std::vector<uint8_t> first;
        for (size_t j = 0; j < c->n_shared; ++j) {
            const uint32_t r = c->sh_rows_host[j];
            if (new_row[r] == UINT32_MAX) continue;
            src.push_back(static_cast<uint32_t>(j));
            rows.push_back(new_row[r]);
            slots.push_back(c->sh_slots_host[j]);
            first.push_back(c->sh_first_host[j]);
        }
        const size_t ns = rows.size();
        if (ns != c->n_shared) {
            uint32_t* src_dev = nullptr;
            float *nz = nullptr, *nu = nullptr;
            BSG_CUDA(cudaMalloc(&src_dev, std::max<size_t>(ns, 1) * sizeof(uint32_t)));
            BSG_CUDA(cudaMalloc(&nz, c->D * std::max<size_t>(ns, 1) * sizeof(float)));
            BSG_CUDA(cudaMalloc(&nu, c->D * std::max<size_t>(ns, 1) * sizeof(float)));
            if (ns) {
                BSG_CUDA(cudaMemcpyAsync(src_dev, src.data(), ns * 4, cudaMemcpyHostToDevice, c->stream));
                gather_cols_kernel<<<static_cast<unsigned>((ns + 255) / 256), 256, 0, c->stream>>>(c->z, c->n_shared,
                                                                                              src_dev, ns, c->D, nz);
                BSG_LAUNCHED(c);
                gather_cols_kernel<<<static_cast<unsigned>((ns + 255) / 256), 256, 0, c->stream>>>(c->u, c->n_shared,
                                                                                              src_dev, ns, c->D, nu);
                BSG_LAUNCHED(c);
            }
            BSG_CUDA(cudaStreamSynchronize(c->stream));
            cudaFree(src_dev);
            cudaFree(c->z);
            cudaFree(c->u);
            c->z = nz;
            c->u = nu;
        }
        realloc_dev(&c->sh_rows, ns);
        realloc_dev(&c->sh_slots, ns);
        realloc_dev(&c->sh_first, ns);
        if (ns) {
            BSG_CUDA(cudaMemcpyAsync(c->sh_rows, rows.data(), ns * 4, cudaMemcpyHostToDevice, c->stream));
            BSG_CUDA(cudaMemcpyAsync(c->sh_slots, slots.data(), ns * 4, cudaMemcpyHostToDevice, c->stream));
            BSG_CUDA(cudaMemcpyAsync(c->sh_first, first.data(), ns, cudaMemcpyHostToDevice, c->stream));
        }
        c->n_shared = ns;
        c->sh_rows_host = std::move(rows);
        c->sh_slots_host = std::move(slots);
        c->sh_first_host = std::move(first);
    }
    install_shared_masks(c);
}

}  // namespace bsg
