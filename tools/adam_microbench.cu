// Microbenchmark of dense-Adam streaming variants on B200 (not product code).
// Measures GB/s of: a 3-in/3-out pure stream (ceiling), the production-style
// per-component kernel, and variants with hoisted loads / interleaved m,v.
// build: nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o /tmp/amb tools/adam_microbench.cu
#include <cstdio>
#include <cstdint>
#include <cuda_runtime.h>

#include "../paper_2405_13943_b200/csrc/adam.cu"  // production kernels, same TU

#define CK(x) do { cudaError_t e = (x); if (e != cudaSuccess) { printf("%s: %s\n", #x, cudaGetErrorString(e)); return 1; } } while (0)

struct St { float lr, b1, b2, omb1, omb2, eps, ibc1, ibc2; };

__device__ __forceinline__ float upd(float x, float g, float& m, float& v, const St& s) {
    m = s.b1 * m + s.omb1 * g;
    v = s.b2 * v + s.omb2 * g * g;
    return x - s.lr * (m * s.ibc1) / (sqrtf(v * s.ibc2) + s.eps);
}

// pure stream: 3 float4 in, 3 float4 out per thread
__global__ void k_copy3(float4* x, float4* m, float4* v, size_t n4) {
    for (size_t i = blockIdx.x * (size_t)blockDim.x + threadIdx.x; i < n4; i += (size_t)gridDim.x * blockDim.x) {
        float4 a = x[i], b = m[i], c = v[i];
        a.x += 1.f; b.x += 1.f; c.x += 1.f;
        x[i] = a; m[i] = b; v[i] = c;
    }
}

// production-like: one quad per thread per component, visibility bit + conditional gradient load
template <int Q>
__global__ __launch_bounds__(256) void k_adam(float* x, float* m, float* v, const uint32_t* vis, const float* g,
                                              size_t cap, uint32_t n, St s) {
    const int c = blockIdx.y;
#pragma unroll
    for (int q = 0; q < Q; ++q) {
        const uint32_t r0 = 4 * ((blockIdx.x * blockDim.x + threadIdx.x) * Q + q);
        if (r0 >= n) break;
        const uint32_t vb = (vis[r0 >> 5] >> (r0 & 31)) & 0xfu;
        const size_t off = c * cap + r0;
        float4 x4 = *(float4*)(x + off), m4 = *(float4*)(m + off), v4 = *(float4*)(v + off);
        float gg[4];
        for (int r = 0; r < 4; ++r) gg[r] = ((vb >> r) & 1) ? g[off + r] : 0.f;
        x4.x = upd(x4.x, gg[0], m4.x, v4.x, s); x4.y = upd(x4.y, gg[1], m4.y, v4.y, s);
        x4.z = upd(x4.z, gg[2], m4.z, v4.z, s); x4.w = upd(x4.w, gg[3], m4.w, v4.w, s);
        *(float4*)(x + off) = x4; *(float4*)(m + off) = m4; *(float4*)(v + off) = v4;
    }
}

// hoisted: all loads of Q quads first, then gradients, then compute + stores
template <int Q>
__global__ __launch_bounds__(256) void k_adam_h(float* x, float* m, float* v, const uint32_t* vis, const float* g,
                                                size_t cap, uint32_t n, St s) {
    const int c = blockIdx.y;
    float4 x4[Q], m4[Q], v4[Q];
    uint32_t vb[Q];
    const uint32_t base = 4 * (blockIdx.x * blockDim.x * Q) ;
#pragma unroll
    for (int q = 0; q < Q; ++q) {
        const uint32_t r0 = base + 4 * (q * blockDim.x + threadIdx.x);  // quads strided by blockDim: coalesced per q
        const uint32_t rr = r0 < n ? r0 : 0;
        const size_t off = c * cap + rr;
        x4[q] = *(float4*)(x + off); m4[q] = *(float4*)(m + off); v4[q] = *(float4*)(v + off);
        vb[q] = r0 < n ? (vis[rr >> 5] >> (rr & 31)) & 0xfu : 0u;
    }
    float gg[Q][4];
#pragma unroll
    for (int q = 0; q < Q; ++q) {
        const uint32_t r0 = base + 4 * (q * blockDim.x + threadIdx.x);
        const size_t off = c * cap + r0;
        for (int r = 0; r < 4; ++r) gg[q][r] = ((vb[q] >> r) & 1) ? g[off + r] : 0.f;
    }
#pragma unroll
    for (int q = 0; q < Q; ++q) {
        const uint32_t r0 = base + 4 * (q * blockDim.x + threadIdx.x);
        if (r0 >= n) break;
        const size_t off = c * cap + r0;
        x4[q].x = upd(x4[q].x, gg[q][0], m4[q].x, v4[q].x, s); x4[q].y = upd(x4[q].y, gg[q][1], m4[q].y, v4[q].y, s);
        x4[q].z = upd(x4[q].z, gg[q][2], m4[q].z, v4[q].z, s); x4[q].w = upd(x4[q].w, gg[q][3], m4[q].w, v4[q].w, s);
        *(float4*)(x + off) = x4[q]; *(float4*)(m + off) = m4[q]; *(float4*)(v + off) = v4[q];
    }
}

// interleaved moments: mv[c][i/2] = {m_i, v_i, m_i+1, v_i+1}
template <int Q>
__global__ __launch_bounds__(256) void k_adam_mv(float* x, float* mv, const uint32_t* vis, const float* g,
                                                 size_t cap, uint32_t n, St s) {
    const int c = blockIdx.y;
    float4 x4[Q], a4[Q], b4[Q];
    uint32_t vb[Q];
    const uint32_t base = 4 * (blockIdx.x * blockDim.x * Q);
#pragma unroll
    for (int q = 0; q < Q; ++q) {
        const uint32_t r0 = base + 4 * (q * blockDim.x + threadIdx.x);
        const uint32_t rr = r0 < n ? r0 : 0;
        const size_t off = c * cap + rr;
        x4[q] = *(float4*)(x + off);
        a4[q] = *(float4*)(mv + 2 * off);
        b4[q] = *(float4*)(mv + 2 * off + 4);
        vb[q] = r0 < n ? (vis[rr >> 5] >> (rr & 31)) & 0xfu : 0u;
    }
    float gg[Q][4];
#pragma unroll
    for (int q = 0; q < Q; ++q) {
        const uint32_t r0 = base + 4 * (q * blockDim.x + threadIdx.x);
        const size_t off = c * cap + r0;
        for (int r = 0; r < 4; ++r) gg[q][r] = ((vb[q] >> r) & 1) ? g[off + r] : 0.f;
    }
#pragma unroll
    for (int q = 0; q < Q; ++q) {
        const uint32_t r0 = base + 4 * (q * blockDim.x + threadIdx.x);
        if (r0 >= n) break;
        const size_t off = c * cap + r0;
        x4[q].x = upd(x4[q].x, gg[q][0], a4[q].x, a4[q].y, s); x4[q].y = upd(x4[q].y, gg[q][1], a4[q].z, a4[q].w, s);
        x4[q].z = upd(x4[q].z, gg[q][2], b4[q].x, b4[q].y, s); x4[q].w = upd(x4[q].w, gg[q][3], b4[q].z, b4[q].w, s);
        *(float4*)(x + off) = x4[q];
        *(float4*)(mv + 2 * off) = a4[q];
        *(float4*)(mv + 2 * off + 4) = b4[q];
    }
}

// quaternion group: R rows per thread (vector width R), 4 components, then canonicalise
template <int R> struct Vec;
template <> struct Vec<1> { using T = float; };
template <> struct Vec<2> { using T = float2; };
template <> struct Vec<4> { using T = float4; };
template <int R, int MODE = 0>
__global__ __launch_bounds__(256) void k_rot(float* x, float* m, float* v, const uint32_t* vis, const float* g,
                                             size_t cap, uint32_t n, St s) {
    using V = typename Vec<R>::T;
    const uint32_t r0 = R * (blockIdx.x * blockDim.x + threadIdx.x);
    if (r0 >= n) return;
    const uint32_t vb = (vis[r0 >> 5] >> (r0 & 31)) & ((1u << R) - 1u);
    float xs[4][R], ms[4][R], vs[4][R];
#pragma unroll
    for (int k = 0; k < 4; ++k) {
        const size_t off = (3 + k) * cap + r0;
        V a = *(V*)(x + off), b = *(V*)(m + off), c = *(V*)(v + off);
        const float* pa = (const float*)&a; const float* pb = (const float*)&b; const float* pc = (const float*)&c;
#pragma unroll
        for (int r = 0; r < R; ++r) { xs[k][r] = pa[r]; ms[k][r] = pb[r]; vs[k][r] = pc[r]; }
    }
#pragma unroll
    for (int k = 0; k < 4; ++k) {
        const size_t off = (3 + k) * cap + r0;
#pragma unroll
        for (int r = 0; r < R; ++r) {
            const float gg = ((vb >> r) & 1) ? g[off + r] : 0.f;
            if (MODE == 2) { xs[k][r] += 1.f; ms[k][r] += gg; vs[k][r] += 1.f; continue; }
            xs[k][r] = upd(xs[k][r], gg, ms[k][r], vs[k][r], s);
        }
    }
#pragma unroll
    for (int r = 0; r < R; ++r) {
        if (MODE != 0) break;
        float qw = xs[0][r], qx = xs[1][r], qy = xs[2][r], qz = xs[3][r];
        const float qn = sqrtf(qw * qw + qx * qx + qy * qy + qz * qz);
        if (qn == 0.f) { qw = 1.f; qx = qy = qz = 0.f; } else { qw /= qn; qx /= qn; qy /= qn; qz /= qn; }
        if (qw < 0.f) { qw = -qw; qx = -qx; qy = -qy; qz = -qz; }
        xs[0][r] = qw; xs[1][r] = qx; xs[2][r] = qy; xs[3][r] = qz;
    }
#pragma unroll
    for (int k = 0; k < 4; ++k) {
        const size_t off = (3 + k) * cap + r0;
        V a, b, c;
        float* pa = (float*)&a; float* pb = (float*)&b; float* pc = (float*)&c;
#pragma unroll
        for (int r = 0; r < R; ++r) { pa[r] = xs[k][r]; pb[r] = ms[k][r]; pc[r] = vs[k][r]; }
        *(V*)(x + off) = a; *(V*)(m + off) = b; *(V*)(v + off) = c;
    }
}

int main() {
    const uint32_t n = 2000000;
    const size_t cap = (n + 31) / 32 * 32;
    const int D = 10;
    float *x, *m, *v, *g, *mv;
    uint32_t* vis;
    CK(cudaMalloc(&x, D * cap * 4)); CK(cudaMalloc(&m, D * cap * 4)); CK(cudaMalloc(&v, D * cap * 4));
    CK(cudaMalloc(&g, D * cap * 4)); CK(cudaMalloc(&mv, 2 * D * cap * 4)); CK(cudaMalloc(&vis, cap / 8));
    CK(cudaMemset(x, 0, D * cap * 4)); CK(cudaMemset(m, 0, D * cap * 4)); CK(cudaMemset(v, 0, D * cap * 4));
    CK(cudaMemset(g, 0, D * cap * 4)); CK(cudaMemset(mv, 0, 2 * D * cap * 4));
    // ~10% visible, random bits
    {
        uint32_t* h = new uint32_t[cap / 32];
        uint64_t st = 12345;
        for (size_t w = 0; w < cap / 32; ++w) {
            uint32_t b = 0;
            for (int k = 0; k < 32; ++k) { st = st * 6364136223846793005ull + 1442695040888963407ull; if ((st >> 33) % 10 == 0) b |= 1u << k; }
            h[w] = b;
        }
        CK(cudaMemcpy(vis, h, cap / 8, cudaMemcpyHostToDevice));
        delete[] h;
    }
    St s{1e-3f, 0.9f, 0.999f, 0.1f, 0.001f, 1e-8f, 10.f, 1000.f};
    float* flush; CK(cudaMalloc(&flush, 256 << 20));
    cudaEvent_t e0, e1; cudaEventCreate(&e0); cudaEventCreate(&e1);
    const double bytes = 6.0 * 4 * D * (double)n;  // x,m,v read + write
    auto run = [&](const char* name, auto launch) {
        float best = 1e9, sum = 0; int reps = 20;
        for (int it = 0; it < reps + 3; ++it) {
            cudaMemsetAsync(flush, it, 256 << 20);
            cudaEventRecord(e0);
            launch();
            cudaEventRecord(e1);
            cudaEventSynchronize(e1);
            float ms; cudaEventElapsedTime(&ms, e0, e1);
            if (it >= 3) { best = ms < best ? ms : best; sum += ms; }
        }
        printf("%-28s best %7.1f us  mean %7.1f us  %6.0f GB/s (best)\n", name, best * 1e3, sum / reps * 1e3, bytes / (best * 1e-3) / 1e9);
    };
    const size_t n4 = D * cap / 4;
    for (int blocks : {148 * 4, 148 * 8, 148 * 16, 148 * 32}) {
        char nm[64]; snprintf(nm, 64, "copy3 grid %d", blocks);
        run(nm, [&] { k_copy3<<<blocks, 256>>>((float4*)x, (float4*)m, (float4*)v, n4); });
    }
    run("adam Q=1", [&] { k_adam<1><<<dim3((n + 1023) / 1024, D), 256>>>(x, m, v, vis, g, cap, n, s); });
    run("adam Q=2", [&] { k_adam<2><<<dim3((n + 2047) / 2048, D), 256>>>(x, m, v, vis, g, cap, n, s); });
    run("adam hoisted Q=2", [&] { k_adam_h<2><<<dim3((n + 2047) / 2048, D), 256>>>(x, m, v, vis, g, cap, n, s); });
    run("adam hoisted Q=4", [&] { k_adam_h<4><<<dim3((n + 4095) / 4096, D), 256>>>(x, m, v, vis, g, cap, n, s); });
    run("adam mv Q=2", [&] { k_adam_mv<2><<<dim3((n + 2047) / 2048, D), 256>>>(x, mv, vis, g, cap, n, s); });
    run("adam mv Q=4", [&] { k_adam_mv<4><<<dim3((n + 4095) / 4096, D), 256>>>(x, mv, vis, g, cap, n, s); });
    const double rbytes = 6.0 * 4 * 4 * (double)n;
    auto runr = [&](const char* name, auto launch) {
        float best = 1e9;
        for (int it = 0; it < 23; ++it) {
            cudaMemsetAsync(flush, it, 256 << 20);
            cudaEventRecord(e0); launch(); cudaEventRecord(e1); cudaEventSynchronize(e1);
            float ms; cudaEventElapsedTime(&ms, e0, e1);
            if (it >= 3) best = ms < best ? ms : best;
        }
        printf("%-28s best %7.1f us  %6.0f GB/s\n", name, best * 1e3, rbytes / (best * 1e-3) / 1e9);
    };
    runr("rot R=1", [&] { k_rot<1, 0><<<(n + 255) / 256, 256>>>(x, m, v, vis, g, cap, n, s); });
    runr("rot R=4", [&] { k_rot<4, 0><<<(n + 1023) / 1024, 256>>>(x, m, v, vis, g, cap, n, s); });
    runr("rot R=1 no normalise", [&] { k_rot<1, 1><<<(n + 255) / 256, 256>>>(x, m, v, vis, g, cap, n, s); });
    // production kernels on 14 components
    {
        float *X, *M, *Vv, *G;
        const int DD = 14;
        CK(cudaMalloc(&X, DD * cap * 4)); CK(cudaMalloc(&M, DD * cap * 4)); CK(cudaMalloc(&Vv, DD * cap * 4));
        CK(cudaMalloc(&G, DD * cap * 4));
        CK(cudaMemset(X, 0, DD * cap * 4)); CK(cudaMemset(M, 0, DD * cap * 4)); CK(cudaMemset(Vv, 0, DD * cap * 4));
        CK(cudaMemset(G, 0, DD * cap * 4));
        bsg::AdamStep st{};
        for (int k = 0; k < 23; ++k) st.lr[k] = 1e-3f;
        float* rho_d; CK(cudaMalloc(&rho_d, 23 * 4)); CK(cudaMemset(rho_d, 0, 23 * 4));
        st.b1 = 0.9f; st.b2 = 0.999f; st.omb1 = 0.1f; st.omb2 = 0.001f; st.eps = 1e-8f; st.inv_bc1 = 10.f; st.inv_bc2 = 1000.f;
        st.has_anchor = 0;
        double* pen; CK(cudaMalloc(&pen, 8));
        const double b10 = 6.0 * 4 * 10 * (double)n, b4 = 6.0 * 4 * 4 * (double)n;
        auto runp = [&](const char* name, double bytes, auto launch) {
            float best = 1e9;
            for (int it = 0; it < 23; ++it) {
                cudaMemsetAsync(flush, it, 256 << 20);
                cudaEventRecord(e0); launch(); cudaEventRecord(e1); cudaEventSynchronize(e1);
                float ms; cudaEventElapsedTime(&ms, e0, e1);
                if (it >= 3) best = ms < best ? ms : best;
            }
            printf("%-28s best %7.1f us  %6.0f GB/s\n", name, best * 1e3, bytes / (best * 1e-3) / 1e9);
        };
        runp("prod scalar (10 comps)", b10, [&] {
            bsg::adam_kernel<1><<<dim3((n + 1023) / 1024, 10), 256>>>(X, M, Vv, cap, n, vis, vis, G, nullptr, nullptr,
                                                                            nullptr, nullptr, 0, rho_d, st, pen); });
        runp("prod rot (4 comps)", b4, [&] {
            bsg::adam_rot_kernel<<<(n + 255) / 256, 256>>>(X, M, Vv, cap, n, vis, vis, G, nullptr, nullptr,
                                                                          nullptr, nullptr, 0, rho_d, st, pen); });
        runp("prod both", b10 + b4, [&] {
            bsg::adam_kernel<1><<<dim3((n + 1023) / 1024, 10), 256>>>(X, M, Vv, cap, n, vis, vis, G, nullptr, nullptr,
                                                                            nullptr, nullptr, 0, rho_d, st, pen);
            bsg::adam_rot_kernel<<<(n + 255) / 256, 256>>>(X, M, Vv, cap, n, vis, vis, G, nullptr, nullptr,
                                                                          nullptr, nullptr, 0, rho_d, st, pen); });
    }
    CK(cudaDeviceSynchronize());
    return 0;
}
