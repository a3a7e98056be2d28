// tsw_kernels.cuh — sm_100a kernels of the leapfrog hot path (DESIGN.md §1 rows S1–S6).
//
// Written from PAPER.md and DESIGN.md's readings; shares nothing with oracle/.
// Arithmetic of the stepper uses the __d*_rn / __f*_rn intrinsics (never contracted into FMA)
// in the canonical tree of DESIGN.md §2, so every node's value is the same IEEE operation
// sequence as any other implementation of that tree (R19).  The library is also built with
// --fmad=false.
#pragma once

#include <cuda_runtime.h>
#include <cooperative_groups.h>
#include <stdint.h>
#include <climits>

#include <type_traits>

namespace tsw {

// PAPER.md §3.1, "c ≃ 2.2523 to get ∫φ = 1" (R4: 1/∫_{-1}^{1} e^{1/(x²−1)} dx).
constexpr double TSW_MOLLIFIER_C = 2.252283621043581;

enum CoeffMode { MODE_LINE = 0, MODE_DENSE = 1 };

// ------------------------------------------------------------------------------------------
// rounding-explicit arithmetic (no contraction)
// ------------------------------------------------------------------------------------------
__device__ __forceinline__ double r_add(double a, double b) { return __dadd_rn(a, b); }
__device__ __forceinline__ double r_sub(double a, double b) { return __dsub_rn(a, b); }
__device__ __forceinline__ double r_mul(double a, double b) { return __dmul_rn(a, b); }
__device__ __forceinline__ float r_add(float a, float b) { return __fadd_rn(a, b); }
__device__ __forceinline__ float r_sub(float a, float b) { return __fsub_rn(a, b); }
__device__ __forceinline__ float r_mul(float a, float b) { return __fmul_rn(a, b); }
// fl(2u − p) in one instruction: 2u is exact (a doubling), so the fused form rounds exactly like
// the canonical r_sub(r_mul(2, u), p) — bit-identical (R19), one FP op fewer per update
__device__ __forceinline__ double twice_minus(double u, double p) { return __fma_rn(2.0, u, -p); }
__device__ __forceinline__ float twice_minus(float u, float p) { return __fmaf_rn(2.0f, u, -p); }

template <typename T> struct Vec16;
template <> struct Vec16<double> { using type = double2; static constexpr int N = 2; };
template <> struct Vec16<float> { using type = float4; static constexpr int N = 4; };
// two-element vectors (the temporally blocked kernel uses 2 columns per thread in both precisions)
template <typename T> struct Vec2;
template <> struct Vec2<double> { using type = double2; };
template <> struct Vec2<float> { using type = float2; };

template <typename T>
__device__ __forceinline__ void vload(const T* __restrict__ p, T (&v)[Vec16<T>::N]) {
    using VT = typename Vec16<T>::type;
    VT x = __ldg(reinterpret_cast<const VT*>(p));
    const T* e = reinterpret_cast<const T*>(&x);
#pragma unroll
    for (int k = 0; k < Vec16<T>::N; ++k) v[k] = e[k];
}

// streaming load (read once: u^{n-1})
template <typename T>
__device__ __forceinline__ void vload_cs(const T* p, T (&v)[Vec16<T>::N]) {
    using VT = typename Vec16<T>::type;
    VT x = __ldcs(reinterpret_cast<const VT*>(p));
    const T* e = reinterpret_cast<const T*>(&x);
#pragma unroll
    for (int k = 0; k < Vec16<T>::N; ++k) v[k] = e[k];
}

template <typename T>
__device__ __forceinline__ void vstore(T* p, const T (&v)[Vec16<T>::N]) {
    using VT = typename Vec16<T>::type;
    VT x;
    T* e = reinterpret_cast<T*>(&x);
#pragma unroll
    for (int k = 0; k < Vec16<T>::N; ++k) e[k] = v[k];
    __stcs(reinterpret_cast<VT*>(p), x);
}

// One node of S2/S3 (DESIGN.md §2 canonical tree):
//   lap = (c1r·(u_{i+1}−u_i) − c1l·(u_i−u_{i−1})) + (c2u·(u_{j+1}−u_j) − c2d·(u_j−u_{j−1}))
//   START: u¹ = (u⁰ + dt·v) + ½·lap        else: u^{n+1} = (2u^n − u^{n−1}) + lap
template <typename T, bool START, bool TWO_D>
__device__ __forceinline__ T node_update(T u, T ul, T ur, T ud, T uu, T p, T c1l, T c1r, T c2d, T c2u,
                                         T dtT) {
    T dxp = r_sub(ur, u);
    T dxm = r_sub(u, ul);
    T lap = r_sub(r_mul(c1r, dxp), r_mul(c1l, dxm));
    if (TWO_D) {
        T dyp = r_sub(uu, u);
        T dym = r_sub(u, ud);
        lap = r_add(lap, r_sub(r_mul(c2u, dyp), r_mul(c2d, dym)));
    }
    if (START) return r_add(r_add(u, r_mul(dtT, p)), r_mul((T)0.5, lap));
    return r_add(twice_minus(u, p), lap);
}

// ------------------------------------------------------------------------------------------
// S2/S3: 2D stencil, warp column strips marching in y (register-rotated u^{n}[j−1..j+1])
// ------------------------------------------------------------------------------------------
// Storage: fields [B][rows_alloc][pitch]; storage row s ↔ global row g = r0 + s − 1 (s = 0 and
// s = ny_local + 1 are ghost rows).  pitch is a multiple of 32·V elements.
// Coefficients: LINE  c1[b][cpitch] (face i+1/2), c2[b] scalar;
//               DENSE c1[b][rows_alloc][pitch] (face (i+1/2, s)), c2[b][rows_alloc][pitch]
//               where c2 row s = face between storage rows s−1 and s.
template <typename T>
struct StepArgs {
    const T* __restrict__ ucur;  // u^n
    T* __restrict__ uprev;       // u^{n−1} in, u^{n+1} out (in place; START: u1 in, u¹ out)
    const T* __restrict__ c1;
    const T* __restrict__ c2;
    int64_t pitch;         // elements per stored row
    int64_t mstride;       // elements per member (rows_alloc·pitch)
    int64_t cstride1;      // elements per member of c1
    int64_t cstride2;      // elements per member of c2
    int64_t nx;            // global nodes per row
    int32_t s_lo, s_hi;    // storage rows updated: [s_lo, s_hi)
    int32_t rows_per_item; // R
    int32_t chunks;        // ceil((s_hi − s_lo)/R)
    int64_t strips;        // pitch / (32·V)
    int64_t items;         // strips · chunks · B
    T dtT;
};

template <typename T, int MODE, bool START>
__global__ void __launch_bounds__(256) k_step2d(const StepArgs<T> a) {
    constexpr int V = Vec16<T>::N;
    const int lane = threadIdx.x & 31;
    const int64_t gwarp = (int64_t(blockIdx.x) * blockDim.x + threadIdx.x) >> 5;
    const int64_t nwarps = (int64_t(gridDim.x) * blockDim.x) >> 5;

    for (int64_t item = gwarp; item < a.items; item += nwarps) {
        const int64_t strip = item % a.strips;
        const int64_t rest = item / a.strips;
        const int chunk = int(rest % a.chunks);
        const int b = int(rest / a.chunks);
        const int64_t cs = strip * 32 * V;       // first column of the strip
        const int64_t col = cs + int64_t(lane) * V;
        const int s0 = a.s_lo + chunk * a.rows_per_item;
        const int s1 = min(s0 + a.rows_per_item, a.s_hi);
        const T* __restrict__ ub = a.ucur + b * a.mstride;
        T* __restrict__ pb = a.uprev + b * a.mstride;
        const bool has_l = (lane == 0) && (cs > 0);
        const bool has_r = (lane == 31) && (cs + 32 * V < a.pitch);

        bool interior[V];
#pragma unroll
        for (int k = 0; k < V; ++k) interior[k] = (col + k >= 1) && (col + k <= a.nx - 2);

        // LINE coefficients are row-invariant: load once per item (c2 per node column).
        T c1r[V], c1l[V], c2v[V];
        if (MODE == MODE_LINE) {
            const T* c1b = a.c1 + b * a.cstride1;
            vload(c1b + col, c1r);
            T left = __shfl_up_sync(0xffffffffu, c1r[V - 1], 1);
            if (lane == 0) left = has_l ? c1b[cs - 1] : (T)0;
            c1l[0] = left;
#pragma unroll
            for (int k = 1; k < V; ++k) c1l[k] = c1r[k - 1];
            vload(a.c2 + b * a.cstride2 + col, c2v);
        }

        // register window: up = row s−1, cu = row s, dn = row s+1 ; pv = u^{n−1} row s
        T up[V], cu[V], dn[V], pv[V];
        T hl_c = 0, hr_c = 0, hl_d = 0, hr_d = 0;
        vload(ub + (s0 - 1) * a.pitch + col, up);
        vload(ub + s0 * a.pitch + col, cu);
        if (has_l) hl_c = ub[s0 * a.pitch + cs - 1];
        if (has_r) hr_c = ub[s0 * a.pitch + cs + 32 * V];
        if (s0 < s1) {
            vload(ub + (s0 + 1) * a.pitch + col, dn);
            vload_cs(pb + s0 * a.pitch + col, pv);
            if (has_l) hl_d = ub[(s0 + 1) * a.pitch + cs - 1];
            if (has_r) hr_d = ub[(s0 + 1) * a.pitch + cs + 32 * V];
        }
        // DENSE: c2 face below row s (= c2 row s) carried between iterations
        T c2lo[V];
        if (MODE == MODE_DENSE) vload(a.c2 + b * a.cstride2 + s0 * a.pitch + col, c2lo);

        for (int s = s0; s < s1; ++s) {
            // prefetch row s+2 of u^n and row s+1 of u^{n−1}
            T dn2[V], pv2[V];
            T hl_d2 = 0, hr_d2 = 0;
            const bool more = (s + 1 < s1);
            if (more) {
                vload(ub + (s + 2) * a.pitch + col, dn2);
                vload_cs(pb + (s + 1) * a.pitch + col, pv2);
                if (has_l) hl_d2 = ub[(s + 2) * a.pitch + cs - 1];
                if (has_r) hr_d2 = ub[(s + 2) * a.pitch + cs + 32 * V];
            }
            T c1r_d[V], c1l_d[V], c2hi[V];
            if (MODE == MODE_DENSE) {
                const T* c1row = a.c1 + b * a.cstride1 + s * a.pitch;
                vload(c1row + col, c1r_d);
                T left = __shfl_up_sync(0xffffffffu, c1r_d[V - 1], 1);
                if (lane == 0) left = has_l ? c1row[cs - 1] : (T)0;
                c1l_d[0] = left;
#pragma unroll
                for (int k = 1; k < V; ++k) c1l_d[k] = c1r_d[k - 1];
                vload(a.c2 + b * a.cstride2 + (s + 1) * a.pitch + col, c2hi);
            }
            // x neighbours across lanes
            T left = __shfl_up_sync(0xffffffffu, cu[V - 1], 1);
            T right = __shfl_down_sync(0xffffffffu, cu[0], 1);
            if (lane == 0) left = hl_c;
            if (lane == 31) right = hr_c;
            T out[V];
#pragma unroll
            for (int k = 0; k < V; ++k) {
                T ul = (k == 0) ? left : cu[k - 1];
                T ur = (k == V - 1) ? right : cu[k + 1];
                T l1 = (MODE == MODE_LINE) ? c1l[k] : c1l_d[k];
                T r1 = (MODE == MODE_LINE) ? c1r[k] : c1r_d[k];
                T d2 = (MODE == MODE_LINE) ? c2v[k] : c2lo[k];
                T u2 = (MODE == MODE_LINE) ? c2v[k] : c2hi[k];
                T v = node_update<T, START, true>(cu[k], ul, ur, up[k], dn[k], pv[k], l1, r1, d2, u2, a.dtT);
                out[k] = interior[k] ? v : (T)0;
            }
            vstore(pb + s * a.pitch + col, out);
            // rotate
#pragma unroll
            for (int k = 0; k < V; ++k) {
                up[k] = cu[k];
                cu[k] = dn[k];
                if (more) {
                    dn[k] = dn2[k];
                    pv[k] = pv2[k];
                }
                if (MODE == MODE_DENSE) c2lo[k] = c2hi[k];
            }
            hl_c = hl_d;
            hr_c = hr_d;
            hl_d = hl_d2;
            hr_d = hr_d2;
        }
    }
}

// ------------------------------------------------------------------------------------------
// S2/S3: 2D stencil, CTA-wide TMA bulk-copy row pipeline (the production kernel on sm_100a)
// ------------------------------------------------------------------------------------------
// Same per-node arithmetic as k_step2d.  A CTA owns a strip of WC = NC·32·V columns (4 KB of a
// row in either precision) and marches down a chunk of rows.  A dedicated producer warp streams
// rows into a ring of D shared-memory stages with cp.async.bulk (TMA 1D bulk copies, SASS UBLKCP;
// one ≈4 KB request per row and field, so the TMA request rate is no limit), completing each
// stage on a "full" mbarrier (expect_tx bytes); the NC consumer warps arrive on an "empty"
// mbarrier when a stage can be refilled.  The vertical window u^n[s−1], u^n[s], u^n[s+1] lives
// in registers; horizontal neighbours come from the centre row's stage (16-byte halo on each
// side, so every thread reads its left/right neighbour the same way).
//
// The CTA walks a STREAM of stages over its items (strip, row chunk, member); item rows [s0, s1)
// are the stages t = 0 .. (s1 − s0) + 1 and
//   stage t loads u^n row r = s0 − 1 + t (+ halos)            (DENSE: + c2 row r when t ≥ 1)
//            and, when t ≥ 2, u^{n−1} row r − 1               (DENSE: + c1 row r − 1 + halos)
//   and emits output row r − 1.  The producer runs up to D stages ahead, across items.
__device__ __forceinline__ uint32_t smem_u32(const void* p) { return (uint32_t)__cvta_generic_to_shared(p); }

__device__ __forceinline__ void mbar_init(uint64_t* bar, uint32_t count) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(bar)), "r"(count) : "memory");
}
__device__ __forceinline__ void fence_barrier_init() {
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
}
__device__ __forceinline__ void fence_proxy_async_smem() {
    asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
}
__device__ __forceinline__ void mbar_arrive_expect_tx(uint64_t* bar, uint32_t bytes) {
    asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(bar)), "r"(bytes) : "memory");
}
__device__ __forceinline__ void mbar_arrive(uint64_t* bar) {
    asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(smem_u32(bar)) : "memory");
}
__device__ __forceinline__ void bulk_g2s(void* dst, const void* src, uint32_t bytes, uint64_t* bar) {
    asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(
                     smem_u32(dst)),
                 "l"(src), "r"(bytes), "r"(smem_u32(bar))
                 : "memory");
}
__device__ __forceinline__ bool mbar_try_wait(uint64_t* bar, uint32_t parity) {
    uint32_t ok;
    asm volatile(
        "{\n\t.reg .pred p;\n\t"
        "mbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2;\n\t"
        "selp.u32 %0, 1, 0, p;\n\t}"
        : "=r"(ok)
        : "r"(smem_u32(bar)), "r"(parity)
        : "memory");
    return ok != 0;
}
__device__ __forceinline__ void mbar_wait(uint64_t* bar, uint32_t parity) {
    while (!mbar_try_wait(bar, parity)) {
    }
}

// one lane of the (fully active) warp returns true
__device__ __forceinline__ bool elect_one() {
    uint32_t pred = 0;
    asm volatile(
        "{\n\t.reg .pred p;\n\t"
        "elect.sync _|p, 0xffffffff;\n\t"
        "selp.u32 %0, 1, 0, p;\n\t}"
        : "=r"(pred));
    return pred != 0;
}

constexpr int TMA_NC = 8;  // consumer warps per CTA (+1 producer warp)

template <typename T>
struct TmaGeom {
    static constexpr int V = Vec16<T>::N;      // elements per thread
    static constexpr int H = 16 / sizeof(T);   // halo elements (16 bytes) on each side
    static constexpr int WC = TMA_NC * 32 * V; // strip width in elements (4 KB)
    static constexpr int WH = WC + 2 * H;      // strip + halos
};

template <typename T, int MODE>
__host__ __device__ constexpr int tma_slot_bytes() {
    return int(sizeof(T)) * (TmaGeom<T>::WH + TmaGeom<T>::WC + (MODE == MODE_DENSE ? TmaGeom<T>::WH + TmaGeom<T>::WC : 0));
}

template <typename T>
__device__ __forceinline__ void lds_vec(const T* p, T (&v)[Vec16<T>::N]) {
    using VT = typename Vec16<T>::type;
    VT x = *reinterpret_cast<const VT*>(p);
    const T* e = reinterpret_cast<const T*>(&x);
#pragma unroll
    for (int k = 0; k < Vec16<T>::N; ++k) v[k] = e[k];
}

// a.strips counts WC-wide strips for this kernel
template <typename T, int MODE, bool START>
__global__ void __launch_bounds__((TMA_NC + 1) * 32) k_step2d_tma(const StepArgs<T> a, int depth) {
    using G = TmaGeom<T>;
    constexpr int V = G::V, H = G::H, WC = G::WC, WH = G::WH;
    constexpr int SLOT = tma_slot_bytes<T, MODE>();
    extern __shared__ __align__(128) unsigned char smem[];
    uint64_t* full = reinterpret_cast<uint64_t*>(smem + size_t(depth) * SLOT);
    uint64_t* empty = full + depth;
    const int warp = threadIdx.x >> 5;
    const int lane = threadIdx.x & 31;

    if (threadIdx.x == 0) {
        for (int k = 0; k < depth; ++k) {
            mbar_init(&full[k], 1);
            mbar_init(&empty[k], TMA_NC);
        }
        fence_barrier_init();
    }
    __syncthreads();

    auto item_geom = [&](int64_t item, int64_t& cs, int& s0, int& s1, int& b) {
        const int64_t strip = item % a.strips;
        const int64_t rest = item / a.strips;
        const int chunk = int(rest % a.chunks);
        b = int(rest / a.chunks);
        cs = strip * WC;
        s0 = a.s_lo + chunk * a.rows_per_item;
        s1 = min(s0 + a.rows_per_item, a.s_hi);
    };

    if (warp == TMA_NC) {
        // ------------------------------ producer warp ------------------------------
        if (lane != 0) return;
        int64_t it = 0;
        for (int64_t item = blockIdx.x; item < a.items; item += gridDim.x) {
            int64_t cs;
            int s0, s1, b;
            item_geom(item, cs, s0, s1, b);
            const int L = s1 - s0 + 2;
            const T* ub = a.ucur + b * a.mstride;
            const T* pb = a.uprev + b * a.mstride;
            for (int t = 0; t < L; ++t, ++it) {
                const int slot = int(it % depth);
                if (it >= depth) mbar_wait(&empty[slot], uint32_t(((it / depth) - 1) & 1));
                T* un_s = reinterpret_cast<T*>(smem + size_t(slot) * SLOT);
                T* pv_s = un_s + WH;
                T* c1_s = pv_s + WC;
                T* c2_s = c1_s + WH;
                const int r = s0 - 1 + t;
                uint32_t bytes = WH * sizeof(T);
                if (t >= 2) bytes += WC * sizeof(T);
                if (MODE == MODE_DENSE) {
                    if (t >= 1) bytes += WC * sizeof(T);
                    if (t >= 2) bytes += WH * sizeof(T);
                }
                mbar_arrive_expect_tx(&full[slot], bytes);
                bulk_g2s(un_s, ub + r * a.pitch + cs - H, WH * sizeof(T), &full[slot]);
                if (t >= 2) bulk_g2s(pv_s, pb + (r - 1) * a.pitch + cs, WC * sizeof(T), &full[slot]);
                if (MODE == MODE_DENSE) {
                    if (t >= 2)
                        bulk_g2s(c1_s, a.c1 + b * a.cstride1 + (r - 1) * a.pitch + cs - H, WH * sizeof(T), &full[slot]);
                    if (t >= 1) bulk_g2s(c2_s, a.c2 + b * a.cstride2 + r * a.pitch + cs, WC * sizeof(T), &full[slot]);
                }
            }
        }
        return;
    }

    // ------------------------------ consumer warps ------------------------------
    const int tid = threadIdx.x;  // 0 .. NC·32 − 1
    int64_t it = 0;
    for (int64_t item = blockIdx.x; item < a.items; item += gridDim.x) {
        int64_t cs;
        int s0, s1, b;
        item_geom(item, cs, s0, s1, b);
        const int64_t col = cs + int64_t(tid) * V;
        T* __restrict__ pb = a.uprev + b * a.mstride;
        bool interior[V];
#pragma unroll
        for (int k = 0; k < V; ++k) interior[k] = (col + k >= 1) && (col + k <= a.nx - 2);
        T c1r[V], c1l[V], c2v[V];
        if (MODE == MODE_LINE) {  // row-invariant: c1 per x face, c2 per node column
            const T* c1b = a.c1 + b * a.cstride1;
            vload(c1b + col, c1r);
            c1l[0] = (col > 0) ? __ldg(c1b + col - 1) : (T)0;
#pragma unroll
            for (int k = 1; k < V; ++k) c1l[k] = c1r[k - 1];
            vload(a.c2 + b * a.cstride2 + col, c2v);
        }
        T up[V], cu[V], dn[V], pv[V], c2lo[V], c2hi[V];
        const int L = s1 - s0 + 2;
        int prev_slot = 0;
        for (int t = 0; t < L; ++t, ++it) {
            const int slot = int(it % depth);
            mbar_wait(&full[slot], uint32_t((it / depth) & 1));
            const T* un_s = reinterpret_cast<const T*>(smem + size_t(slot) * SLOT);
            const T* pv_s = un_s + WH;
            const T* c1_s = pv_s + WC;
            const T* c2_s = c1_s + WH;
            if (t == 0) {
                lds_vec(un_s + H + tid * V, up);
            } else if (t == 1) {
                lds_vec(un_s + H + tid * V, cu);
                if (MODE == MODE_DENSE) lds_vec(c2_s + tid * V, c2lo);
            } else {
                lds_vec(un_s + H + tid * V, dn);
                lds_vec(pv_s + tid * V, pv);
                T c1d_r[V], c1d_l[V];
                if (MODE == MODE_DENSE) {
                    lds_vec(c2_s + tid * V, c2hi);
                    lds_vec(c1_s + H + tid * V, c1d_r);
                    c1d_l[0] = c1_s[H + tid * V - 1];
#pragma unroll
                    for (int k = 1; k < V; ++k) c1d_l[k] = c1d_r[k - 1];
                }
                // horizontal neighbours of the centre row (loaded at the previous stage)
                const T* ce = reinterpret_cast<const T*>(smem + size_t(prev_slot) * SLOT);
                const T left = ce[H + tid * V - 1];
                const T right = ce[H + tid * V + V];
                T out[V];
#pragma unroll
                for (int k = 0; k < V; ++k) {
                    T ul = (k == 0) ? left : cu[k - 1];
                    T ur = (k == V - 1) ? right : cu[k + 1];
                    T l1 = (MODE == MODE_LINE) ? c1l[k] : c1d_l[k];
                    T r1 = (MODE == MODE_LINE) ? c1r[k] : c1d_r[k];
                    T d2 = (MODE == MODE_LINE) ? c2v[k] : c2lo[k];
                    T u2 = (MODE == MODE_LINE) ? c2v[k] : c2hi[k];
                    T v = node_update<T, START, true>(cu[k], ul, ur, up[k], dn[k], pv[k], l1, r1, d2, u2, a.dtT);
                    out[k] = interior[k] ? v : (T)0;
                }
                const int s = s0 + t - 2;
                if (col < a.pitch) vstore(pb + s * a.pitch + col, out);  // ragged last strip
#pragma unroll
                for (int k = 0; k < V; ++k) {
                    up[k] = cu[k];
                    cu[k] = dn[k];
                    if (MODE == MODE_DENSE) c2lo[k] = c2hi[k];
                }
            }
            // release the previous stage (its rows are in registers / consumed above); the last
            // stage of an item releases itself too.
            __syncwarp();
            if (lane == 0) {
                if (t >= 1) mbar_arrive(&empty[prev_slot]);
                if (t == L - 1) mbar_arrive(&empty[slot]);
            }
            prev_slot = slot;
        }
    }
}

// ------------------------------------------------------------------------------------------
// S3, temporally blocked: K leapfrog levels per HBM pass, out of place.
// ------------------------------------------------------------------------------------------
// A CTA of 8 warps owns an extended strip of WE = 256·V columns (4 KB of
// a row): WO = WE − 2H output columns plus H ≥ K halo columns per side, recomputed redundantly.
// It marches a chunk of output rows [s0, s1) reading input rows [s0 − K, s1 + K) (clipped at the
// Dirichlet rows).  At input row R it advances a wavefront: level m (1..K) at row R − m, from
// level m−1 rows R−m−1..R−m+1 and level m−2 at row R−m (leapfrog).  Each thread keeps a 3-row
// register window per level for its own V columns; the row each level produced in the previous
// iteration (the next iteration's centre row) sits in shared memory, double-buffered by row
// parity, for the left/right neighbours — one CTA barrier per input row.  Inputs (u^n, u^{n−1})
// arrive by TMA bulk copies (issued by thread 0) into a D-stage ring; outputs u^{n+K}, u^{n+K−1}
// go to two other buffers (out of place: the halo columns of u^n, u^{n−1} are read by the
// neighbouring strips).
// HBM traffic per node and pass: 2 reads + 2 writes for K levels (vs 3K words unblocked).
// Every node value is the same canonical expression as k_step2d (bitwise identical results);
// Dirichlet rows/columns are forced to +0 at every level.
constexpr int TB_NC = 8;
// deepest temporal blocking, and ghost rows per side of a slab (a pass of K levels exchanges K rows)
constexpr int TSW_MAX_TB = 10;
constexpr int TSW_MAX_GHOST = TSW_MAX_TB;

template <typename T, int K, int NC = TB_NC>
struct TbGeom {
    static constexpr int V = 2;                                  // columns per thread
    static constexpr int NT = NC * 32;
    static constexpr int A = (16 / int(sizeof(T))) > V ? (16 / int(sizeof(T))) : V;  // 16-byte TMA alignment
    static constexpr int H = ((K + A - 1) / A) * A;              // halo columns per side (≥ K)
    static constexpr int WE = NT * V;                            // 512 columns
    static constexpr int WO = WE - 2 * H;
};

template <typename T>
__device__ __forceinline__ void lds_v2(const T* p, T (&v)[2]) {
    typename Vec2<T>::type x = *reinterpret_cast<const typename Vec2<T>::type*>(p);
    v[0] = x.x;
    v[1] = x.y;
}
template <typename T>
__device__ __forceinline__ void sts_v2(T* p, const T (&v)[2]) {
    typename Vec2<T>::type x;
    x.x = v[0];
    x.y = v[1];
    *reinterpret_cast<typename Vec2<T>::type*>(p) = x;
}
template <typename T>
__device__ __forceinline__ void stg_v2(T* p, const T (&v)[2]) {
    typename Vec2<T>::type x;
    x.x = v[0];
    x.y = v[1];
    __stcs(reinterpret_cast<typename Vec2<T>::type*>(p), x);
}

template <typename T>
struct TbArgs {
    const T* un;
    const T* unm1;
    T* out_k;    // u^{n+K}
    T* out_km1;  // u^{n+K−1}
    const T* c1;
    const T* c2;
    int64_t pitch, mstride, cstride, nx, ny, r0;
    int32_t s_lo, s_hi;  // output storage rows
    // an optional second range of output rows (a slab's first and last K rows in one launch):
    // chunks [0, chunks1) cover [s_lo, s_hi), the rest [s_lo2, s_hi2)
    int32_t s_lo2 = 0, s_hi2 = 0, chunks1 = INT32_MAX;
    int32_t smin, smax;  // storage rows inside the grid (global rows 0 .. ny−1 of this slab)
    int32_t rows_per_item, chunks;
    int64_t strips, items;
    T dtT;
    // fused halo push (peer mode): output rows ro ≤ push_top are also stored into the
    // upper neighbour's lower ghost rows, rows ro ≥ push_bot into the lower neighbour's upper ghost
    // rows, through mapped peer pointers shifted so that the row index is this slab's
    T* pu_k = nullptr;
    T* pu_km1 = nullptr;
    T* pd_k = nullptr;
    T* pd_km1 = nullptr;
    int64_t pu_mstride = 0, pd_mstride = 0;
    int32_t push_top = 0, push_bot = INT32_MAX;
    // fused discrete energy (EN variant, S5 / R17, node form R30): one fp64 partial per item of
    // Σ over its output nodes of (u^{n+K} − u^{n+K−1})² − u^{n+K}·L(u^{n+K−1})
    double* en_part = nullptr;
};

// centre-row buffers are padded by one 16-byte vector on each side (zeros), so the left/right
// neighbours of every thread are read without bounds checks
template <typename T>
struct TbPad {
    static constexpr int P = 16 / sizeof(T);
};

// Caching the upper y-flux for the next row saves 2 fp ops per update (identical operands, so the
// tree is unchanged bit for bit).  fp32 keeps it in registers (2V per level).  fp64 recomputes it:
// in registers (TSW_TB_YCACHE_F64 = 1) it measured +3 % at K = 7, −2 % at K = 8, −27 % at K = 10
// (spills); in shared or tensor memory it was slower still (measured and rejected).
// TSW_TB_YCACHE_F64_LEVELS = L caches it for the first L levels only (the registers left under
// the 170-register budget).
#ifndef TSW_TB_YCACHE_F64
#define TSW_TB_YCACHE_F64 0
#endif
#ifndef TSW_TB_YCACHE_F64_LEVELS
#define TSW_TB_YCACHE_F64_LEVELS 0
#endif
template <typename T> struct TbYCache {
    // levels 1..levels<K>() keep the flux in registers
    template <int K> __host__ __device__ static constexpr int levels() {
        return (sizeof(T) == 4 || TSW_TB_YCACHE_F64) ? K
                                                      : (TSW_TB_YCACHE_F64_LEVELS < K ? TSW_TB_YCACHE_F64_LEVELS : K);
    }
};

// Register budget and CTA width.  A CTA of NC warps is sized for 16 / NC CTAs per SM (at least
// one): 8 warps → two CTAs of 128 registers per thread; TSW_TB_NCW_F64 = 12 (default) → one
// 12-warp CTA per SM with up to 170 registers per thread (768-column strips) for the deep fp64
// passes (K ≥ TSW_TB_NCW_KMIN): measured fp64 K = 8 918 → 976 Gpt/s (985 with an 8-stage ring),
// K = 7 905 → 943 — the compiler schedules the K-level chain better with the larger budget, and
// 12 warps per SM hide the fp64 latency (10, 11, 14 or 16 warps, or 8 warps at 198 registers
// with the y-flux cache in registers, were slower).  TSW_TB_MINB_F64 = 1 forces one CTA per SM
// for every fp64 width; TSW_TB_YCACHE_F64 = 1 keeps the fp64 y-flux cache in registers.
#ifndef TSW_TB_MINB_F64
#define TSW_TB_MINB_F64 0
#endif
#ifndef TSW_TB_NCW_F64
#define TSW_TB_NCW_F64 12
#endif
#define TSW_TB_MINB(T, NC) ((sizeof(T) == 8 && TSW_TB_MINB_F64) ? TSW_TB_MINB_F64 : (16 / (NC) > 0 ? 16 / (NC) : 1))
// per pass depth: the narrow fp64 CTA (4 warps: slab boundary rows, narrow grids) of depth ≥ 8 is
// sized for 3 CTAs per SM (170 registers, as the wide CTA) — at 4 CTAs (128 registers) K = 10
// spilled 1.3 KB
template <typename T, int K, int NC> constexpr int tb_minb() {
    return (sizeof(T) == 8 && NC == 4 && K >= 8 && !TSW_TB_MINB_F64) ? 3 : TSW_TB_MINB(T, NC);
}
#ifndef TSW_TB_NCW_KMIN
#define TSW_TB_NCW_KMIN 7   // the wide fp64 CTA for passes of depth ≥ this (shallower: 8 warps, 2 CTAs/SM)
#endif
#ifndef TSW_TB_NCW_F32
#define TSW_TB_NCW_F32 8
#endif
template <typename T, int K = 8> constexpr int tb_wide_nc() {
    return K < TSW_TB_NCW_KMIN ? 8 : (sizeof(T) == 8 ? TSW_TB_NCW_F64 : TSW_TB_NCW_F32);
}

// TSW_TB_JITTER=1 (debug builds only): a pseudo-random per-(CTA, warp, row) delay of up to ~2 µs
// before and after every row barrier, so warps reach the barrier, read the centre rows and the
// stages, and issue the refills in changing orders — a race-perturbation test (compute-sanitizer's
// racecheck is unavailable on this GPU pool): results must stay bitwise those of the plain build.
#ifndef TSW_TB_JITTER
#define TSW_TB_JITTER 0
#endif
__device__ __forceinline__ void tb_jitter(int R, int warp, int where) {
    uint32_t h = uint32_t(blockIdx.x) * 0x9E3779B1u ^ uint32_t(R) * 0x85EBCA77u ^ uint32_t(warp * 2 + where) * 0xC2B2AE3Du;
    h ^= h >> 15;
    h *= 0x2C1B3C6Du;
    h ^= h >> 12;
    if ((h & 7u) == 0u) __nanosleep(h % 2048u);   // one row in eight, per warp
}

// Every warp waits on a stage's "full" mbarrier after the per-row CTA barrier: a single waiter
// before the barrier measured 5 % slower (its ≈ 90-cycle try_wait is serialised).
// TSW_TB_STARTUP = 0 runs an item's start-up rows with every level (no level cut, see tb_row).
#ifndef TSW_TB_STARTUP
#define TSW_TB_STARTUP 1
#endif

// Measured and rejected (round 2): the left/right neighbours of every level from the
// adjacent lanes' registers (__shfl_up/down_sync), only warp edges through shared memory —
// fp64 909 → 815 Gpt/s, fp32 1531 → 1355 (the baseline's MIO throttle is ≈ 0; the shuffles and
// edge selects add issue slots).

// Centre-row buffers (one row per level and parity).  Default: columns in order, a thread's two
// columns as one 16-byte store, its left / right neighbours as two 8-byte loads at a 16-byte stride
// (4 wavefronts each).  Split (TSW_TB_SPLIT_CEN_F64 / _F32): even columns then odd columns (with a zero pad
// between), so both neighbour loads are consecutive across the warp (2 wavefronts each) and the
// store becomes two consecutive 8-byte stores.  Measured (interleaved A/B, three rounds): fp64
// K = 10 1007 → 1013 Gpt/s (on by default), fp32 1711 → 1700 (off).
#ifndef TSW_TB_SPLIT_CEN_F64
#define TSW_TB_SPLIT_CEN_F64 1
#endif
#ifndef TSW_TB_SPLIT_CEN_F32
#define TSW_TB_SPLIT_CEN_F32 0
#endif
template <typename T, int K, int NC>
struct TbCen {
    static constexpr int P = TbPad<T>::P, NT = TbGeom<T, K, NC>::NT, WE = TbGeom<T, K, NC>::WE;
    static constexpr bool split = sizeof(T) == 8 ? TSW_TB_SPLIT_CEN_F64 : TSW_TB_SPLIT_CEN_F32;
    static constexpr int WEP = split ? WE + 3 * P : WE + 2 * P;   // one row, pads included
    static constexpr int OOFF = NT + P;                           // split: odd region − even region
    static constexpr int LOFF = split ? OOFF - 1 : -1;            // column 2t − 1 (odd of t − 1)
    static constexpr int ROFF = split ? 1 : 2;                    // column 2t + 2 (even of t + 1)
    __host__ __device__ static constexpr int base(int tid) { return split ? tid : 2 * tid; }
};
template <typename T, int K, int NC>
__device__ __forceinline__ void cen_store(T* p, const T (&v)[2]) {
    if constexpr (TbCen<T, K, NC>::split) {
        p[0] = v[0];
        p[TbCen<T, K, NC>::OOFF] = v[1];
    } else {
        sts_v2(p, v);
    }
}

template <typename T, int K, int NC = TB_NC>
__host__ __device__ constexpr size_t tb_smem_bytes(int depth) {
    return size_t(depth) * 2 * TbGeom<T, K, NC>::WE * sizeof(T) +
           size_t(K) * 2 * TbCen<T, K, NC>::WEP * sizeof(T) +
           (size_t(depth) * sizeof(uint64_t) + 15) / 16 * 16;
}

// Per-thread state of one item's wavefront.  Window slots rotate with the row phase PH ∈ {0,1,2}:
// before row i (phase PH = i mod 3) level m holds rows (r−1, r, r+1) in slots (PH, PH+1, PH+2) mod 3;
// its new row overwrites slot PH, so no register moves are needed.


template <typename T, int K>
struct TbState {
    static constexpr int V = 2;
    T w[K][3][V];
    T gup[TbYCache<T>::template levels<K>() + 1][V];  // level m's y-flux c2·(u_{r+1} − u_r) of level m−1 at its last row r: the next
                      // row's lower flux (identical operands, so the tree is unchanged bit for bit)
    T pm1[V];
    T c1l[V], c1r[V], c2v[V];
    bool colint[V];
};

// Fused energy (EN).  E^{n+½} = (dx·dy/dt²)·[Σ_nodes (u^{n+1} − u^n)² + Σ_faces c·Δu^{n+1}·Δu^n]
// (R17) in its node form: with K̃ = −L symmetric and u = 0 on the Dirichlet ring, summation by parts
// turns the face sum into ⟨u^{n+1}, K̃u^n⟩ = −Σ_nodes u^{n+1}·(L u^n) (reading R30).  At level K of a
// pass the stencil has just evaluated L(u^{n+K−1}) at every node of u^{n+K}, so the energy of the
// pass's outputs is a per-node sum — no neighbours, no seams.  fp64: the stencil's own L; fp32: L
// re-evaluated in fp64 from the same fp32 values (an fp32 L loses digits to cancellation).
__device__ __forceinline__ double warp_sum_d(double v) {
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
    return v;
}

// One input row of the wavefront.  `cr` / `cw`: this thread's element in the centre-row buffers
// of the previous / current row parity (level m at offset m·2·WEP).  MASKED: force the Dirichlet
// rows/columns to +0 (only items whose dependency cone touches them need it).
// SU (start-up rows of an item, TSW_TB_STARTUP): only levels m ≤ mcount are computed — at input row
// i of an unclamped item, level m yields row s0 − K + i − m, which a level-K output needs only when
// i ≥ 2m, so mcount = ⌊i/2⌋ skips the K(K+1) level-rows per item that no output depends on.
template <typename T, int K, int PH, bool MASKED, int NC, bool EN = false, bool SU = false>
__device__ __forceinline__ void tb_row(TbState<T, K>& S, const T* __restrict__ cr, T* __restrict__ cw, int rowlo,
                                       int rowhi, int R, const T (&nw)[2], const T (&pv_new)[2], T (&lastk)[2],
                                       const T (&lr1)[2], int lane, bool en_on = false,
                                       double* en_acc = nullptr, int mcount = K) {
    constexpr int V = 2;
    constexpr int WEP = TbCen<T, K, NC>::WEP;
    constexpr int O = PH % 3, C = (PH + 1) % 3, N = (PH + 2) % 3;  // pre-update roles
    // level 0
#pragma unroll
    for (int k = 0; k < V; ++k) S.w[0][O][k] = nw[k];
    // left/right neighbours of level m−1's centre row (written in the previous row, other parity
    // buffer): level 1's were loaded by the caller before the stage wait; level m+1's are loaded
    // before level m's arithmetic and store, so no level waits on a shared-memory load
    T left = lr1[0], right = lr1[1];
#pragma unroll
    for (int m = 1; m <= K; ++m) {
        if constexpr (SU) {
            if (m > mcount) {   // this and every higher level: rows no output depends on
                if (m == 1) cen_store<T, K, NC>(cw, nw);   // level 0's centre row is still read by the next row
                break;
            }
        }
        // level m−1 after its update: rows (r−1, r, r+1) in slots (C, N, O); level m−2: row r in C
        T nleft = (T)0, nright = (T)0;
        if (m < K) {
            const T* cn = cr + m * 2 * WEP;
            nleft = cn[TbCen<T, K, NC>::LOFF];
            nright = cn[TbCen<T, K, NC>::ROFF];
        }
        if (m == 1) cen_store<T, K, NC>(cw, nw);
        // canonical tree with shared face fluxes:
        //   F_{i+1/2} = c1_{i+1/2}·(u_{i+1} − u_i) is node i's right and node i+1's left x-flux,
        //   G_{j+1/2} = c2·(u_{j+1} − u_j) is row j's upper and row j+1's lower y-flux
        //   lap = (F_{i+1/2} − F_{i−1/2}) + (G_{j+1/2} − G_{j−1/2});  u' = (2u − p) + lap
        const T u0 = S.w[m - 1][N][0], u1 = S.w[m - 1][N][1];
        const T F0 = r_mul(S.c1l[0], r_sub(u0, left));
        const T F1 = r_mul(S.c1r[0], r_sub(u1, u0));
        const T F2 = r_mul(S.c1r[1], r_sub(right, u1));
        T nv[V];
        bool rowok = true;
        if (MASKED) rowok = unsigned(R - m - rowlo) <= unsigned(rowhi - rowlo);
#pragma unroll
        for (int k = 0; k < V; ++k) {
            const T cu = S.w[m - 1][N][k];
            const T gu = r_mul(S.c2v[k], r_sub(S.w[m - 1][O][k], cu));
            T gd;
            if (m <= TbYCache<T>::template levels<K>()) {
                // SU rows: the cached flux of a level computed for the first time is not there yet —
                // recomputed from the same operands (the cache's gu of the previous row), bit for bit
                gd = SU ? r_mul(S.c2v[k], r_sub(cu, S.w[m - 1][C][k])) : S.gup[m][k];
                S.gup[m][k] = gu;
            } else {
                gd = r_mul(S.c2v[k], r_sub(cu, S.w[m - 1][C][k]));
            }
            const T lapx = (k == 0) ? r_sub(F1, F0) : r_sub(F2, F1);
            const T lap = r_add(lapx, r_sub(gu, gd));
            const T pr = (m == 1) ? S.pm1[k] : S.w[(m >= 2) ? m - 2 : 0][C][k];
            const T v = r_add(twice_minus(cu, pr), lap);
            if (MASKED) {
                const bool ok = rowok & S.colint[k];
                nv[k] = ok ? v : (T)0;
            } else {
                nv[k] = v;
            }
            if constexpr (EN) {
                if (m == K && en_on) {
                    // node form of the energy of (u^{n+K}, u^{n+K−1}) = (nv, cu): (a − b)² − a·L(b)
                    double lapd;
                    if constexpr (sizeof(T) == 8) {
                        lapd = (double)lap;
                    } else {
                        const double ul = (k == 0) ? (double)left : (double)S.w[m - 1][N][0];
                        const double ur = (k == 0) ? (double)S.w[m - 1][N][1] : (double)right;
                        const double uc = cu, uu = S.w[m - 1][O][k], ud = S.w[m - 1][C][k];
                        const double cl = (k == 0) ? (double)S.c1l[0] : (double)S.c1r[0];
                        const double crr = (double)S.c1r[k], c2 = (double)S.c2v[k];
                        lapd = (crr * (ur - uc) - cl * (uc - ul)) + (c2 * (uu - uc) - c2 * (uc - ud));
                    }
                    // accumulated with two fused multiply-adds (the energy is a diagnostic, not the
                    // canonical stepping tree): acc + (a − b)² − a·L(b)
                    const double A = (double)nv[k], D = A - (double)cu;
                    *en_acc = __fma_rn(-A, lapd, __fma_rn(D, D, *en_acc));
                }
            }
        }
        if (m < K) {
#pragma unroll
            for (int k = 0; k < V; ++k) S.w[m][O][k] = nv[k];
            cen_store<T, K, NC>(cw + m * 2 * WEP, nv);
        } else {
#pragma unroll
            for (int k = 0; k < V; ++k) lastk[k] = nv[k];
        }
        left = nleft;
        right = nright;
    }
#pragma unroll
    for (int k = 0; k < V; ++k) S.pm1[k] = pv_new[k];
}

// The producer is thread 0: after every second input row it refills the two stages consumed by
// the previous rows (every thread has passed the per-row barrier, so they are free) with the next
// stages of its stream (needs a ring of ≥ 3 stages).
template <typename T, int K, bool PEER = false, int NC = TB_NC, bool EN = false>
__global__ void __launch_bounds__(NC * 32, tb_minb<T, K, NC>()) k_step2d_tb(const TbArgs<T> a, int depth) {
    using G = TbGeom<T, K, NC>;
    constexpr int V = G::V, H = G::H, WE = G::WE, WO = G::WO;
    constexpr int PAD = TbPad<T>::P, WEP = TbCen<T, K, NC>::WEP;
    extern __shared__ __align__(128) unsigned char smem[];
    T* ring = reinterpret_cast<T*>(smem);                    // [depth][2][WE]
    T* cenp = ring + size_t(depth) * 2 * WE;                 // [K][2][WEP], row data at +PAD
    constexpr size_t CEN_ELEMS = size_t(K) * 2 * WEP;
    uint64_t* full = reinterpret_cast<uint64_t*>(cenp + CEN_ELEMS);
    T* cen = cenp + PAD;
    const int tid = threadIdx.x;
    const int lane = tid & 31;
    for (int e = tid; e < int(CEN_ELEMS); e += blockDim.x) cenp[e] = (T)0;  // pads stay 0
    __shared__ double en_red[EN ? NC : 1];   // EN: per-item warp sums
    if (tid == 0) {
        for (int k = 0; k < depth; ++k) mbar_init(&full[k], 1);
        fence_barrier_init();
    }
    __syncthreads();

    auto geom = [&](int64_t item, int64_t& cs, int& s0, int& s1, int& b, int& in_lo, int& in_hi) {
        const int64_t strip = item % a.strips;
        const int64_t rest = item / a.strips;
        const int chunk = int(rest % a.chunks);
        b = int(rest / a.chunks);
        cs = strip * WO;
        if (chunk < a.chunks1) {
            s0 = a.s_lo + chunk * a.rows_per_item;
            s1 = min(s0 + a.rows_per_item, a.s_hi);
        } else {
            s0 = a.s_lo2 + (chunk - a.chunks1) * a.rows_per_item;
            s1 = min(s0 + a.rows_per_item, a.s_hi2);
        }
        in_lo = max(s0 - K, a.smin);
        in_hi = min(s1 + K, a.smax + 1);
    };

    // ---- producer: stages are issued per item — its first `depth` loaded rows at the item's start
    // (after a barrier: every stage of the previous item is consumed), then, after each row's
    // barrier, the stage the previous row consumed is refilled with the row `depth` further on by
    // one elected lane of a rotating warp.  No cross-item prefetch: a CTA holds one or a few items
    // of hundreds of rows, so the refill drain at an item start (one load latency) is ≪ 1 %, and no
    // thread carries a stream position across items on every row.
    const int warp = __shfl_sync(0xffffffffu, tid >> 5, 0);  // warp-uniform by construction
    auto issue_stage = [&](int slot, int64_t e) {
        T* st = ring + size_t(slot) * 2 * WE;
        mbar_arrive_expect_tx(&full[slot], 2 * WE * sizeof(T));
        bulk_g2s(st, a.un + e, WE * sizeof(T), &full[slot]);
        bulk_g2s(st + WE, a.unm1 + e, WE * sizeof(T), &full[slot]);
    };
    // the ring depth is a power of two (the runtime checks): slot = loaded-row count & dmask
    const int dmask = depth - 1;
    const int dlog = __ffs(depth) - 1;

    const int e0 = tid * V;  // my first column of the extended strip
    const int ce0 = TbCen<T, K, NC>::base(tid);
    T* const cen0 = cen + ce0;         // my element in the centre-row buffers of parity 0 / 1
    T* const cen1 = cen + WEP + ce0;
    // interior storage rows of the global grid: g ∈ [1, ny−2] ⇔ storage s ∈ [rowlo, rowhi]
    const int rowlo = int(1 - a.r0 + 1), rowhi = int(a.ny - 2 - a.r0 + 1);
    int gs = 0;         // rows loaded from the ring so far: slot gs & dmask, phase parity (gs >> dlog) & 1
    TbState<T, K> S;
    // EN: this thread's sum over its output nodes of the current item.  In registers: a running
    // sum in a shared-memory slot (one read-modify-write per row) removed the 16-byte spill of the
    // fp64 K = 10 EN pass but raised its cost over the plain pass from 5.1 % to 8.5 % (measured).
    double en_acc = 0.0;
    for (int64_t item = blockIdx.x; item < a.items; item += gridDim.x) {
        int64_t cs;
        int s0, s1, b, in_lo, in_hi;
        geom(item, cs, s0, s1, b, in_lo, in_hi);
        const int64_t gc0 = cs - H + e0;  // global column of my first element
        const T* c1b = a.c1 + b * a.cstride;
        const T* c2b = a.c2 + b * a.cstride;
#pragma unroll
        for (int k = 0; k < V; ++k) {
            const int64_t gcol = gc0 + k;
            S.colint[k] = (gcol >= 1) && (gcol <= a.nx - 2);
            // face coefficients wherever the face exists (the shared x-flux of column k's right face
            // is column k+1's left flux even when column k is a boundary node)
            S.c1r[k] = (gcol >= 0 && gcol <= a.nx - 2) ? __ldg(c1b + gcol) : (T)0;
            S.c1l[k] = (gcol >= 1 && gcol <= a.nx - 1) ? __ldg(c1b + gcol - 1) : (T)0;
            S.c2v[k] = S.colint[k] ? __ldg(c2b + gcol) : (T)0;
        }
        const bool out_cols = (e0 >= H) && (e0 < H + WO) && (cs - H + e0 < a.pitch);
        // running output pointers: row ro = R − K of the current input row R = in_lo + i
        // (u^{n+K−1} at the same element: an item-uniform distance from u^{n+K})
        T* okp = a.out_k + b * a.mstride + gc0 + int64_t(in_lo - K) * a.pitch;
        const int64_t dkm1 = a.out_km1 - a.out_k;
        // PEER: element distances from the local outputs to the neighbours' ghost rows (uniform)
        int64_t pdist[4] = {0, 0, 0, 0};
        if constexpr (PEER) {
            pdist[0] = (a.pu_k + b * a.pu_mstride) - (a.out_k + b * a.mstride);
            pdist[1] = (a.pu_km1 + b * a.pu_mstride) - (a.out_k + b * a.mstride);
            pdist[2] = (a.pd_k + b * a.pd_mstride) - (a.out_k + b * a.mstride);
            pdist[3] = (a.pd_km1 + b * a.pd_mstride) - (a.out_k + b * a.mstride);
        }
        // Dirichlet masking is only needed where the item's dependency cone (rows in_lo − K ..
        // s1 + K − 1, the extended strip's columns) touches a boundary row/column or the grid edge
        const bool col_clear = (cs - H >= 1) && (cs - H + WE <= a.nx - 1);
        const bool masked = !((in_lo - K >= rowlo) && (s1 + K - 1 <= rowhi) && col_clear);
#pragma unroll
        for (int m = 0; m < K; ++m)
#pragma unroll
            for (int q = 0; q < 3; ++q)
#pragma unroll
                for (int k = 0; k < V; ++k) S.w[m][q][k] = (T)0;
#pragma unroll
        for (int k = 0; k < V; ++k) S.pm1[k] = (T)0;
#pragma unroll
            for (int m = 0; m <= TbYCache<T>::template levels<K>(); ++m)
#pragma unroll
                for (int k = 0; k < V; ++k) S.gup[m][k] = (T)0;
        const int nload = in_hi - in_lo;
        const int L = s1 + K - in_lo;
        // this item's stage stream: input row in_lo + j at element ibase + j·pitch; prefill
        const int64_t ibase = b * a.mstride + int64_t(in_lo) * a.pitch + cs - H;
        __syncthreads();
        if (warp == 0 && elect_one()) {
            const int pre = min(depth, nload);
            for (int r = 0; r < pre; ++r) issue_stage((gs + r) & dmask, ibase + int64_t(r) * a.pitch);
        }

        // one input row: barrier, refill, stage read, wavefront (phase PH), output
        auto row = [&](auto ph, auto msk, auto su, int i) {
            constexpr int PH = decltype(ph)::value;
            constexpr bool MASKED = decltype(msk)::value;
            constexpr bool SU = decltype(su)::value;
            const int R = in_lo + i;
            if (TSW_TB_JITTER) tb_jitter(R, warp, 0);
            __syncthreads();  // the previous rows' stages and centre rows are consumed / published
            if (TSW_TB_JITTER) tb_jitter(R, warp, 1);
            // refill the stage consumed by the previous row (its shared-memory reads completed
            // before this barrier: the values were used in that row's arithmetic) with the item's
            // row `depth` further on
            if (i >= 1 && i - 1 + depth < nload) {   // row i − 1 consumed slot (gs − 1) & dmask
                if (warp == (i % NC) && elect_one())
                    issue_stage((gs - 1) & dmask, ibase + int64_t(i - 1 + depth) * a.pitch);
            }
            const int par = R & 1;
            T* cw;
            const T* cr;
            T lr1[V];  // level 1's left/right neighbours, before the stage wait
            if constexpr (sizeof(T) == 4) {   // fp32 (issue-bound): two precomputed bases
                cw = par ? cen1 : cen0;
                cr = par ? cen0 : cen1;
            } else {                            // fp64 (no spare registers): recomputed per row
                cw = cen + par * WEP + ce0;
                cr = cen + (par ^ 1) * WEP + ce0;
            }
            lr1[0] = cr[TbCen<T, K, NC>::LOFF];
            lr1[1] = cr[TbCen<T, K, NC>::ROFF];
            T nw[V], pv_new[V];
            const bool refill = (i < nload);
            if (refill) {
                const int cslot = gs & dmask;
                mbar_wait(&full[cslot], uint32_t(gs >> dlog) & 1u);
                const T* st = ring + size_t(cslot) * 2 * WE;
                lds_v2(st + e0, nw);
                lds_v2(st + WE + e0, pv_new);
                ++gs;
            } else {
#pragma unroll
                for (int k = 0; k < V; ++k) nw[k] = pv_new[k] = (T)0;
            }
            T lastk[V];
            const bool en_on = EN && out_cols && (R - K >= s0) && (R - K < s1);
            tb_row<T, K, PH, MASKED, NC, EN, SU>(S, cr, cw, rowlo, rowhi, R, nw, pv_new, lastk, lr1, lane,
                                                en_on, &en_acc, i >> 1);
            const int ro = R - K;
            if (out_cols && ro >= s0 && ro < s1) {
                // level K−1 after this row: rows (ro−1, ro, ro+1) in slots (C, N, O) of phase PH
                constexpr int NS = (PH + 2) % 3;
                T o2[V];
#pragma unroll
                for (int k = 0; k < V; ++k) o2[k] = S.w[K - 1][NS][k];
                stg_v2(okp, lastk);
                stg_v2(okp + dkm1, o2);
                if constexpr (PEER) {
                    // peer stores over NVLink (rare rows): the neighbour's element is the local
                    // output element plus an item-uniform distance (no per-thread pointer is held)
                    if (ro <= a.push_top) {
                        stg_v2(okp + pdist[0], lastk);
                        stg_v2(okp + pdist[1], o2);
                    }
                    if (ro >= a.push_bot) {
                        stg_v2(okp + pdist[2], lastk);
                        stg_v2(okp + pdist[3], o2);
                    }
                }
            }
            okp += a.pitch;
        };
        // rows [i0, i1) of the item; i0 is a multiple of 3 (the window phase is i mod 3)
        auto run_rows = [&](auto msk, auto su, int i0, int i1) {
            int i = i0;
            for (; i + 3 <= i1; i += 3) {
                row(std::integral_constant<int, 0>{}, msk, su, i);
                row(std::integral_constant<int, 1>{}, msk, su, i + 1);
                row(std::integral_constant<int, 2>{}, msk, su, i + 2);
            }
            if (i < i1) row(std::integral_constant<int, 0>{}, msk, su, i++);
            if (i < i1) row(std::integral_constant<int, 1>{}, msk, su, i++);
        };
        constexpr std::integral_constant<bool, false> no_su{};
        // Input row i computes levels m = 1..K at rows R − m (R = in_lo + i); it needs the
        // boundary selects only while one of those rows lies outside [rowlo, rowhi].  In a strip
        // clear of the boundary columns the item runs masked only at its ends (segment limits
        // rounded to the window phase).
        int ua = 0, ub = 0;
        if (masked && col_clear) {
            ua = rowlo + K - in_lo;
            ub = rowhi + 2 - in_lo;
            ua = (ua <= 0) ? 0 : (ua + 2) / 3 * 3;
            ub = (ub >= L) ? L : (ub <= 0 ? 0 : ub / 3 * 3);
            if (ub <= ua) ua = ub = 0;
        } else if (!masked) {
            ub = L;
        }
        if (ub <= ua) ua = ub = L;  // all masked: segment 0 covers the item
        // segments [0, ua) masked, [ua, ub) unmasked, [ub, L) masked (one call site per variant)
#pragma unroll 1
        for (int sg = 0; sg < 3; ++sg) {
            const int lo = (sg == 0) ? 0 : (sg == 1 ? ua : ub);
            const int hi = (sg == 0) ? ua : (sg == 1 ? ub : L);
            if (lo >= hi) continue;
            if (sg == 1) {
                // an unclamped item's first ⌊2K/3⌋·3 rows compute only the levels its outputs need
                // (a multiple of 3: the window phase) with the y-flux cache, up to a row at which
                // every level was computed, so that the rows after it (plain or masked) find every
                // cached flux
                constexpr int YCL = TbYCache<T>::template levels<K>();
                constexpr int SU_ROWS = (2 * K / 3) * 3 >= 2 * YCL + 1 ? (2 * K / 3) * 3 : (2 * YCL + 3) / 3 * 3;
                int mid = lo;
                if (TSW_TB_STARTUP && lo == 0 && in_lo == s0 - K && hi >= SU_ROWS) {
                    mid = SU_ROWS;
                    run_rows(std::integral_constant<bool, false>{}, std::integral_constant<bool, true>{}, 0, mid);
                }
                run_rows(std::integral_constant<bool, false>{}, no_su, mid, hi);
            } else {
                run_rows(std::integral_constant<bool, true>{}, no_su, lo, hi);
            }
        }
        if constexpr (EN) {
            const double v = warp_sum_d(en_acc);
            en_acc = 0.0;
            if (lane == 0) en_red[warp] = v;
            __syncthreads();
            if (tid == 0) {
                double t = 0.0;
#pragma unroll
                for (int w = 0; w < NC; ++w) t += en_red[w];
                a.en_part[item] = t;
            }
        }
    }
}

// Launch wrappers, defined and instantiated in tsw_tb.cu (one translation unit per precision).
template <typename T, int K, int NC, bool EN>
cudaError_t tb_setup(size_t smem, int* occ);
template <typename T, int K, int NC, bool EN>
cudaError_t tb_launch(bool push, unsigned blocks, size_t smem, cudaStream_t stream, const TbArgs<T>& a, int depth);

#ifndef TSW_TB_UNIT  // the rest is compiled in the runtime's translation unit only
// ------------------------------------------------------------------------------------------
// S2/S3: 1D, persistent — one CTA per member, both levels resident in shared memory, all
// steps in one launch (config 1: 2000 fp64 nodes × 3 arrays = 48 KB).
// ------------------------------------------------------------------------------------------
template <typename T>
__global__ void __launch_bounds__(1024) k_step1d_smem(T* __restrict__ ucur, T* __restrict__ uprev,
                                                      const T* __restrict__ c1, int64_t nx, int64_t pitch,
                                                      int64_t cpitch, int64_t nsteps, int start, T dtT) {
    extern __shared__ __align__(16) unsigned char smem_raw[];
    T* A = reinterpret_cast<T*>(smem_raw);  // u^n
    T* P = A + pitch;                       // u^{n−1} → u^{n+1}
    T* C = P + pitch;                       // c1
    const int b = blockIdx.x;
    T* ug = ucur + b * pitch;
    T* pg = uprev + b * pitch;
    const T* cg = c1 + b * cpitch;
    for (int64_t i = threadIdx.x; i < nx; i += blockDim.x) {
        A[i] = ug[i];
        P[i] = pg[i];
        if (i < nx - 1) C[i] = cg[i];
    }
    __syncthreads();
    int64_t k = 0;
    if (start && nsteps > 0) {
        for (int64_t i = 1 + threadIdx.x; i < nx - 1; i += blockDim.x)
            P[i] = node_update<T, true, false>(A[i], A[i - 1], A[i + 1], (T)0, (T)0, P[i], C[i - 1], C[i], (T)0,
                                               (T)0, dtT);
        __syncthreads();
        T* t = A; A = P; P = t;
        k = 1;
    }
    for (; k < nsteps; ++k) {
        for (int64_t i = 1 + threadIdx.x; i < nx - 1; i += blockDim.x)
            P[i] = node_update<T, false, false>(A[i], A[i - 1], A[i + 1], (T)0, (T)0, P[i], C[i - 1], C[i],
                                                (T)0, (T)0, dtT);
        __syncthreads();
        T* t = A; A = P; P = t;
    }
    for (int64_t i = threadIdx.x; i < nx; i += blockDim.x) {
        ug[i] = A[i];
        pg[i] = P[i];
    }
}

// 1D fallback when the row does not fit in shared memory: one launch per step.
template <typename T, bool START>
__global__ void k_step1d_global(const T* __restrict__ ucur, T* __restrict__ uprev, const T* __restrict__ c1,
                                int64_t nx, int64_t pitch, int64_t cpitch, T dtT) {
    const int b = blockIdx.y;
    const T* u = ucur + b * pitch;
    T* p = uprev + b * pitch;
    const T* c = c1 + b * cpitch;
    for (int64_t i = 1 + blockIdx.x * int64_t(blockDim.x) + threadIdx.x; i < nx - 1;
         i += int64_t(gridDim.x) * blockDim.x)
        p[i] = node_update<T, START, false>(u[i], u[i - 1], u[i + 1], (T)0, (T)0, p[i], c[i - 1], c[i], (T)0, (T)0,
                                            dtT);
}

// ------------------------------------------------------------------------------------------
// S1: coefficient builder — h_ε at half-grid faces in fp64
// ------------------------------------------------------------------------------------------
// φ_ε(d) = (c/ε)·exp(1/(t² − 1)), t = d/ε, for |t| < 1; exactly 0 otherwise (R25).
__device__ __forceinline__ double phi_eps(double d, double eps) {
    double t = d / eps;
    if (!(fabs(t) < 1.0)) return 0.0;
    return (TSW_MOLLIFIER_C / eps) * exp(1.0 / (t * t - 1.0));
}
// R9: node i at ((2i+1−n)·d)/2, face i+1/2 at ((2i+2−n)·d)/2.
__device__ __forceinline__ double grid_node(int64_t i, int64_t n, double d) { return (double(2 * i + 1 - n) * d) / 2.0; }
__device__ __forceinline__ double grid_face(int64_t i, int64_t n, double d) { return (double(2 * i + 2 - n) * d) / 2.0; }

struct CoeffArgs {
    int kind, order;
    double hb, xs, ys, dx, dy;
    const double* eps;  // [B] device
    const double* amp;  // [B] device
    int64_t nx, ny;
    int64_t r0;         // first global row of the slab
    int64_t rows_alloc, pitch, cpitch;
    int B;
    int s_base;         // storage row of blockIdx.y = 0 (1 − G: the deepest ghost row)
};

// LINE (and CONST): h1[b][i], i < nx−1 (pad 0), h2[b] = h_b.
__global__ void k_coeff_line(CoeffArgs a, double* __restrict__ h1, double* __restrict__ h2) {
    const int b = blockIdx.y;
    for (int64_t i = blockIdx.x * int64_t(blockDim.x) + threadIdx.x; i < a.cpitch; i += int64_t(gridDim.x) * blockDim.x) {
        double h = 0.0;
        if (i < a.nx - 1) {
            if (a.kind == 0) {
                h = a.hb;
            } else {
                double bump = phi_eps(grid_face(i, a.nx, a.dx) - a.xs, a.eps[b]);
                if (a.order == 2) bump = bump * bump;
                h = a.hb + a.amp[b] * bump;
            }
        }
        h1[b * a.cpitch + i] = h;
        h2[b * a.cpitch + i] = (i < a.nx) ? a.hb : 0.0;  // R6: h2 ≡ h_b (per node column)
    }
}

// ---- x-only profiles: piecewise-constant depth + singular terms ----------
// Φ(t) = ∫_{−1}^{t} φ (the mollifier's primitive; no closed form) by tanh-sinh quadrature:
// x = m + r·tanh(π/2·sinh u), u = k/32, |k| ≤ 140 (error ≈ 1e−15 absolute).
__device__ double mollifier_primitive(double t) {
    if (t <= -1.0) return 0.0;
    if (t >= 1.0) return 1.0;
    const double r = 0.5 * (t + 1.0), m = 0.5 * (t - 1.0);
    const double hstep = 1.0 / 32.0, half_pi = 1.5707963267948966;
    double acc = 0.0;
    for (int k = -140; k <= 140; ++k) {
        const double u = k * hstep;
        const double sh = half_pi * sinh(u);
        const double ch = cosh(sh);
        const double w = half_pi * cosh(u) / (ch * ch);
        const double x = m + r * tanh(sh);
        if (fabs(x) < 1.0) acc += w * (TSW_MOLLIFIER_C * exp(1.0 / (x * x - 1.0)));
    }
    return r * hstep * acc;
}

struct ProfileArgs {
    int nseg, nsing, isotropic;
    const double* data;  // [nseg values][nseg−1 breaks][nsing loc][nsing amp][nsing order]
    const double* eps;   // [B]
    const double* scale; // [B] multiplies every singular amplitude
    int64_t nx, cpitch;
    double dx;
};

// h_ε(x) = v_0 + Σ_k (v_k − v_{k−1}) Φ((x − b_k)/ε) + Σ_j A_j·scale·φ_ε(x − x_j)^{o_j}
// (h_{1,ε} = h_{0,ε} + φ_ε(x − 70), h_{2,ε} = h_{0,ε} + φ_ε²(x − 70)).
__device__ double profile_eval(const ProfileArgs& a, double x, double eps, double scale, bool with_sing) {
    const double* v = a.data;
    const double* br = v + a.nseg;
    const double* loc = br + (a.nseg - 1);
    const double* amp = loc + a.nsing;
    const double* ord = amp + a.nsing;
    double h = v[0];
    for (int k = 1; k < a.nseg; ++k) h += (v[k] - v[k - 1]) * mollifier_primitive((x - br[k - 1]) / eps);
    if (with_sing)
        for (int j = 0; j < a.nsing; ++j) {
            double p = phi_eps(x - loc[j], eps);
            if (ord[j] == 2.0) p = p * p;
            h += (scale * amp[j]) * p;
        }
    return h;
}

// LINE storage: h1[b][i] at x faces (with the singular terms), h2[b][i] at node columns
// (with them when isotropic — scalar depth H(x), P:1145–1149 — else segments only).
__global__ void k_coeff_profile(ProfileArgs a, double* __restrict__ h1, double* __restrict__ h2) {
    const int b = blockIdx.y;
    const double eps = a.eps[b], sc = a.scale[b];
    for (int64_t i = blockIdx.x * int64_t(blockDim.x) + threadIdx.x; i < a.cpitch; i += int64_t(gridDim.x) * blockDim.x) {
        h1[b * a.cpitch + i] = (i < a.nx - 1) ? profile_eval(a, grid_face(i, a.nx, a.dx), eps, sc, true) : 0.0;
        h2[b * a.cpitch + i] = (i < a.nx) ? profile_eval(a, grid_node(i, a.nx, a.dx), eps, sc, a.isotropic != 0) : 0.0;
    }
}

// POINT, dense storage layout: h1[b][s][i] = face (i+1/2, g), h2[b][s][i] = face (i, g−1/2),
// g = r0 + s − 1; entries outside the global grid are 0.
__global__ void k_coeff_point(CoeffArgs a, double* __restrict__ h1, double* __restrict__ h2) {
    const int b = blockIdx.z;
    const int64_t s = int64_t(blockIdx.y) + a.s_base;
    const int64_t g = a.r0 + s - 1;
    const double eps = a.eps[b], amp = a.amp[b];
    for (int64_t i = blockIdx.x * int64_t(blockDim.x) + threadIdx.x; i < a.pitch; i += int64_t(gridDim.x) * blockDim.x) {
        double v1 = 0.0, v2 = 0.0;
        if (g >= 0 && g < a.ny && i < a.nx - 1) {
            double bump = phi_eps(grid_face(i, a.nx, a.dx) - a.xs, eps) * phi_eps(grid_node(g, a.ny, a.dy) - a.ys, eps);
            if (a.order == 2) bump = bump * bump;
            v1 = a.hb + amp * bump;
        }
        if (g >= 1 && g < a.ny && i < a.nx) {
            double bump = phi_eps(grid_node(i, a.nx, a.dx) - a.xs, eps) * phi_eps(grid_face(g - 1, a.ny, a.dy) - a.ys, eps);
            if (a.order == 2) bump = bump * bump;
            v2 = a.hb + amp * bump;
        }
        const int64_t o = (b * a.rows_alloc + s) * a.pitch + i;
        h1[o] = v1;
        h2[o] = v2;
    }
}

// O3-equivalent prescale: c = fl_T(r·h), r = (dt·dt)/(d·d) computed on the device in fp64.
template <typename T>
__global__ void k_prescale(const double* __restrict__ h, T* __restrict__ c, int64_t n, double dt, double d) {
    const double r = (dt * dt) / (d * d);
    for (int64_t k = blockIdx.x * int64_t(blockDim.x) + threadIdx.x; k < n; k += int64_t(gridDim.x) * blockDim.x)
        c[k] = (T)(r * h[k]);
}

// S1b: Gershgorin ρ_G = max over updated nodes of 2·(Σ h_x/dx² + Σ h_y/dy²) (R16); atomicMax on
// the bit pattern (non-negative doubles order like their int64 bits).
__device__ __forceinline__ void atomic_max_pos(unsigned long long* addr, double v) {
    if (v >= 0.0) atomicMax(addr, (unsigned long long)__double_as_longlong(v));
}

__device__ __forceinline__ double warp_max(double v) {
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) v = fmax(v, __shfl_xor_sync(0xffffffffu, v, o));
    return v;
}

struct CflArgs {
    int dim, mode;
    const double* h1;
    const double* h2;
    int64_t nx, pitch, cpitch, rows_alloc;
    int32_t s_lo, s_hi;  // storage rows of updated nodes
    double dx, dy;
    int B;
};

__global__ void k_cfl(CflArgs a, unsigned long long* __restrict__ out) {
    const int b = blockIdx.z;
    double m = 0.0;
    // x-only coefficients (1D, LINE): every row has the same row sums, so one row decides the max
    const int64_t rows = (a.dim == 1 || a.mode == MODE_LINE) ? 1 : (a.s_hi - a.s_lo);
    const int64_t total = rows * (a.nx - 2);
    for (int64_t k = blockIdx.x * int64_t(blockDim.x) + threadIdx.x; k < total; k += int64_t(gridDim.x) * blockDim.x) {
        const int64_t i = 1 + k % (a.nx - 2);
        double r;
        if (a.dim == 1) {
            const double* h = a.h1 + b * a.cpitch;
            r = 2.0 * ((h[i - 1] + h[i]) / (a.dx * a.dx));
        } else if (a.mode == MODE_LINE) {
            const double* h = a.h1 + b * a.cpitch;
            const double hy = a.h2[b * a.cpitch + i];
            r = 2.0 * ((h[i - 1] + h[i]) / (a.dx * a.dx) + (hy + hy) / (a.dy * a.dy));
        } else {
            const int64_t s = a.s_lo + k / (a.nx - 2);
            const double* h1r = a.h1 + (b * a.rows_alloc + s) * a.pitch;
            const double* h2b = a.h2 + b * a.rows_alloc * a.pitch;
            r = 2.0 * ((h1r[i - 1] + h1r[i]) / (a.dx * a.dx) + (h2b[s * a.pitch + i] + h2b[(s + 1) * a.pitch + i]) / (a.dy * a.dy));
        }
        m = fmax(m, r);
    }
    m = warp_max(m);
    if ((threadIdx.x & 31) == 0) atomic_max_pos(out, m);
}

// Minimum over faces (positivity check).
__global__ void k_min_pos(const double* __restrict__ h, int64_t n, unsigned long long* __restrict__ out_neg_count) {
    unsigned long long c = 0;
    for (int64_t k = blockIdx.x * int64_t(blockDim.x) + threadIdx.x; k < n; k += int64_t(gridDim.x) * blockDim.x)
        c += (h[k] <= 0.0 || !(h[k] == h[k])) ? 1ull : 0ull;
    if (c) atomicAdd(out_neg_count, c);
}

// ------------------------------------------------------------------------------------------
// S5: discrete energy E^{n+1/2} partials (R17), fp64, warp-shuffle then block reduction.
// Terms owned by node (s, i) of the slab: its kinetic term (interior node), its x face
// (i+1/2) if its row is interior, and its y face (g+1/2) if g ≤ ny−2 and i interior.
// ------------------------------------------------------------------------------------------
struct EnergyArgs {
    int dim, mode;
    const void* unp1;  // u^{n}   of the ctx (the newer level)
    const void* un;    // u^{n−1}
    const void* c1;
    const void* c2;
    int64_t nx, ny, r0, pitch, mstride, cstride1, cstride2, ny_local;
    int nblk;
};

__device__ __forceinline__ double warp_sum(double v) {
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
    return v;
}

template <typename T>
__global__ void __launch_bounds__(256) k_energy(EnergyArgs a, double* __restrict__ partial) {
    const int b = blockIdx.y;
    const T* A = static_cast<const T*>(a.unp1) + b * a.mstride;
    const T* Bv = static_cast<const T*>(a.un) + b * a.mstride;
    const T* C1 = static_cast<const T*>(a.c1) + b * a.cstride1;
    const T* C2 = static_cast<const T*>(a.c2) + b * a.cstride2;
    const int64_t rows = (a.dim == 1) ? 1 : a.ny_local;
    const int64_t total = rows * a.nx;
    double acc = 0.0;
    for (int64_t k = blockIdx.x * int64_t(blockDim.x) + threadIdx.x; k < total; k += int64_t(gridDim.x) * blockDim.x) {
        const int64_t i = k % a.nx;
        const int64_t s = (a.dim == 1) ? 0 : 1 + k / a.nx;
        const int64_t g = (a.dim == 1) ? 0 : a.r0 + s - 1;
        const bool row_int = (a.dim == 1) || (g >= 1 && g <= a.ny - 2);
        const bool col_int = (i >= 1 && i <= a.nx - 2);
        const int64_t o = s * a.pitch + i;
        const double a0 = (double)A[o], b0 = (double)Bv[o];
        if (row_int && col_int) {
            const double d = a0 - b0;
            acc += d * d;
        }
        if (row_int && i <= a.nx - 2) {
            const double c = (a.dim == 1 || a.mode == MODE_LINE) ? (double)C1[i] : (double)C1[s * a.pitch + i];
            acc += (c * ((double)A[o + 1] - a0)) * ((double)Bv[o + 1] - b0);
        }
        if (a.dim == 2 && col_int && g <= a.ny - 2) {
            const double c = (a.mode == MODE_LINE) ? (double)C2[i] : (double)C2[(s + 1) * a.pitch + i];
            acc += (c * ((double)A[o + a.pitch] - a0)) * ((double)Bv[o + a.pitch] - b0);
        }
    }
    __shared__ double red[32];
    acc = warp_sum(acc);
    if ((threadIdx.x & 31) == 0) red[threadIdx.x >> 5] = acc;
    __syncthreads();
    if (threadIdx.x < 32) {
        double v = (threadIdx.x < (blockDim.x >> 5)) ? red[threadIdx.x] : 0.0;
        v = warp_sum(v);
        if (threadIdx.x == 0) partial[b * a.nblk + blockIdx.x] = v;
    }
}

// 2D energy, row march: a warp owns 32·V columns of a chunk of rows and reads each of the two
// levels once, vectorised (the x-face right neighbour of a lane's last element comes from the
// next lane; lane 31 reads one scalar).  One CTA (8 warps) = one item; partial[b][item].
struct Energy2Args {
    int mode;
    const void* unp1;  // newer level (u^n of the ctx)
    const void* un;    // older level (u^{n−1})
    const void* c1;
    const void* c2;
    int64_t nx, ny, r0, pitch, mstride, cstride1, cstride2;
    int32_t rows;          // owned rows: storage rows 1..rows
    int32_t rows_per_item;
    int32_t chunks;
    int64_t cta_strips;    // ceil(pitch / (8·32·V))
    int64_t items_per_member;
};

template <typename T, int MODE>
__global__ void __launch_bounds__(256, 3) k_energy2d(const Energy2Args a, double* __restrict__ partial) {
    constexpr int V = Vec16<T>::N;
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    const int64_t item = blockIdx.x;
    const int b = blockIdx.y;
    const int64_t cstrip = item % a.cta_strips;
    const int chunk = int(item / a.cta_strips);
    const int64_t cs = (cstrip * 8 + warp) * 32 * V;
    const int64_t col = cs + int64_t(lane) * V;
    const int s0 = 1 + chunk * a.rows_per_item;
    const int s1 = min(s0 + a.rows_per_item, a.rows + 1);
    const T* A = static_cast<const T*>(a.unp1) + b * a.mstride;
    const T* Bv = static_cast<const T*>(a.un) + b * a.mstride;
    const T* C1 = static_cast<const T*>(a.c1) + b * a.cstride1;
    const T* C2 = static_cast<const T*>(a.c2) + b * a.cstride2;
    double acc = 0.0;
    if (cs < a.pitch) {
        bool colint[V], xface[V];
#pragma unroll
        for (int k = 0; k < V; ++k) {
            colint[k] = (col + k >= 1) && (col + k <= a.nx - 2);
            xface[k] = (col + k <= a.nx - 2);
        }
        T c1l[V], c2l[V];
        if (MODE == MODE_LINE) {
            vload(C1 + col, c1l);
            vload(C2 + col, c2l);
        }
        // lane 31 needs the first column of the next strip (its right neighbour): prefetched one
        // row ahead together with the row itself, so no load sits on an iteration's critical path
        const bool rok = (lane == 31) && (cs + 32 * V < a.pitch);
        const int64_t rcol = cs + 32 * V;
        // two rows in flight ahead of the one being reduced (the loads are long-latency; storage
        // rows up to rows + 1 exist)
        T ac[V], bc[V], an[V], bn[V], a2[V], b2[V];
        vload(A + s0 * a.pitch + col, ac);
        vload(Bv + s0 * a.pitch + col, bc);
        vload(A + (s0 + 1) * a.pitch + col, a2);
        vload(Bv + (s0 + 1) * a.pitch + col, b2);
        T xr = rok ? A[s0 * a.pitch + rcol] : (T)0, yr = rok ? Bv[s0 * a.pitch + rcol] : (T)0;
        T x2 = rok ? A[(s0 + 1) * a.pitch + rcol] : (T)0, y2 = rok ? Bv[(s0 + 1) * a.pitch + rcol] : (T)0;
        for (int s = s0; s < s1; ++s) {
            const int64_t g = a.r0 + s - 1;
#pragma unroll
            for (int k = 0; k < V; ++k) {
                an[k] = a2[k];
                bn[k] = b2[k];
            }
            const T xn = x2, yn = y2;
            if (s + 2 <= a.rows + 1) {
                vload(A + (s + 2) * a.pitch + col, a2);
                vload(Bv + (s + 2) * a.pitch + col, b2);
                x2 = rok ? A[(s + 2) * a.pitch + rcol] : (T)0;
                y2 = rok ? Bv[(s + 2) * a.pitch + rcol] : (T)0;
            }
            T ar = __shfl_down_sync(0xffffffffu, ac[0], 1);
            T br = __shfl_down_sync(0xffffffffu, bc[0], 1);
            if (lane == 31) {
                ar = xr;
                br = yr;
            }
            T c1d[V], c2d[V];
            if (MODE == MODE_DENSE) {
                vload(C1 + s * a.pitch + col, c1d);
                vload(C2 + (s + 1) * a.pitch + col, c2d);
            }
            const bool row_int = (g >= 1) && (g <= a.ny - 2);
            const bool yface = (g <= a.ny - 2);
#pragma unroll
            for (int k = 0; k < V; ++k) {
                const double a0 = (double)ac[k], b0 = (double)bc[k];
                if (row_int && colint[k]) {
                    const double d = a0 - b0;
                    acc += d * d;
                }
                if (row_int && xface[k]) {
                    const double a1 = (double)((k == V - 1) ? ar : ac[k + 1]);
                    const double b1 = (double)((k == V - 1) ? br : bc[k + 1]);
                    const double c = (MODE == MODE_LINE) ? (double)c1l[k] : (double)c1d[k];
                    acc += (c * (a1 - a0)) * (b1 - b0);
                }
                if (yface && colint[k]) {
                    const double c = (MODE == MODE_LINE) ? (double)c2l[k] : (double)c2d[k];
                    acc += (c * ((double)an[k] - a0)) * ((double)bn[k] - b0);
                }
            }
            xr = xn;
            yr = yn;
#pragma unroll
            for (int k = 0; k < V; ++k) {
                ac[k] = an[k];
                bc[k] = bn[k];
            }
        }
    }
    __shared__ double red[8];
    acc = warp_sum(acc);
    if (lane == 0) red[warp] = acc;
    __syncthreads();
    if (threadIdx.x < 32) {
        double v = (threadIdx.x < 8) ? red[threadIdx.x] : 0.0;
        v = warp_sum(v);
        if (threadIdx.x == 0) partial[b * a.items_per_member + item] = v;
    }
}

// Final pass: one warp per member sums its partials in a fixed order (deterministic) and scales.
__global__ void k_energy_final(const double* __restrict__ partial, int nblk, double w, double* __restrict__ out) {
    const int b = blockIdx.x;
    double v = 0.0;
    for (int k = threadIdx.x; k < nblk; k += 32) v += partial[b * nblk + k];
    v = warp_sum(v);
    if (threadIdx.x == 0) out[b] = w * v;
}

// ------------------------------------------------------------------------------------------
// S6: second-wave amplitude (R18) — max/min of fl_T(u_b − u_bg) over x_i ≤ xs − ε_b with the
// first (smallest global row-major index) extremum; warp shuffle arg-reductions.
// ------------------------------------------------------------------------------------------
struct Wave2Args {
    int dim;
    const void* u;
    int64_t nx, ny, r0, pitch, mstride, ny_local;
    int bg;
    double dx, xs;
    const double* eps;  // [B] device
    int nblk;           // CTAs per member = tiles × chunks
    int64_t tiles;      // column tiles of 256·V columns
    int32_t rows_per_chunk;
};

struct ArgVal {
    double v;
    long long i;
};
__device__ __forceinline__ void arg_better_max(double& v, long long& i, double v2, long long i2) {
    if (i2 >= 0 && (i < 0 || v2 > v || (v2 == v && i2 < i))) { v = v2; i = i2; }
}
__device__ __forceinline__ void arg_better_min(double& v, long long& i, double v2, long long i2) {
    if (i2 >= 0 && (i < 0 || v2 < v || (v2 == v && i2 < i))) { v = v2; i = i2; }
}

// A CTA owns a tile of 256·V columns (V = 16 bytes per thread) and a chunk of rows of one member:
// 128-bit loads along rows, the region test once per column, tiles wholly outside the region
// skipped (only the region's nodes are read).  Within a thread rows and columns are visited in
// increasing row-major order and only a strictly better value replaces the running one, so the
// first extremum is kept; CTAs and the final pass break ties by the smaller index.
template <typename T>
__global__ void __launch_bounds__(256) k_wave2(Wave2Args a, ArgVal* __restrict__ partial) {
    constexpr int V = Vec16<T>::N;
    const int b = blockIdx.y;
    const T* U = static_cast<const T*>(a.u) + b * a.mstride;
    const T* G = static_cast<const T*>(a.u) + a.bg * a.mstride;
    const double xlim = a.xs - a.eps[b];
    const int64_t tile = blockIdx.x % a.tiles;
    const int chunk = int(blockIdx.x / a.tiles);
    const int64_t col = (tile * 256 + threadIdx.x) * V;
    const int64_t rows = (a.dim == 1) ? 1 : a.ny_local;
    const int64_t r_lo = int64_t(chunk) * a.rows_per_chunk;
    const int64_t r_hi = min(r_lo + int64_t(a.rows_per_chunk), rows);
    double vmax = 0.0, vmin = 0.0;
    long long imax = -1, imin = -1;
    bool inreg[V];
    bool any = false;
#pragma unroll
    for (int k = 0; k < V; ++k) {
        inreg[k] = (col + k < a.nx) && (grid_node(col + k, a.nx, a.dx) <= xlim);
        any = any || inreg[k];
    }
    if (any && sizeof(T) == 8) {
        for (int64_t r = r_lo; r < r_hi; ++r) {
            const int64_t s = (a.dim == 1) ? 0 : 1 + r;
            const int64_t g = (a.dim == 1) ? 0 : a.r0 + r;
            T uv[V], gv[V];
            vload(U + s * a.pitch + col, uv);
            vload(G + s * a.pitch + col, gv);
#pragma unroll
            for (int k = 0; k < V; ++k) {
                if (!inreg[k]) continue;
                const double d = (double)r_sub(uv[k], gv[k]);
                const long long gi = (long long)(g * a.nx + col + k);
                if (imax < 0 || d > vmax) { vmax = d; imax = gi; }
                if (imin < 0 || d < vmin) { vmin = d; imin = gi; }
            }
        }
    } else if (any) {
        // fp32: software-pipelined — the next row's two 16-byte loads are issued before this row's
        // compare chain (two rows in flight per thread): 0.352 → 0.242 ms on config 5 (the same
        // change made fp64 slower: 0.334 → 0.38 ms, so fp64 keeps the plain loop)
        const int64_t s_of = (a.dim == 1) ? 0 : 1;
        T uv[V], gv[V], un[V], gn[V];
        if (r_lo < r_hi) {
            vload(U + (s_of + r_lo) * a.pitch + col, un);
            vload(G + (s_of + r_lo) * a.pitch + col, gn);
        }
        for (int64_t r = r_lo; r < r_hi; ++r) {
            const int64_t g = (a.dim == 1) ? 0 : a.r0 + r;
#pragma unroll
            for (int k = 0; k < V; ++k) {
                uv[k] = un[k];
                gv[k] = gn[k];
            }
            if (r + 1 < r_hi && a.dim != 1) {
                vload(U + (s_of + r + 1) * a.pitch + col, un);
                vload(G + (s_of + r + 1) * a.pitch + col, gn);
            }
            const long long gbase = (long long)(g * a.nx + col);
#pragma unroll
            for (int k = 0; k < V; ++k) {
                if (!inreg[k]) continue;
                const double d = (double)r_sub(uv[k], gv[k]);
                if (imax < 0 || d > vmax) { vmax = d; imax = gbase + k; }
                if (imin < 0 || d < vmin) { vmin = d; imin = gbase + k; }
            }
        }
    }
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) {
        double v2 = __shfl_xor_sync(0xffffffffu, vmax, o);
        long long i2 = __shfl_xor_sync(0xffffffffu, imax, o);
        arg_better_max(vmax, imax, v2, i2);
        v2 = __shfl_xor_sync(0xffffffffu, vmin, o);
        i2 = __shfl_xor_sync(0xffffffffu, imin, o);
        arg_better_min(vmin, imin, v2, i2);
    }
    __shared__ ArgVal smax[32], smin[32];
    const int w = threadIdx.x >> 5;
    if ((threadIdx.x & 31) == 0) {
        smax[w] = {vmax, imax};
        smin[w] = {vmin, imin};
    }
    __syncthreads();
    if (threadIdx.x == 0) {
        double bv = 0.0, cv = 0.0;
        long long bi = -1, ci = -1;
        for (int k = 0; k < int(blockDim.x >> 5); ++k) {
            arg_better_max(bv, bi, smax[k].v, smax[k].i);
            arg_better_min(cv, ci, smin[k].v, smin[k].i);
        }
        partial[(b * a.nblk + blockIdx.x) * 2 + 0] = {bv, bi};
        partial[(b * a.nblk + blockIdx.x) * 2 + 1] = {cv, ci};
    }
}

__global__ void k_wave2_final(const ArgVal* __restrict__ partial, int nblk, double* __restrict__ out,
                              long long* __restrict__ idx) {
    const int b = blockIdx.x;
    if (threadIdx.x != 0) return;
    double bv = 0.0, cv = 0.0;
    long long bi = -1, ci = -1;
    for (int k = 0; k < nblk; ++k) {
        arg_better_max(bv, bi, partial[(b * nblk + k) * 2].v, partial[(b * nblk + k) * 2].i);
        arg_better_min(cv, ci, partial[(b * nblk + k) * 2 + 1].v, partial[(b * nblk + k) * 2 + 1].i);
    }
    out[2 * b] = (bi >= 0) ? bv : 0.0;
    out[2 * b + 1] = (ci >= 0) ? cv : 0.0;
    idx[2 * b] = bi;
    idx[2 * b + 1] = ci;
}

// ------------------------------------------------------------------------------------------
// NEXT 2 diagnostics of an ε-family: pairwise L² distances (§3.2.1,
// P:831–838 ‖u_{ε1}(t) − u_{ε2}(t)‖_{L²}), the L² pieces of Theorem lem 1's energy estimate
// and the W^{1,∞} norms of the regularised depth (Assumption).
// ------------------------------------------------------------------------------------------
// Pairwise Σ_nodes (u_i − u_j)²: a dense all-pairs reduction, bound by the fp64 pipe (a
// subtraction and a fused multiply-add per member pair and node), not by HBM.  A thread owns the
// 4 × 4 accumulators of one block of member pairs (I ≤ J; register blocking: 8 shared-memory
// loads for 16 pairs); a CTA holds up to 512 consecutive blocks (blockIdx.y: the group of blocks,
// for batches above 88) and a contiguous range of node tiles (blockIdx.x).  Tiles of FAM_TN nodes
// of all B members are double-buffered in shared memory, the next one prefetched into registers
// while the current one is consumed (one barrier per tile).  Member m's row starts at
// m·FAM_TP + (m >> 2): consecutive pair blocks of a warp read rows 4J + k whose starts differ by
// 4·FAM_TP + 1 ≡ 1 (mod 16) doubles, i.e. distinct banks; lanes of one I share x (broadcast).
// Member rows B .. 4·nblk − 1 stay zero.
constexpr int FAM_TN = 32;                 // nodes per tile
constexpr int FAM_TP = FAM_TN;             // row pitch (a multiple of 4: see the skew above)
constexpr int FAM_EPT = 16;                // prefetch registers per thread: B · FAM_TN ≤ 16 · threads
constexpr int FAM_MAXT = 512;              // threads per CTA (≤ 512 blocks per group)
struct FamilyArgs {
    const void* u;
    int64_t nx, pitch, mstride;
    int32_t rows;      // rows of the slab (1D: 1)
    int32_t row0;      // first storage row (2D: 1, 1D: 0)
    int32_t B, nblk;   // members, member blocks of 4
    int64_t tiles_per_row;
    int64_t ntiles, tiles_per_cta;
};
__host__ __device__ constexpr int fam_rows_elems(int nblk) { return 4 * nblk * FAM_TP + nblk; }

template <typename T>
__global__ void __launch_bounds__(FAM_MAXT) k_family_l2(const FamilyArgs a, double* __restrict__ partial) {
    extern __shared__ __align__(16) double fam_smem[];   // [2][fam_rows_elems(nblk)]
    const int nt = blockDim.x;
    const int tid = threadIdx.x;
    const int BUF = fam_rows_elems(a.nblk);
    const int npairs = a.nblk * (a.nblk + 1) / 2;
    const int p = blockIdx.y * nt + tid;                  // my pair block
    const bool owner = p < npairs;
    int I = 0, J = 0;
    if (owner) {
        int q = p, row = 0;
        while (q >= a.nblk - row) { q -= a.nblk - row; ++row; }
        I = row;
        J = row + q;
    }
    double acc[4][4];
#pragma unroll
    for (int k = 0; k < 4; ++k)
#pragma unroll
        for (int l = 0; l < 4; ++l) acc[k][l] = 0.0;
    for (int e = tid; e < 2 * BUF; e += nt) fam_smem[e] = 0.0;   // padding rows stay 0
    const T* U = static_cast<const T*>(a.u);
    const int64_t t0 = int64_t(blockIdx.x) * a.tiles_per_cta;
    const int64_t t1 = min(t0 + a.tiles_per_cta, a.ntiles);
    const int nel = a.B * FAM_TN;
    // fp64: the next tile goes straight to shared memory (cp.async, zero-filled past the row end:
    // no prefetch registers, more CTAs per SM); fp32: through registers (converted on the store)
    constexpr bool ASYNC = sizeof(T) == 8;
    auto fetch_async = [&](int64_t t, int buf) {
        const int64_t r = a.row0 + t / a.tiles_per_row;
        const int64_t c0 = (t % a.tiles_per_row) * FAM_TN;
        const T* base = U + r * a.pitch + c0;
        const int64_t lim = a.nx - c0;
        double* tb = fam_smem + buf * BUF;
        for (int e = tid; e < nel; e += nt) {
            const int m = e / FAM_TN, cc = e % FAM_TN;
            const bool in = cc < lim;
            const uint32_t dst = smem_u32(tb + m * FAM_TP + (m >> 2) + cc);
            const T* src = in ? base + m * a.mstride + cc : base;
            asm volatile("cp.async.ca.shared.global [%0], [%1], 8, %2;" ::"r"(dst), "l"(src), "r"(in ? 8 : 0)
                         : "memory");
        }
        asm volatile("cp.async.commit_group;" ::: "memory");
    };
    T pf[ASYNC ? 1 : FAM_EPT];
    auto fetch = [&](int64_t t) {
        const int64_t r = a.row0 + t / a.tiles_per_row;
        const int64_t c0 = (t % a.tiles_per_row) * FAM_TN;
        const T* base = U + r * a.pitch + c0;
        const int64_t lim = a.nx - c0;
#pragma unroll
        for (int q = 0; q < (ASYNC ? 1 : FAM_EPT); ++q) {
            const int e = tid + q * nt;
            pf[q] = (T)0;
            if (e < nel) {
                const int m = e / FAM_TN, cc = e % FAM_TN;
                if (cc < lim) pf[q] = __ldg(base + m * a.mstride + cc);
            }
        }
    };
    auto stash = [&](int buf) {
        double* tb = fam_smem + buf * BUF;
#pragma unroll
        for (int q = 0; q < (ASYNC ? 1 : FAM_EPT); ++q) {
            const int e = tid + q * nt;
            if (e < nel) {
                const int m = e / FAM_TN, cc = e % FAM_TN;
                tb[m * FAM_TP + (m >> 2) + cc] = (double)pf[q];
            }
        }
    };
    __syncthreads();   // the zero fill precedes the first stash
    if (t0 < t1) {
        if constexpr (ASYNC) {
            fetch_async(t0, 0);
            asm volatile("cp.async.wait_all;" ::: "memory");
        } else {
            fetch(t0);
            stash(0);
        }
    }
    __syncthreads();
    for (int64_t t = t0; t < t1; ++t) {
        const int buf = int(t - t0) & 1;
        if (t + 1 < t1) {   // in flight during the arithmetic below (buffer buf ^ 1 was last read
                            // before the previous barrier)
            if constexpr (ASYNC) fetch_async(t + 1, buf ^ 1);
            else fetch(t + 1);
        }
        if (owner) {
            const double* tb = fam_smem + buf * BUF;
            const double* xr = tb + 4 * I * FAM_TP + I;
            const double* yr = tb + 4 * J * FAM_TP + J;
#pragma unroll 4
            for (int n = 0; n < FAM_TN; ++n) {
                double x[4], y[4];
#pragma unroll
                for (int k = 0; k < 4; ++k) {
                    x[k] = xr[k * FAM_TP + n];
                    y[k] = yr[k * FAM_TP + n];
                }
#pragma unroll
                for (int k = 0; k < 4; ++k)
#pragma unroll
                    for (int l = 0; l < 4; ++l) {
                        const double d = x[k] - y[l];
                        acc[k][l] = __fma_rn(d, d, acc[k][l]);
                    }
            }
        }
        if (t + 1 < t1) {
            if constexpr (ASYNC) asm volatile("cp.async.wait_all;" ::: "memory");
            else stash(buf ^ 1);
        }
        __syncthreads();
    }
    if (owner) {
        double* out = partial + size_t(blockIdx.x) * a.B * a.B;
#pragma unroll
        for (int k = 0; k < 4; ++k)
#pragma unroll
            for (int l = 0; l < 4; ++l) {
                const int i = 4 * I + k, j = 4 * J + l;
                if (i < a.B && j < a.B && i < j) out[i * a.B + j] = acc[k][l];
            }
    }
}

// out[i][j] = out[j][i] = sqrt(w · Σ_cta partial[cta][i][j]) (fixed order), diagonal 0.
// out[i][j] = Σ_k partial[k][i][j] (fixed order) for i < j, mirrored; 0 on the diagonal — the
// unweighted sums Σ (u_i − u_j)² (summed over ranks, weighted and rooted by the caller)
__global__ void k_family_final(const double* __restrict__ partial, int ncta, int B, double* __restrict__ out) {
    for (int e = blockIdx.x * blockDim.x + threadIdx.x; e < B * B; e += gridDim.x * blockDim.x) {
        const int i = e / B, j = e % B;
        if (i >= j) continue;
        double s = 0.0;
        for (int k = 0; k < ncta; ++k) s += partial[size_t(k) * B * B + e];
        out[i * B + j] = s;
        out[j * B + i] = s;
    }
    if (blockIdx.x == 0)
        for (int i = threadIdx.x; i < B; i += blockDim.x) out[i * B + i] = 0.0;
}

// Σ u², Σ (u − u_prev)², Σ (Δx u)², Σ (Δy u)² per member (all nodes / all faces of the slab).
struct NormArgs {
    int dim;
    const void* un;
    const void* unm1;
    int64_t nx, ny, r0, pitch, mstride;
    int32_t rows;
    int nblk;
};

template <typename T>
__global__ void __launch_bounds__(256) k_norms(const NormArgs a, double* __restrict__ partial) {
    const int b = blockIdx.y;
    const T* A = static_cast<const T*>(a.un) + b * a.mstride;
    const T* P = static_cast<const T*>(a.unm1) + b * a.mstride;
    double s[4] = {0.0, 0.0, 0.0, 0.0};
    const int64_t total = int64_t(a.rows) * a.nx;
    for (int64_t k = blockIdx.x * int64_t(blockDim.x) + threadIdx.x; k < total; k += int64_t(gridDim.x) * blockDim.x) {
        const int64_t i = k % a.nx;
        const int64_t sr = (a.dim == 1) ? 0 : 1 + k / a.nx;
        const int64_t g = (a.dim == 1) ? 0 : a.r0 + sr - 1;
        const int64_t o = sr * a.pitch + i;
        const double u = (double)A[o], p = (double)P[o];
        s[0] += u * u;
        s[1] += (u - p) * (u - p);
        if (i <= a.nx - 2) {
            const double d = (double)A[o + 1] - u;
            s[2] += d * d;
        }
        if (a.dim == 2 && g <= a.ny - 2) {
            const double d = (double)A[o + a.pitch] - u;
            s[3] += d * d;
        }
    }
    __shared__ double red[4][8];
    const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
#pragma unroll
    for (int q = 0; q < 4; ++q) {
        const double v = warp_sum(s[q]);
        if (lane == 0) red[q][w] = v;
    }
    __syncthreads();
    if (threadIdx.x < 4) {
        double v = 0.0;
        for (int k = 0; k < int(blockDim.x >> 5); ++k) v += red[threadIdx.x][k];
        partial[(size_t(b) * a.nblk + blockIdx.x) * 4 + threadIdx.x] = v;
    }
}

__global__ void k_norms_final(const double* __restrict__ partial, int nblk, int B, double* __restrict__ out) {
    const int b = blockIdx.x, q = threadIdx.x;
    if (q >= 4) return;
    double v = 0.0;
    for (int k = 0; k < nblk; ++k) v += partial[(size_t(b) * nblk + k) * 4 + q];
    out[b * 4 + q] = v;
}

// W^{1,∞}: sup |h| over all stored faces and sup |∇h| from the analytic derivative of the
// regulariser at the x faces (φ_ε′(d) = φ_ε(d)·(−2t/((t²−1)²·ε)), t = d/ε).
__device__ __forceinline__ double dphi_eps(double d, double eps) {
    const double t = d / eps;
    if (!(fabs(t) < 1.0)) return 0.0;
    const double q = t * t - 1.0;
    return phi_eps(d, eps) * (-2.0 * t / (q * q * eps));
}

struct CoeffNormArgs {
    int kind, order;
    double hb, xs, ys, dx, dy;
    const double* eps;
    const double* amp;     // δ kinds: amplitude per member; profile: scale per member
    const double* prof;    // profile data (kind 4) or nullptr
    int nseg, nsing;
    const double* h1;
    const double* h2;
    int64_t nx, ny, r0, rows, pitch, cstride1, cstride2, mstride;
    int mode;
};

__global__ void k_coeff_norms(const CoeffNormArgs a, unsigned long long* __restrict__ out /* [B][3] */) {
    const int b = blockIdx.y;
    const double eps = a.eps[b], am = a.amp[b];
    double mh = 0.0, md = 0.0, mh2 = 0.0;
    const int64_t nrow = (a.mode == MODE_LINE) ? 1 : a.rows;
    const int64_t total = nrow * a.nx;
    for (int64_t k = blockIdx.x * int64_t(blockDim.x) + threadIdx.x; k < total; k += int64_t(gridDim.x) * blockDim.x) {
        const int64_t i = k % a.nx;
        const int64_t sr = (a.mode == MODE_LINE) ? 0 : 1 + k / a.nx;
        if (i <= a.nx - 2) {
            const double h = (a.mode == MODE_LINE) ? a.h1[b * a.cstride1 + i] : a.h1[b * a.cstride1 + sr * a.pitch + i];
            mh = fmax(mh, fabs(h));
            const double x = grid_face(i, a.nx, a.dx);
            double d = 0.0;
            if (a.kind == 1) {
                const double p = phi_eps(x - a.xs, eps), q = dphi_eps(x - a.xs, eps);
                d = am * ((a.order == 2) ? 2.0 * p * q : q);
            } else if (a.kind == 2) {
                const double y = grid_node(a.r0 + sr - 1, a.ny, a.dy);
                const double px = phi_eps(x - a.xs, eps), py = phi_eps(y - a.ys, eps);
                const double gx = dphi_eps(x - a.xs, eps) * py, gy = px * dphi_eps(y - a.ys, eps);
                const double f = (a.order == 2) ? 2.0 * px * py : 1.0;
                d = am * f * sqrt(gx * gx + gy * gy);
            } else if (a.kind == 4) {
                const double* v = a.prof;
                const double* br = v + a.nseg;
                const double* loc = br + (a.nseg - 1);
                const double* amp = loc + a.nsing;
                const double* ord = amp + a.nsing;
                for (int s = 1; s < a.nseg; ++s) d += (v[s] - v[s - 1]) * phi_eps(x - br[s - 1], eps);
                for (int j = 0; j < a.nsing; ++j) {
                    const double p = phi_eps(x - loc[j], eps), q = dphi_eps(x - loc[j], eps);
                    d += am * amp[j] * ((ord[j] == 2.0) ? 2.0 * p * q : q);
                }
            } else if (i >= 1) {  // caller faces: finite difference at node i
                const double* hr = a.h1 + b * a.cstride1 + ((a.mode == MODE_LINE) ? 0 : sr * a.pitch);
                d = (hr[i] - hr[i - 1]) / a.dx;
            }
            md = fmax(md, fabs(d));
        }
        if (a.h2) {
            const double h = (a.mode == MODE_LINE) ? a.h2[b * a.cstride2 + i] : a.h2[b * a.cstride2 + sr * a.pitch + i];
            mh2 = fmax(mh2, fabs(h));
        }
    }
    mh = warp_max(mh);
    md = warp_max(md);
    mh2 = warp_max(mh2);
    if ((threadIdx.x & 31) == 0) {
        atomic_max_pos(&out[b * 3 + 0], mh);
        atomic_max_pos(&out[b * 3 + 1], md);
        atomic_max_pos(&out[b * 3 + 2], mh2);
    }
}

// ------------------------------------------------------------------------------------------
// NEXT 3: the paper's 2D method (§3.3 P:1140 "implicit finite difference scheme and the
// cyclic reduction method"; Table 1) — reading R26: factorised three-level CN
//   (I − ½L_x)(I − ½L_y)(u^{n+1} + u^{n−1}) = 2u^n,   start (R27) u¹ = B⁻¹u⁰ + dt·u₁.
// Line solves by cyclic reduction (Hockney–Golub) with the whole line resident in shared memory:
// one CTA per line, a/b/c/d arrays of N = 2^q − 1 ≥ m entries (identity padding).
// ------------------------------------------------------------------------------------------
struct CrArgs {
    const void* src;   // right-hand side lines (rows of a [B][rows][pitch] array, view row 1 = first)
    void* dst;         // solution lines (may alias src)
    const void* cf;    // DIR 0: c1 [B][cpitch] x faces;  DIR 1: c2 [B][cpitch] one value per line
    int64_t pitch, mstride, cpitch;
    int64_t m;         // unknowns per line (line length − 2)
    int32_t q;         // N = 2^q − 1 ≥ m
    int32_t row0;      // first line (array row) to solve; lines row0 .. row0 + nlines − 1
    int32_t nlines;
    int32_t line_coef0;  // DIR 1: coefficient index of line row0 (the original column index)
    double scale;      // rhs = scale · src
};

template <typename T, int DIR>
__global__ void __launch_bounds__(512) k_cr_rows(const CrArgs a) {
    extern __shared__ __align__(16) unsigned char smem_raw[];
    const int N = (1 << a.q) - 1;
    T* A = reinterpret_cast<T*>(smem_raw);
    T* Bd = A + N;
    T* C = Bd + N;
    T* D = C + N;
    const int line = blockIdx.x;
    const int b = blockIdx.y;
    const int64_t row = a.row0 + line;
    const T* src = static_cast<const T*>(a.src) + b * a.mstride + row * a.pitch;
    T* dst = static_cast<T*>(a.dst) + b * a.mstride + row * a.pitch;
    const T* cf = static_cast<const T*>(a.cf) + b * a.cpitch;
    const T half = (T)0.5, one = (T)1, sc = (T)a.scale;
    for (int i = threadIdx.x; i < N; i += blockDim.x) {
        if (i < a.m) {
            T cl, cr;
            if (DIR == 0) {
                cl = cf[i];       // face (i+1) − 1/2 of line position i+1
                cr = cf[i + 1];   // face (i+1) + 1/2
            } else {
                cl = cr = cf[a.line_coef0 + line];
            }
            A[i] = (i == 0) ? (T)0 : -(half * cl);
            C[i] = (i == a.m - 1) ? (T)0 : -(half * cr);
            Bd[i] = one + half * (cl + cr);
            D[i] = sc * src[i + 1];
        } else {
            A[i] = (T)0;
            C[i] = (T)0;
            Bd[i] = one;
            D[i] = (T)0;
        }
    }
    // forward reduction: level l updates i = k·2^l − 1 from i ± 2^{l−1}
    for (int l = 1; l < a.q; ++l) {
        __syncthreads();
        const int h = 1 << (l - 1), s = 1 << l;
        for (int k = 1 + threadIdx.x; k * s - 1 < N; k += blockDim.x) {
            const int i = k * s - 1;
            const T al = -A[i] / Bd[i - h];
            const T ga = -C[i] / Bd[i + h];
            const T na = al * A[i - h];
            const T nc = ga * C[i + h];
            const T nb = Bd[i] + al * C[i - h] + ga * A[i + h];
            const T nd = D[i] + al * D[i - h] + ga * D[i + h];
            A[i] = na;
            C[i] = nc;
            Bd[i] = nb;
            D[i] = nd;
        }
    }
    __syncthreads();
    if (threadIdx.x == 0) {
        const int r = (1 << (a.q - 1)) - 1;
        D[r] = D[r] / Bd[r];
    }
    // back substitution: level l solves i = h − 1 + k·2^l (h = 2^{l−1}) from i ± h
    for (int l = a.q - 1; l >= 1; --l) {
        __syncthreads();
        const int h = 1 << (l - 1), s = 1 << l;
        for (int k = threadIdx.x; h - 1 + k * s < N; k += blockDim.x) {
            const int i = h - 1 + k * s;
            const T xl = (i - h >= 0) ? D[i - h] : (T)0;
            const T xr = (i + h < N) ? D[i + h] : (T)0;
            D[i] = (D[i] - A[i] * xl - C[i] * xr) / Bd[i];
        }
    }
    __syncthreads();
    for (int i = threadIdx.x; i < a.m; i += blockDim.x) dst[i + 1] = D[i];
    if (threadIdx.x == 0) {
        dst[0] = (T)0;
        dst[a.m + 1] = (T)0;
    }
}

// Tiled transpose of the storage rows 1..ny (global rows 0..ny−1) × columns 0..nx−1 of every
// member: out[b][i][j] = in[b][1 + j][i] (out row i = original column i, pitch pt).
template <typename T>
__global__ void k_transpose(const T* __restrict__ in, T* __restrict__ out, int64_t nx, int64_t ny, int64_t pitch,
                            int64_t mstride, int64_t pt, int64_t tstride) {
    __shared__ T tile[32][33];
    const int b = blockIdx.z;
    const int64_t i0 = int64_t(blockIdx.x) * 32, j0 = int64_t(blockIdx.y) * 32;
    const T* ib = in + b * mstride;
    T* ob = out + b * tstride;
    for (int r = threadIdx.y; r < 32; r += blockDim.y) {
        const int64_t j = j0 + r, i = i0 + threadIdx.x;
        tile[r][threadIdx.x] = (j < ny && i < nx) ? ib[(1 + j) * pitch + i] : (T)0;
    }
    __syncthreads();
    for (int r = threadIdx.y; r < 32; r += blockDim.y) {
        const int64_t i = i0 + r, j = j0 + threadIdx.x;
        if (i < nx && j < pt) ob[i * pt + j] = tile[threadIdx.x][r];
    }
}

// Transpose back the y-solved w and finish the level on the interior nodes, in place in `prev`:
//   MODE 0: u^{n+1} = w − u^{n−1}   (prev holds u^{n−1});   MODE 1: u¹ = w + dt·u₁ (prev holds u₁).
template <typename T, int MODE>
__global__ void k_transpose_finish(const T* __restrict__ wt, T* __restrict__ prev, int64_t nx, int64_t ny,
                                   int64_t pitch, int64_t mstride, int64_t pt, int64_t tstride, T dtT) {
    __shared__ T tile[32][33];
    const int b = blockIdx.z;
    const int64_t i0 = int64_t(blockIdx.x) * 32, j0 = int64_t(blockIdx.y) * 32;
    const T* wb = wt + b * tstride;
    T* pb = prev + b * mstride;
    for (int r = threadIdx.y; r < 32; r += blockDim.y) {
        const int64_t i = i0 + r, j = j0 + threadIdx.x;
        tile[r][threadIdx.x] = (i < nx && j < ny) ? wb[i * pt + j] : (T)0;
    }
    __syncthreads();
    for (int r = threadIdx.y; r < 32; r += blockDim.y) {
        const int64_t j = j0 + r, i = i0 + threadIdx.x;
        if (j >= 1 && j <= ny - 2 && i >= 1 && i <= nx - 2) {
            T* p = pb + (1 + j) * pitch + i;
            const T w = tile[threadIdx.x][r];
            *p = (MODE == 0) ? r_sub(w, *p) : r_add(w, r_mul(dtT, *p));
        }
    }
}

// 1D implicit level: one thread per member runs the Thomas algorithm on its line (three-level CN
// (I − ½L_x)(u^{n+1} + u^{n−1}) = 2u^n).  MODE 0: rhs 2u^n, result w − u^{n−1};  MODE 1: rhs u⁰,
// result w + dt·u₁ (R27).  The result is written in place over `prev`.  cp/dp: [B][pitch] scratch.
template <typename T, int MODE>
__global__ void k_implicit_1d(const T* __restrict__ un, T* __restrict__ prev, const T* __restrict__ c1, int64_t nx,
                              int64_t pitch, int64_t cpitch, T* __restrict__ cp, T* __restrict__ dp, int B, T dtT) {
    const int b = blockIdx.x * blockDim.x + threadIdx.x;
    if (b >= B) return;
    const T* u = un + b * pitch;
    T* p = prev + b * pitch;
    const T* c = c1 + b * cpitch;
    T* cq = cp + b * pitch;
    T* dq = dp + b * pitch;
    const T half = (T)0.5;
    const int64_t m = nx - 2;
    for (int64_t i = 1; i <= m; ++i) {
        const T cl = c[i - 1], cr = c[i];
        const T a = -r_mul(half, cl), bb = r_add((T)1, r_mul(half, r_add(cl, cr))), cc = -r_mul(half, cr);
        const T d = (MODE == 0) ? r_mul((T)2, u[i]) : u[i];
        if (i == 1) {
            cq[i] = cc / bb;
            dq[i] = d / bb;
        } else {
            const T den = r_sub(bb, r_mul(a, cq[i - 1]));
            cq[i] = cc / den;
            dq[i] = r_sub(d, r_mul(a, dq[i - 1])) / den;
        }
    }
    T x = dq[m];
    for (int64_t i = m; i >= 1; --i) {
        if (i < m) x = r_sub(dq[i], r_mul(cq[i], x));
        p[i] = (MODE == 0) ? r_sub(x, p[i]) : r_add(x, r_mul(dtT, p[i]));
    }
}

// ------------------------------------------------------------------------------------------
// Implicit scheme, scan solvers (NEXT 3, R28).  Both factors of B = (I − ½L_x)(I − ½L_y) have
// coefficients that depend on x only (δ-line / profile kinds), which the line solvers exploit:
//  * x lines: one tridiagonal matrix shared by every row.  Its LU (l_p, 1/u_p, e_p = c_p/u_p) is
//    computed once (k_imp_xfactor); each row then needs the two first-order recurrences
//    y_p = d_p − l_p y_{p−1} and x_p = y_p/u_p − e_p x_{p+1}, run as affine scans across a CTA
//    (warp shuffles inside a 32-position sub-block, sub-blocks in sequence per warp, warp totals
//    through shared memory) — coalesced, in place along the row, no transposes (k_imp_x).
//  * y lines: column i is Toeplitz, T = tridiag(−γ/2, 1 + γ, −γ/2) with γ = c2(i), and
//    T = κ[(I − ρS)(I − ρSᵀ) + ρ² e₁e₁ᵀ] (κρ = γ/2, κ(1 + ρ²) = 1 + γ, 0 ≤ ρ < 1), so
//    T⁻¹r = (1/κ)[z − β z₁ P⁻¹e₁] with z = P⁻¹r = (L_j + R_j − ρ^{m+1−j}A₂)/(1 − ρ²),
//    L_j = Σ_{i≤j} ρ^{j−i} r_i, R_j = Σ_{i>j} ρ^{i−j} r_i, A₂ = Σ ρ^{m+1−i} r_i,
//    z₁ = (A₁ − ρ^m A₂)/(1 − ρ²), A₁ = Σ ρ^{i−1} r_i, β = ρ²/(1 + ρ²(1 − ρ^{2m})/(1 − ρ²)),
//    P⁻¹e₁ = (ρ^{j−1} − ρ^{2m+1−j})/(1 − ρ²): exponential scans with a constant factor per column,
//    done column-parallel in place (k_imp_y), fused with the three-level update.
// All recurrences have |factor| < 1 (diagonal dominance), so the scans are stable.
// ------------------------------------------------------------------------------------------
__device__ __forceinline__ double fmaT(double a, double b, double c) { return __fma_rn(a, b, c); }
__device__ __forceinline__ float fmaT(float a, float b, float c) { return __fmaf_rn(a, b, c); }

template <typename T>
__device__ __forceinline__ T powi_T(T x, int n) {  // x^n, n ≥ 0, by squaring (0^0 = 1)
    T r = (T)1;
    while (n > 0) {
        if (n & 1) r = r * x;
        x = x * x;
        n >>= 1;
    }
    return r;
}

// LU of the x-line matrix of member b (one thread per member): unknown p ↔ column p + 1,
// a_p = −½c1[p], b_p = 1 + ½(c1[p] + c1[p+1]), c_p = −½c1[p+1]; in fp64, stored as T.  The pivots
// u_p = θ_p/θ_{p−1} come from the continuants θ_p = b_p θ_{p−1} − a_p c_{p−1} θ_{p−2} (the leading
// principal minors; growing solution of a three-term recurrence, hence stable), rescaled by exact
// powers of two — one dependent FMA per step instead of a dependent division.
template <typename T>
__global__ void k_imp_xfactor(const T* __restrict__ c1, int64_t cpitch, T* __restrict__ tab, int64_t tpitch, int m,
                              int B) {
    // One CTA per member.  Thread 0 runs the serial continuant recurrence (one FMA per step) and
    // records each pivot as a (numerator, denominator) pair at a common scale; all threads then
    // form l_p, 1/u_p, e_p in parallel.  Shared memory: c (m + 1), num (m), den (m), fp64.
    extern __shared__ __align__(16) unsigned char smem_raw[];
    double* c = reinterpret_cast<double*>(smem_raw);
    double* num = c + (m + 1);
    double* den = num + m;
    const int b = blockIdx.x;
    for (int i = threadIdx.x; i <= m; i += blockDim.x) c[i] = (double)c1[b * cpitch + i];
    __syncthreads();
    if (threadIdx.x == 0) {
        double th2 = 1.0, th1 = 1.0;   // θ_{p−2}, θ_{p−1} (θ_{−1} = 1)
        for (int p = 0; p < m; ++p) {
            const double cl = c[p], cr = c[p + 1];
            const double bb = 1.0 + 0.5 * (cl + cr);
            // a_p c_{p−1} = (−½c[p])(−½c[p]) = ¼c[p]²
            const double th = (p == 0) ? bb : fma(bb, th1, -(0.25 * cl * cl) * th2);
            num[p] = th;
            den[p] = th1;
            th2 = th1;
            th1 = th;
            if ((p & 15) == 15) {  // exact rescale
                const int e = ilogb(th1);
                th1 = scalbn(th1, -e);
                th2 = scalbn(th2, -e);
            }
        }
    }
    __syncthreads();
    T* t = tab + b * 3 * tpitch;
    for (int p = threadIdx.x; p < m; p += blockDim.x) {
        const double u = num[p] / den[p];
        const double cl = c[p], cr = c[p + 1];
        const double l = (p > 0) ? (-0.5 * cl) * (den[p - 1] / num[p - 1]) : 0.0;
        const double cc = (p < m - 1) ? -0.5 * cr : 0.0;
        t[p] = (T)l;
        t[tpitch + p] = (T)(1.0 / u);
        t[2 * tpitch + p] = (T)(cc / u);
    }
}

struct ImpXArgs {
    const void* src;   // right-hand side field (view rows), scaled by `scale`
    void* dst;         // x-solve output z (same layout)
    const void* tab;   // [B][3][tpitch]: l, 1/u, e of unknown p (column p + 1)
    int64_t pitch, mstride, tpitch;
    int32_t nx;
    int32_t row0;      // view row of the first line; lines row0 .. row0 + nrows − 1
    int32_t nrows;
    double scale;
};

constexpr int IMPX_THREADS = 512;
constexpr int IMPX_WARPS = IMPX_THREADS / 32;

// Affine inclusive scan inside a warp, forward (lane 0 → 31): (A, V) ← (A·A_up, V + A·V_up).
template <typename T>
__device__ __forceinline__ void warp_affine_fwd(T& A, T& V, int lane, int from = 1) {
#pragma unroll
    for (int off = 1; off < 32; off <<= 1) {
        if (off < from) continue;
        const T Vu = __shfl_up_sync(0xffffffffu, V, off);
        const T Au = __shfl_up_sync(0xffffffffu, A, off);
        if (lane >= off) {
            V = fmaT(A, Vu, V);
            A = A * Au;
        }
    }
}
template <typename T>
__device__ __forceinline__ void warp_affine_bwd(T& A, T& V, int lane, int from = 1) {
#pragma unroll
    for (int off = 1; off < 32; off <<= 1) {
        if (off < from) continue;
        const T Vd = __shfl_down_sync(0xffffffffu, V, off);
        const T Ad = __shfl_down_sync(0xffffffffu, A, off);
        if (lane + off < 32) {
            V = fmaT(A, Vd, V);
            A = A * Ad;
        }
    }
}

// 32-byte vector accesses (sm_100: LDG/STG .256) for a thread's span of R consecutive columns.
template <typename T>
__device__ __forceinline__ void ld32(const T* p, T* v) {
    if constexpr (sizeof(T) == 8)
        asm volatile("ld.global.v4.f64 {%0,%1,%2,%3}, [%4];" : "=d"(v[0]), "=d"(v[1]), "=d"(v[2]), "=d"(v[3]) : "l"(p));
    else
        asm volatile("ld.global.v8.f32 {%0,%1,%2,%3,%4,%5,%6,%7}, [%8];"
                     : "=f"(v[0]), "=f"(v[1]), "=f"(v[2]), "=f"(v[3]), "=f"(v[4]), "=f"(v[5]), "=f"(v[6]), "=f"(v[7])
                     : "l"(p));
}
template <typename T>
__device__ __forceinline__ void st32(T* p, const T* v) {
    if constexpr (sizeof(T) == 8)
        asm volatile("st.global.v4.f64 [%0], {%1,%2,%3,%4};" ::"l"(p), "d"(v[0]), "d"(v[1]), "d"(v[2]), "d"(v[3]) : "memory");
    else
        asm volatile("st.global.v8.f32 [%0], {%1,%2,%3,%4,%5,%6,%7,%8};" ::"l"(p), "f"(v[0]), "f"(v[1]), "f"(v[2]),
                     "f"(v[3]), "f"(v[4]), "f"(v[5]), "f"(v[6]), "f"(v[7])
                     : "memory");
}

template <typename T, int R>
__device__ __forceinline__ void load_span(const T* __restrict__ row, int c0, int nx, T (&v)[R]) {
    constexpr int W = 32 / int(sizeof(T));  // elements per 32-byte access
    if (c0 + R <= nx && R % W == 0) {
#pragma unroll
        for (int k = 0; k < R; k += W) ld32<T>(row + c0 + k, v + k);
    } else {
#pragma unroll
        for (int k = 0; k < R; ++k) v[k] = (c0 + k < nx) ? row[c0 + k] : (T)0;
    }
}

template <typename T, int R>
__device__ __forceinline__ void store_span(T* __restrict__ row, int c0, int lo, int hi, const T (&v)[R]) {
    // columns [lo, hi) only
    constexpr int W = 32 / int(sizeof(T));
    if (c0 >= lo && c0 + R <= hi && R % W == 0) {
#pragma unroll
        for (int k = 0; k < R; k += W) st32<T>(row + c0 + k, v + k);
    } else {
#pragma unroll
        for (int k = 0; k < R; ++k)
            if (c0 + k >= lo && c0 + k < hi) row[c0 + k] = v[k];
    }
}

// One CTA (blockDim.x = nthreads ≤ 1024, a multiple of 32) solves rows row0 + blockIdx.x +
// k·gridDim.x of member blockIdx.y.  Thread t owns the R consecutive columns [tR, tR + R) — one
// 32-byte access when R·sizeof(T) = 32 (column 0 and columns ≥ nx − 1 carry zero table entries,
// so they stay out of the system) — and keeps their LU table entries in registers.  Per row and
// direction: a sequential local recurrence over the span; a warp-level scan of the span totals in
// which only the values move (the factors are products of LU entries — data-independent — so the
// per-level factors are computed once per CTA and kept in shared memory); the warp totals are
// scanned by one warp; then the fix-up.  Two barriers per row.
constexpr int IMPX_MAXW = 32;

template <typename T, int R>
__global__ void __launch_bounds__(1024, 1) k_imp_x(const ImpXArgs a) {
    __shared__ T fwv[IMPX_MAXW], bwv[IMPX_MAXW];          // warp totals (values) per row
    __shared__ T fwc[IMPX_MAXW], bwc[IMPX_MAXW];          // per-warp carry-in (values) per row
    __shared__ T fwa[IMPX_MAXW], bwa[IMPX_MAXW];          // warp-total factors (constant)
    __shared__ T fxa[5][IMPX_MAXW], bxa[5][IMPX_MAXW];    // cross-warp scan level factors (constant)
    extern __shared__ __align__(16) unsigned char smem_raw[];
    T* lvf = reinterpret_cast<T*>(smem_raw);               // [5][nthreads] intra-warp level factors, forward
    T* lvb = lvf + 5 * blockDim.x;                          // backward
    const int b = blockIdx.y;
    const int nx = a.nx, m = nx - 2;
    const int t = threadIdx.x, nt = blockDim.x;
    const int nwarps = nt >> 5;
    const int c0 = t * R;
    const int lane = t & 31, warp = t >> 5;
    T tl[R], tiu[R], te[R];
    T aexf, aexb;   // product of the span factors of the earlier (later) lanes in the warp
    {
        const T* tab = static_cast<const T*>(a.tab) + b * 3 * a.tpitch;
#pragma unroll
        for (int k = 0; k < R; ++k) {
            const int c = c0 + k;
            const bool ok = c >= 1 && c <= m;
            tl[k] = ok ? -tab[c - 1] : (T)0;                 // stored negated: the recurrence factor
            tiu[k] = ok ? tab[a.tpitch + c - 1] : (T)0;
            te[k] = ok ? -tab[2 * a.tpitch + c - 1] : (T)0;  // negated
        }
        // constant factors of the scans
        T Af = (T)1, Ab = (T)1;
#pragma unroll
        for (int k = 0; k < R; ++k) {
            Af = Af * tl[k];
            Ab = Ab * te[k];
        }
        int lv = 0;
#pragma unroll
        for (int off = 1; off < 32; off <<= 1, ++lv) {
            const T Au = __shfl_up_sync(0xffffffffu, Af, off);
            const T Ad = __shfl_down_sync(0xffffffffu, Ab, off);
            lvf[lv * nt + t] = (lane >= off) ? Af : (T)0;
            lvb[lv * nt + t] = (lane + off < 32) ? Ab : (T)0;
            if (lane >= off) Af = Af * Au;
            if (lane + off < 32) Ab = Ab * Ad;
        }
        aexf = __shfl_up_sync(0xffffffffu, Af, 1);
        aexb = __shfl_down_sync(0xffffffffu, Ab, 1);
        if (lane == 0) aexf = (T)1;
        if (lane == 31) aexb = (T)1;
        if (lane == 31) fwa[warp] = Af;   // product over the warp's spans
        if (lane == 0) bwa[warp] = Ab;
        __syncthreads();
        if (warp == 0) {   // level factors of the cross-warp scans (lane = warp index)
            T A = (lane < nwarps) ? fwa[lane] : (T)1;
            T B = (lane < nwarps) ? bwa[lane] : (T)1;
            int l2 = 0;
#pragma unroll
            for (int off = 1; off < 32; off <<= 1, ++l2) {
                const T Au = __shfl_up_sync(0xffffffffu, A, off);
                const T Bd = __shfl_down_sync(0xffffffffu, B, off);
                fxa[l2][lane] = (lane >= off) ? A : (T)0;
                bxa[l2][lane] = (lane + off < 32) ? B : (T)0;
                if (lane >= off) A = A * Au;
                if (lane + off < 32) B = B * Bd;
            }
        }
        __syncthreads();
    }
    const T sc = (T)a.scale;
    const T* srcb = static_cast<const T*>(a.src) + b * a.mstride;
    T* dstb = static_cast<T*>(a.dst) + b * a.mstride;
    int line = blockIdx.x;
    T nxt[R];
    if (line < a.nrows) load_span<T, R>(srcb + int64_t(a.row0 + line) * a.pitch, c0, nx, nxt);
    for (; line < a.nrows; line += gridDim.x) {
        T d[R];
#pragma unroll
        for (int k = 0; k < R; ++k) d[k] = sc * nxt[k];
        const int nline = line + gridDim.x;
        if (nline < a.nrows) load_span<T, R>(srcb + int64_t(a.row0 + nline) * a.pitch, c0, nx, nxt);
        // forward y_c = d_c − l_c y_{c−1}: local (zero carry-in)
        T v = (T)0;
#pragma unroll
        for (int k = 0; k < R; ++k) {
            v = fmaT(tl[k], v, d[k]);
            d[k] = v;
        }
        {
            int lv = 0;
#pragma unroll
            for (int off = 1; off < 32; off <<= 1, ++lv) v = fmaT(lvf[lv * nt + t], __shfl_up_sync(0xffffffffu, v, off), v);
        }
        T vex = __shfl_up_sync(0xffffffffu, v, 1);
        if (lane == 0) vex = (T)0;
        if (lane == 31) fwv[warp] = v;
        __syncthreads();
        if (warp == 0) {   // exclusive scan of the warp totals
            T V = (lane < nwarps) ? fwv[lane] : (T)0;
            int l2 = 0;
#pragma unroll
            for (int off = 1; off < 32; off <<= 1, ++l2) V = fmaT(fxa[l2][lane], __shfl_up_sync(0xffffffffu, V, off), V);
            const T Vx = __shfl_up_sync(0xffffffffu, V, 1);
            if (lane < nwarps) fwc[lane] = (lane == 0) ? (T)0 : Vx;
        } else if (warp == 1 || nwarps == 1) {
            // (backward carries are computed after the fix-up)
        }
        __syncthreads();
        T cin = fmaT(aexf, fwc[warp], vex);
        {
            T pi = (T)1;
#pragma unroll
            for (int k = 0; k < R; ++k) {
                pi = pi * tl[k];
                d[k] = fmaT(pi, cin, d[k]);
            }
        }
        // backward x_c = y_c/u_c − e_c x_{c+1}
        v = (T)0;
#pragma unroll
        for (int k = R - 1; k >= 0; --k) {
            v = fmaT(te[k], v, d[k] * tiu[k]);
            d[k] = v;
        }
        {
            int lv = 0;
#pragma unroll
            for (int off = 1; off < 32; off <<= 1, ++lv) v = fmaT(lvb[lv * nt + t], __shfl_down_sync(0xffffffffu, v, off), v);
        }
        vex = __shfl_down_sync(0xffffffffu, v, 1);
        if (lane == 31) vex = (T)0;
        if (lane == 0) bwv[warp] = v;
        __syncthreads();
        if (warp == 0) {
            T V = (lane < nwarps) ? bwv[lane] : (T)0;
            int l2 = 0;
#pragma unroll
            for (int off = 1; off < 32; off <<= 1, ++l2) V = fmaT(bxa[l2][lane], __shfl_down_sync(0xffffffffu, V, off), V);
            const T Vx = __shfl_down_sync(0xffffffffu, V, 1);
            if (lane < nwarps) bwc[lane] = (lane == nwarps - 1) ? (T)0 : Vx;
        }
        __syncthreads();
        cin = fmaT(aexb, bwc[warp], vex);
        {
            T pi = (T)1;
#pragma unroll
            for (int k = R - 1; k >= 0; --k) {
                pi = pi * te[k];
                d[k] = fmaT(pi, cin, d[k]);
            }
        }
        store_span<T, R>(dstb + int64_t(a.row0 + line) * a.pitch, c0, 1, nx - 1, d);
    }
}

// Two rows per iteration (rows line and line + gridDim.x): the dependent scan chains of the two
// rows interleave and the four barriers per iteration serve both.  The LU tables live in shared
// memory as [k][thread] (conflict-free) so both rows' data and prefetch fit the 64 registers.
template <typename T, int R>
__global__ void __launch_bounds__(1024, 1) k_imp_x2(const ImpXArgs a) {
    __shared__ T fwv[2][IMPX_MAXW], bwv[2][IMPX_MAXW], fwc[2][IMPX_MAXW], bwc[2][IMPX_MAXW];
    __shared__ T fwa[IMPX_MAXW], bwa[IMPX_MAXW];
    __shared__ T fxa[5][IMPX_MAXW], bxa[5][IMPX_MAXW];
    extern __shared__ __align__(16) unsigned char smem_raw[];
    const int t = threadIdx.x, nt = blockDim.x;
    T* lvf = reinterpret_cast<T*>(smem_raw);   // [5][nt]
    T* lvb = lvf + 5 * nt;                      // [5][nt]
    T* stl = lvb + 5 * nt;                      // [R][nt]  −l
    T* siu = stl + R * nt;                      // [R][nt]  1/u
    T* ste = siu + R * nt;                      // [R][nt]  −e
    const int b = blockIdx.y;
    const int nx = a.nx, m = nx - 2;
    const int nwarps = nt >> 5;
    const int c0 = t * R;
    const int lane = t & 31, warp = t >> 5;
    T aexf, aexb;
    {
        const T* tab = static_cast<const T*>(a.tab) + b * 3 * a.tpitch;
        T Af = (T)1, Ab = (T)1;
#pragma unroll
        for (int k = 0; k < R; ++k) {
            const int c = c0 + k;
            const bool ok = c >= 1 && c <= m;
            const T l = ok ? -tab[c - 1] : (T)0;
            const T e = ok ? -tab[2 * a.tpitch + c - 1] : (T)0;
            stl[k * nt + t] = l;
            siu[k * nt + t] = ok ? tab[a.tpitch + c - 1] : (T)0;
            ste[k * nt + t] = e;
            Af = Af * l;
            Ab = Ab * e;
        }
        int lv = 0;
#pragma unroll
        for (int off = 1; off < 32; off <<= 1, ++lv) {
            const T Au = __shfl_up_sync(0xffffffffu, Af, off);
            const T Ad = __shfl_down_sync(0xffffffffu, Ab, off);
            lvf[lv * nt + t] = (lane >= off) ? Af : (T)0;
            lvb[lv * nt + t] = (lane + off < 32) ? Ab : (T)0;
            if (lane >= off) Af = Af * Au;
            if (lane + off < 32) Ab = Ab * Ad;
        }
        aexf = __shfl_up_sync(0xffffffffu, Af, 1);
        aexb = __shfl_down_sync(0xffffffffu, Ab, 1);
        if (lane == 0) aexf = (T)1;
        if (lane == 31) aexb = (T)1;
        if (lane == 31) fwa[warp] = Af;
        if (lane == 0) bwa[warp] = Ab;
        __syncthreads();
        if (warp == 0) {
            T A = (lane < nwarps) ? fwa[lane] : (T)1;
            T B = (lane < nwarps) ? bwa[lane] : (T)1;
            int l2 = 0;
#pragma unroll
            for (int off = 1; off < 32; off <<= 1, ++l2) {
                const T Au = __shfl_up_sync(0xffffffffu, A, off);
                const T Bd = __shfl_down_sync(0xffffffffu, B, off);
                fxa[l2][lane] = (lane >= off) ? A : (T)0;
                bxa[l2][lane] = (lane + off < 32) ? B : (T)0;
                if (lane >= off) A = A * Au;
                if (lane + off < 32) B = B * Bd;
            }
        }
        __syncthreads();
    }
    const T sc = (T)a.scale;
    const T* srcb = static_cast<const T*>(a.src) + b * a.mstride;
    T* dstb = static_cast<T*>(a.dst) + b * a.mstride;
    const int G = gridDim.x;
    int line = blockIdx.x;
    T nA[R], nB[R];
    auto fetch = [&](int l0, T (&x)[R], T (&y)[R]) {
        if (l0 < a.nrows) load_span<T, R>(srcb + int64_t(a.row0 + l0) * a.pitch, c0, nx, x);
        if (l0 + G < a.nrows) load_span<T, R>(srcb + int64_t(a.row0 + l0 + G) * a.pitch, c0, nx, y);
        else {
#pragma unroll
            for (int k = 0; k < R; ++k) y[k] = (T)0;
        }
    };
    fetch(line, nA, nB);
    for (; line < a.nrows; line += 2 * G) {
        const bool hasB = line + G < a.nrows;
        T dA[R], dB[R];
#pragma unroll
        for (int k = 0; k < R; ++k) {
            dA[k] = sc * nA[k];
            dB[k] = sc * nB[k];
        }
        fetch(line + 2 * G, nA, nB);
        // forward y_c = d_c − l_c y_{c−1}
        T vA = (T)0, vB = (T)0;
#pragma unroll
        for (int k = 0; k < R; ++k) {
            const T l = stl[k * nt + t];
            vA = fmaT(l, vA, dA[k]);
            vB = fmaT(l, vB, dB[k]);
            dA[k] = vA;
            dB[k] = vB;
        }
        {
            int lv = 0;
#pragma unroll
            for (int off = 1; off < 32; off <<= 1, ++lv) {
                const T f = lvf[lv * nt + t];
                const T uA = __shfl_up_sync(0xffffffffu, vA, off), uB = __shfl_up_sync(0xffffffffu, vB, off);
                vA = fmaT(f, uA, vA);
                vB = fmaT(f, uB, vB);
            }
        }
        T xA = __shfl_up_sync(0xffffffffu, vA, 1), xB = __shfl_up_sync(0xffffffffu, vB, 1);
        if (lane == 0) {
            xA = (T)0;
            xB = (T)0;
        }
        if (lane == 31) {
            fwv[0][warp] = vA;
            fwv[1][warp] = vB;
        }
        __syncthreads();
        if (warp < 2) {   // warp 0: row A, warp 1: row B
            T V = (lane < nwarps) ? fwv[warp][lane] : (T)0;
            int l2 = 0;
#pragma unroll
            for (int off = 1; off < 32; off <<= 1, ++l2) V = fmaT(fxa[l2][lane], __shfl_up_sync(0xffffffffu, V, off), V);
            const T Vx = __shfl_up_sync(0xffffffffu, V, 1);
            if (lane < nwarps) fwc[warp][lane] = (lane == 0) ? (T)0 : Vx;
        }
        __syncthreads();
        {
            const T cA = fmaT(aexf, fwc[0][warp], xA), cB = fmaT(aexf, fwc[1][warp], xB);
            T pi = (T)1;
#pragma unroll
            for (int k = 0; k < R; ++k) {
                pi = pi * stl[k * nt + t];
                dA[k] = fmaT(pi, cA, dA[k]);
                dB[k] = fmaT(pi, cB, dB[k]);
            }
        }
        // backward x_c = y_c/u_c − e_c x_{c+1}
        vA = (T)0;
        vB = (T)0;
#pragma unroll
        for (int k = R - 1; k >= 0; --k) {
            const T e = ste[k * nt + t], iu = siu[k * nt + t];
            vA = fmaT(e, vA, dA[k] * iu);
            vB = fmaT(e, vB, dB[k] * iu);
            dA[k] = vA;
            dB[k] = vB;
        }
        {
            int lv = 0;
#pragma unroll
            for (int off = 1; off < 32; off <<= 1, ++lv) {
                const T f = lvb[lv * nt + t];
                const T uA = __shfl_down_sync(0xffffffffu, vA, off), uB = __shfl_down_sync(0xffffffffu, vB, off);
                vA = fmaT(f, uA, vA);
                vB = fmaT(f, uB, vB);
            }
        }
        xA = __shfl_down_sync(0xffffffffu, vA, 1);
        xB = __shfl_down_sync(0xffffffffu, vB, 1);
        if (lane == 31) {
            xA = (T)0;
            xB = (T)0;
        }
        if (lane == 0) {
            bwv[0][warp] = vA;
            bwv[1][warp] = vB;
        }
        __syncthreads();
        if (warp < 2) {
            T V = (lane < nwarps) ? bwv[warp][lane] : (T)0;
            int l2 = 0;
#pragma unroll
            for (int off = 1; off < 32; off <<= 1, ++l2) V = fmaT(bxa[l2][lane], __shfl_down_sync(0xffffffffu, V, off), V);
            const T Vx = __shfl_down_sync(0xffffffffu, V, 1);
            if (lane < nwarps) bwc[warp][lane] = (lane == nwarps - 1) ? (T)0 : Vx;
        }
        __syncthreads();
        {
            const T cA = fmaT(aexb, bwc[0][warp], xA), cB = fmaT(aexb, bwc[1][warp], xB);
            T pi = (T)1;
#pragma unroll
            for (int k = R - 1; k >= 0; --k) {
                pi = pi * ste[k * nt + t];
                dA[k] = fmaT(pi, cA, dA[k]);
                dB[k] = fmaT(pi, cB, dB[k]);
            }
        }
        store_span<T, R>(dstb + int64_t(a.row0 + line) * a.pitch, c0, 1, nx - 1, dA);
        if (hasB) store_span<T, R>(dstb + int64_t(a.row0 + line + G) * a.pitch, c0, 1, nx - 1, dB);
    }
}

struct ImpYArgs {
    const void* z;     // x-solve output (field layout, view rows)
    void* prev;        // u^{n−1} (MODE 0) or u₁ (MODE 1); overwritten by u^{n+1}
    const void* cf;    // c2 [B][cpitch], one value per column
    int64_t pitch, mstride, cpitch;
    int32_t nx;
    int32_t m;         // unknowns per column (ny − 2): global rows 1..m
    int32_t seg;       // rows per segment (multiple of 8); 32 segments cover 1..m
    double dt;
};

constexpr int IMPY_COLS = 16;
constexpr int IMPY_SEGS = 32;
constexpr int IMPY_THREADS = IMPY_COLS * IMPY_SEGS;

// One CTA owns 16 interior columns × the full height, as 32 segments of `seg` rows (lanes 0–15 /
// 16–31 of warp w: segments 2w / 2w+1).  Pass 1 reads z and forms per-segment and per-8-row
// decayed sums; the cross-segment carries go through shared memory; pass 2 re-reads z (L2),
// forms L_j, R_j and the boundary corrections and writes u^{n+1} over `prev`.
template <typename T, int MODE>
__global__ void __launch_bounds__(IMPY_THREADS, 2) k_imp_y(const ImpYArgs a) {
    extern __shared__ __align__(16) unsigned char smem_raw[];
    T* Fs = reinterpret_cast<T*>(smem_raw);      // [32][16] forward sums (decayed to last valid row)
    T* Bs = Fs + IMPY_SEGS * IMPY_COLS;          // [32][16] backward sums (decayed to segment start)
    T* subS = Bs + IMPY_SEGS * IMPY_COLS;        // [NS][512] per-8-row backward sums → suffix carries
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    const int cl = lane & 15, sg = 2 * warp + (lane >> 4);
    const int b = blockIdx.y;
    const int64_t col = 1 + int64_t(blockIdx.x) * IMPY_COLS + cl;
    const bool colok = col <= a.nx - 2;
    const int m = a.m, seg = a.seg, NS = seg >> 3;
    const int j0 = 1 + sg * seg;
    // column constants (fp64, rounded once to T)
    const double g = colok ? (double)static_cast<const T*>(a.cf)[b * a.cpitch + col] : 0.0;
    const double sq = sqrt(1.0 + 2.0 * g);
    const double rho_d = g / ((1.0 + g) + sq);
    const double kap_d = 0.5 * ((1.0 + g) + sq);
    const double omr = (1.0 + sq) / ((1.0 + g) + sq);  // 1 − ρ, without cancellation
    const double i1_d = 1.0 / (omr * (1.0 + rho_d));    // 1/(1 − ρ²)
    const T rho = (T)rho_d;
    const T* zb = static_cast<const T*>(a.z) + b * a.mstride + col;
    T* pb = static_cast<T*>(a.prev) + b * a.mstride + col;
    // ---- pass 1 ----
    T F = (T)0;
    for (int t = 0; t < NS; ++t) {
        T Bt = (T)0, pw = (T)1;
        const int jt = j0 + 8 * t;
        T zz[8];
#pragma unroll
        for (int k = 0; k < 8; ++k) zz[k] = (colok && jt + k <= m) ? zb[int64_t(1 + jt + k) * a.pitch] : (T)0;
#pragma unroll
        for (int k = 0; k < 8; ++k) {
            if (jt + k <= m) F = fmaT(rho, F, zz[k]);
            Bt = fmaT(pw, zz[k], Bt);
            pw = pw * rho;
        }
        subS[t * IMPY_THREADS + threadIdx.x] = Bt;
    }
    const T rho8 = powi_T(rho, 8);
    {
        T Bsum = (T)0;
        for (int t = NS - 1; t >= 0; --t) Bsum = fmaT(rho8, Bsum, subS[t * IMPY_THREADS + threadIdx.x]);
        Fs[sg * IMPY_COLS + cl] = F;
        Bs[sg * IMPY_COLS + cl] = Bsum;
    }
    __syncthreads();
    const T rhoS = powi_T(rho, seg);
    T Lin = (T)0;
    for (int k = 0; k < sg; ++k) Lin = fmaT(rhoS, Lin, Fs[k * IMPY_COLS + cl]);
    T Sbelow = (T)0;
    for (int k = IMPY_SEGS - 1; k > sg; --k) Sbelow = fmaT(rhoS, Sbelow, Bs[k * IMPY_COLS + cl]);
    T A1 = Sbelow;
    for (int k = sg; k >= 0; --k) A1 = fmaT(rhoS, A1, Bs[k * IMPY_COLS + cl]);
    // L_m: segments before the last non-empty one are full
    const int klast = (m - 1) / seg;
    T Lm = (T)0;
    for (int k = 0; k < klast; ++k) Lm = fmaT(rhoS, Lm, Fs[k * IMPY_COLS + cl]);
    Lm = fmaT(powi_T(rho, m - klast * seg), Lm, Fs[klast * IMPY_COLS + cl]);
    const T A2 = rho * Lm;
    const T rhom = powi_T(rho, m);
    const T i1 = (T)i1_d;
    const T z1 = (A1 - rhom * A2) * i1;
    const T rr = rho * rho;
    const T beta = rr / ((T)1 + rr * (((T)1 - rhom * rhom) * i1));
    const T bz1 = beta * z1;
    const T A2p = A2 - bz1 * rhom;
    const T K = (T)(i1_d / kap_d);
    // suffix carries per 8-row block: subS[t] ← Σ_{i > end of block t} ρ^{i − end − 1} z_i
    {
        T Sa = Sbelow;
        for (int t = NS - 1; t >= 0; --t) {
            const T tmp = subS[t * IMPY_THREADS + threadIdx.x];
            subS[t * IMPY_THREADS + threadIdx.x] = Sa;
            Sa = fmaT(rho8, Sa, tmp);
        }
    }
    if (!colok || j0 > m) return;
    // ---- pass 2 ----
    const T dtT = (T)a.dt;
    T L = Lin;
    T pu = powi_T(rho, j0 - 1);
    for (int t = 0; t < NS; ++t) {
        const int jt = j0 + 8 * t;
        if (jt > m) break;
        T zz[8], Lc[8];
#pragma unroll
        for (int k = 0; k < 8; ++k) zz[k] = (jt + k <= m) ? zb[int64_t(1 + jt + k) * a.pitch] : (T)0;
#pragma unroll
        for (int k = 0; k < 8; ++k) {
            L = fmaT(rho, L, zz[k]);
            Lc[k] = L - bz1 * pu;
            pu = pu * rho;
        }
        T R = rho * subS[t * IMPY_THREADS + threadIdx.x];
        const int e = jt + 7;
        T pd = powi_T(rho, (m + 1 - e) > 1 ? (m + 1 - e) : 1);
#pragma unroll
        for (int k = 7; k >= 0; --k) {
            const int j = jt + k;
            if (j <= m) {
                const T x = K * ((Lc[k] + R) - pd * A2p);
                T* q = pb + int64_t(1 + j) * a.pitch;
                const T pv = *q;
                *q = (MODE == 0) ? (x - pv) : fmaT(dtT, pv, x);
                pd = pd * rho;
            }
            R = rho * (zz[k] + R);
        }
    }
}

// Resident variant of the y solve (thread-block cluster).  A cluster of CL ≤ 8 CTAs owns COLS =
// 128 B / sizeof(T) interior columns (one 128-byte line per row) × the full height; CTA r of the
// cluster owns rows [1 + r·SEGS·seg, 1 + (r+1)·SEGS·seg) as SEGS = 512 / COLS segments of ≤ SR
// rows (lane = column + COLS × local segment).  Each thread stages its segment of z in shared
// memory with cp.async and holds its rows of u^{n−1} in registers, so everything it reads from HBM
// is in flight at once.  Segment sums → carries: warp shuffles across segments, warp totals
// through shared memory, CTA totals across the cluster through distributed shared memory →
// a forward walk (L_j, folded into the registers) and a backward walk (R_j) over the staged
// segment → u^{n+1} over `prev`.  Forward factors are ρ^{valid rows} (empty / partial segments
// compose exactly); backward factors ρ^{slots}.  HBM traffic: z, u^{n−1} once each, u^{n+1} once.
constexpr int IMPYC_THREADS = 512;

template <typename T>
struct ImpYc {
    static constexpr int COLS = 128 / int(sizeof(T));
    static constexpr int SEGS = IMPYC_THREADS / COLS;  // segments per CTA
    static constexpr int WARPS = IMPYC_THREADS / 32;
    static constexpr int SPW = 32 / COLS;              // segments per warp
    static constexpr int SR = 128 / int(sizeof(T));    // max rows per segment (registers)
    static __host__ __device__ size_t smem_bytes(int seg) {
        return (size_t(SEGS) * seg * COLS + 4 * size_t(WARPS) * COLS + 12 * COLS) * sizeof(T);
    }
};

template <typename T>
__device__ __forceinline__ void cp_async_elem(T* sdst, const T* gsrc, bool valid) {
    const uint32_t sa = static_cast<uint32_t>(__cvta_generic_to_shared(sdst));
    const int n = valid ? int(sizeof(T)) : 0;   // src-size 0 ⇒ zero fill
    if constexpr (sizeof(T) == 8)
        asm volatile("cp.async.ca.shared.global [%0], [%1], 8, %2;\n" ::"r"(sa), "l"(gsrc), "r"(n) : "memory");
    else
        asm volatile("cp.async.ca.shared.global [%0], [%1], 4, %2;\n" ::"r"(sa), "l"(gsrc), "r"(n) : "memory");
}

// Half-warp (16-lane) inclusive affine scans: forward (lane k combines lanes ≤ k), backward.
template <typename T>
__device__ __forceinline__ void half_affine_fwd(T& A, T& V, int k) {
#pragma unroll
    for (int off = 1; off < 16; off <<= 1) {
        const T Vu = __shfl_up_sync(0xffffffffu, V, off, 16);
        const T Au = __shfl_up_sync(0xffffffffu, A, off, 16);
        if (k >= off) {
            V = fmaT(A, Vu, V);
            A = A * Au;
        }
    }
}
template <typename T>
__device__ __forceinline__ void half_affine_bwd(T& A, T& V, int k) {
#pragma unroll
    for (int off = 1; off < 16; off <<= 1) {
        const T Vd = __shfl_down_sync(0xffffffffu, V, off, 16);
        const T Ad = __shfl_down_sync(0xffffffffu, A, off, 16);
        if (k + off < 16) {
            V = fmaT(A, Vd, V);
            A = A * Ad;
        }
    }
}

template <typename T, int MODE>
__global__ void __launch_bounds__(IMPYC_THREADS, 2) k_imp_yc(const ImpYArgs a) {
    using G = ImpYc<T>;
    constexpr int COLS = G::COLS, SR = G::SR, SEGS = G::SEGS, WARPS = G::WARPS;
    static_assert(WARPS == 16, "one half-warp lane per warp of the CTA");
    namespace cg = cooperative_groups;
    cg::cluster_group cluster = cg::this_cluster();
    const int CL = int(cluster.num_blocks());
    const int rk = int(cluster.block_rank());
    extern __shared__ __align__(16) unsigned char smem_raw[];
    const int seg = a.seg;
    T* zs = reinterpret_cast<T*>(smem_raw);                 // [SEGS][seg][COLS]
    T* wF = zs + size_t(SEGS) * seg * COLS;                 // [WARPS][COLS] warp totals: forward value
    T* wFA = wF + WARPS * COLS;                             //   forward factor (→ carry factor into the warp)
    T* wB = wFA + WARPS * COLS;                             //   backward value
    T* wBA = wB + WARPS * COLS;                             //   backward factor
    T* ctot = wBA + WARPS * COLS;                           // [4][COLS] this CTA's totals (read by the cluster)
    T* ccon = ctot + 4 * COLS;                              // [8][COLS] column constants
    const int t = threadIdx.x, lane = t & 31, warp = t >> 5;
    const int cl = lane % COLS, sl = lane / COLS;
    const int sg = warp * G::SPW + sl;
    const int b = blockIdx.z;
    const int64_t colbase = 1 + int64_t(blockIdx.x) * COLS;
    const int64_t col = colbase + cl;
    const bool colok = col <= a.nx - 2;
    const int m = a.m;
    const int j0 = 1 + (rk * SEGS + sg) * seg;
    int nvalid = m - j0 + 1;
    nvalid = nvalid < 0 ? 0 : (nvalid > seg ? seg : nvalid);
    const int nv_ld = colok ? nvalid : 0;
    T* zrow = zs + size_t(sg) * seg * COLS + cl;
    // ---- stage this thread's segment of z (u^{n−1} is read just before pass 2) ----
    {
        const T* zq = static_cast<const T*>(a.z) + b * a.mstride + col + int64_t(1 + j0) * a.pitch;
#pragma unroll
        for (int k = 0; k < SR; ++k) {
            if (k < seg) cp_async_elem(zrow + k * COLS, zq, k < nv_ld);
            zq += a.pitch;
        }
    }
    // ---- column constants (once per column) ----
    if (t < COLS) {
        const int64_t cf = colbase + t;
        const double g = (cf <= a.nx - 2) ? (double)static_cast<const T*>(a.cf)[b * a.cpitch + cf] : 0.0;
        const double sq = sqrt(1.0 + 2.0 * g);
        const double rho_d = g / ((1.0 + g) + sq);
        const double kap_d = 0.5 * ((1.0 + g) + sq);
        const double omr = (1.0 + sq) / ((1.0 + g) + sq);  // 1 − ρ without cancellation
        const double i1_d = 1.0 / (omr * (1.0 + rho_d));    // 1/(1 − ρ²)
        ccon[t] = (T)rho_d;
        ccon[1 * COLS + t] = (T)(i1_d / kap_d);   // K
        ccon[2 * COLS + t] = (T)i1_d;
    }
    __syncthreads();
    const T rho = ccon[cl];
    asm volatile("cp.async.wait_all;\n" ::: "memory");
    // ---- segment sums: F (forward, to the last valid row), B (backward, from the segment start);
    //      both carry factors are ρ^{nvalid} (everything after a partial segment is zero) ----
    T F = (T)0, Bsum = (T)0, pw = (T)1;
    if (nvalid == SR) {
#pragma unroll
        for (int k = 0; k < SR; ++k) {
            const T z = zrow[k * COLS];
            F = fmaT(rho, F, z);
            Bsum = fmaT(pw, z, Bsum);
            pw = pw * rho;
        }
    } else {
        for (int k = 0; k < nvalid; ++k) {
            const T z = zrow[k * COLS];
            F = fmaT(rho, F, z);
            Bsum = fmaT(pw, z, Bsum);
            pw = pw * rho;
        }
    }
    T Af = pw, Vf = F, Ab = pw, Vb = Bsum;
    T vfx = (T)0, afx = (T)1, vbx = (T)0, abx = (T)1;
    if constexpr (G::SPW > 1) {
        warp_affine_fwd(Af, Vf, lane, COLS);
        warp_affine_bwd(Ab, Vb, lane, COLS);
        vfx = __shfl_up_sync(0xffffffffu, Vf, COLS);
        afx = __shfl_up_sync(0xffffffffu, Af, COLS);
        vbx = __shfl_down_sync(0xffffffffu, Vb, COLS);
        abx = __shfl_down_sync(0xffffffffu, Ab, COLS);
        if (sl == 0) {
            vfx = (T)0;
            afx = (T)1;
        }
        if (sl == G::SPW - 1) {
            vbx = (T)0;
            abx = (T)1;
        }
    }
    if (sl == G::SPW - 1) {
        wF[warp * COLS + cl] = Vf;
        wFA[warp * COLS + cl] = Af;
    }
    if (sl == 0) {
        wB[warp * COLS + cl] = Vb;
        wBA[warp * COLS + cl] = Ab;
    }
    __syncthreads();
    // ---- scans over the 16 warps.  Jobs (column, direction) per half-warp; a backward scan runs
    //      as a forward scan over reversed elements, so both halves issue identical shuffles ----
    constexpr int NQ = (COLS == 16) ? 1 : 2;   // rounds
    const int h = lane >> 4, k = lane & 15;
    T exA[NQ], exV[NQ];
#pragma unroll
    for (int q = 0; q < NQ; ++q) {
        const int jc = (COLS == 16) ? warp : 2 * warp + h;   // column of this job
        const int dir = (COLS == 16) ? h : q;
        const int e = dir == 0 ? k : 15 - k;                  // warp index of this lane's element
        T A = dir == 0 ? wFA[e * COLS + jc] : wBA[e * COLS + jc];
        T V = dir == 0 ? wF[e * COLS + jc] : wB[e * COLS + jc];
        half_affine_fwd(A, V, k);
        T Ax = __shfl_up_sync(0xffffffffu, A, 1, 16), Vx = __shfl_up_sync(0xffffffffu, V, 1, 16);
        if (k == 0) {
            Ax = (T)1;
            Vx = (T)0;
        }
        exA[q] = Ax;
        exV[q] = Vx;
        if (k == 15) {
            ctot[(2 * dir) * COLS + jc] = V;
            ctot[(2 * dir + 1) * COLS + jc] = A;
        }
    }
    cluster.sync();
    // ---- scans over the cluster's CTAs (distributed shared memory, one rank per lane) ----
#pragma unroll
    for (int q = 0; q < NQ; ++q) {
        const int jc = (COLS == 16) ? warp : 2 * warp + h;
        const int dir = (COLS == 16) ? h : q;
        const int e = dir == 0 ? k : 15 - k;
        T A = (T)1, V = (T)0;
        if (k < CL) {
            const int r = dir == 0 ? k : CL - 1 - k;
            const T* ot = cluster.map_shared_rank(ctot, r);
            V = ot[(2 * dir) * COLS + jc];
            A = ot[(2 * dir + 1) * COLS + jc];
        }
        half_affine_fwd(A, V, k);
        const int kr = dir == 0 ? rk : CL - 1 - rk;           // lane of this CTA's rank
        const int src = (h << 4) + (kr > 0 ? kr - 1 : 0);
        T A2x = __shfl_sync(0xffffffffu, A, src), V2x = __shfl_sync(0xffffffffu, V, src);
        if (kr == 0) {
            A2x = (T)1;
            V2x = (T)0;
        }
        const T Atot = __shfl_sync(0xffffffffu, A, (h << 4) + 15);
        const T Vtot = __shfl_sync(0xffffffffu, V, (h << 4) + 15);
        // carry into warp e (value and factor: everything before / after it in the column)
        if (dir == 0) {
            wF[e * COLS + jc] = fmaT(exA[q], V2x, exV[q]);
            wFA[e * COLS + jc] = exA[q] * A2x;
            if (k == 0) {
                ccon[3 * COLS + jc] = Vtot;   // L_m
                ccon[4 * COLS + jc] = Atot;   // ρ^m
            }
        } else {
            wB[e * COLS + jc] = fmaT(exA[q], V2x, exV[q]);
            wBA[e * COLS + jc] = exA[q] * A2x;
            if (k == 0) ccon[5 * COLS + jc] = Vtot;   // A1 = Σ ρ^{i−1} z_i
        }
    }
    asm volatile("barrier.cluster.arrive.release.aligned;\n" ::: "memory");   // totals no longer read remotely
    __syncthreads();
    if (t < COLS) {   // column-global constants of the closed form
        const T rh = ccon[t], i1 = ccon[2 * COLS + t];
        const T Lm = ccon[3 * COLS + t], rhom = ccon[4 * COLS + t], A1 = ccon[5 * COLS + t];
        const T A2 = rh * Lm;
        const T z1 = (A1 - rhom * A2) * i1;
        const T rr = rh * rh;
        const T beta = rr / ((T)1 + rr * (((T)1 - rhom * rhom) * i1));
        const T bz1 = beta * z1;
        ccon[6 * COLS + t] = bz1;
        ccon[7 * COLS + t] = A2 - bz1 * rhom;   // A2'
    }
    __syncthreads();
    if (nv_ld > 0) {
        // pass 2 in 8-row blocks, bottom block first: a forward pre-walk records L and ρ^{j−1} at
        // each block start; each block then reads its u^{n−1}, walks forward (L_j) and backward (R_j)
        constexpr int NBLK = SR / 8;
        const T K = ccon[COLS + cl], bz1 = ccon[6 * COLS + cl], A2p = ccon[7 * COLS + cl];
        const T dtT = (T)a.dt;
        T Lb[NBLK], pub[NBLK];
        {
            T L = fmaT(afx, wF[warp * COLS + cl], vfx);   // L_{j0−1}
            T pu = afx * wFA[warp * COLS + cl];           // ρ^{j0−1}
#pragma unroll
            for (int q = 0; q < NBLK; ++q) {
                Lb[q] = L;
                pub[q] = pu;
#pragma unroll
                for (int kk = 0; kk < 8; ++kk) {
                    if (8 * q + kk < nvalid) {
                        L = fmaT(rho, L, zrow[(8 * q + kk) * COLS]);
                        pu = pu * rho;
                    }
                }
            }
        }
        T R = rho * fmaT(abx, wB[warp * COLS + cl], vbx);   // R at the last valid row
        T pd = rho * (abx * wBA[warp * COLS + cl]);         // ρ^{m+1−e}, e = last valid row
        const T* pbase = static_cast<const T*>(a.prev) + b * a.mstride + col + int64_t(1 + j0) * a.pitch;
#pragma unroll
        for (int q = NBLK - 1; q >= 0; --q) {
            if (8 * q < nvalid) {
                T w[8];
                const T* pq = pbase + int64_t(8 * q) * a.pitch;
#pragma unroll
                for (int kk = 0; kk < 8; ++kk) w[kk] = (8 * q + kk < nvalid) ? pq[int64_t(kk) * a.pitch] : (T)0;
                T L = Lb[q], pu = pub[q];
#pragma unroll
                for (int kk = 0; kk < 8; ++kk) {   // w_j ← K·(L_j − βz₁ρ^{j−1}) ∓ prev_j
                    if (8 * q + kk < nvalid) {
                        L = fmaT(rho, L, zrow[(8 * q + kk) * COLS]);
                        const T lc = K * fmaT(-bz1, pu, L);
                        w[kk] = (MODE == 0) ? (lc - w[kk]) : fmaT(dtT, w[kk], lc);
                        pu = pu * rho;
                    }
                }
                T* po = const_cast<T*>(pq);
#pragma unroll
                for (int kk = 7; kk >= 0; --kk) {   // u^{n+1}_j = w_j + K·(R_j − ρ^{m+1−j} A₂')
                    if (8 * q + kk < nvalid) {
                        po[int64_t(kk) * a.pitch] = fmaT(K, fmaT(-pd, A2p, R), w[kk]);
                        pd = pd * rho;
                        R = rho * (zrow[(8 * q + kk) * COLS] + R);
                    }
                }
            }
        }
    }
    asm volatile("barrier.cluster.wait.acquire.aligned;\n" ::: "memory");
}

// ------------------------------------------------------------------------------------------
// Implicit y solve, streaming variant (TSW_OPT_IMPLICIT_SOLVER = 2): the same closed form as
// k_imp_yc in three barrier-free kernels — per-(column, segment) decayed sums; a per-column scan
// of the segments (carries and the column constants of the closed form); the finish (L_j, R_j,
// the boundary terms and the three-level update).  z is read twice (4 words + the small carry
// arrays per node and level) but every kernel is a plain coalesced stream.
// ------------------------------------------------------------------------------------------
constexpr int IMPS_SEG = 16;   // rows per segment

struct ImpSArgs {
    const void* z;      // x-solve output (field layout)
    void* prev;         // u^{n−1} / u₁ → u^{n+1}
    const void* ycol;   // [B][4][ncolp]: ρ, K = 1/(κ(1−ρ²)), i1 = 1/(1−ρ²), spare   (columns 1..nx−2 at 0..)
    void* cF;           // [B][nseg][ncolp]: forward sums → L_in
    void* cB;           // [B][nseg][ncolp]: backward sums → S_below
    void* ccon;         // [B][2][ncolp]: βz₁, A₂'
    int64_t pitch, mstride, ncolp;
    int32_t nx, m, nseg;
    double dt;
};

// column constants from c2 (once per coefficients / dt)
template <typename T>
__global__ void k_imp_ycol(const T* __restrict__ c2, int64_t cpitch, T* __restrict__ ycol, int64_t ncolp, int nx, int B) {
    const int64_t i = blockIdx.x * int64_t(blockDim.x) + threadIdx.x;
    const int b = blockIdx.y;
    if (i >= nx - 2 || b >= B) return;
    const double g = (double)c2[b * cpitch + 1 + i];
    const double sq = sqrt(1.0 + 2.0 * g);
    const double rho = g / ((1.0 + g) + sq);
    const double kap = 0.5 * ((1.0 + g) + sq);
    const double omr = (1.0 + sq) / ((1.0 + g) + sq);
    const double i1 = 1.0 / (omr * (1.0 + rho));
    T* y = ycol + b * 4 * ncolp;
    y[i] = (T)rho;
    y[ncolp + i] = (T)(i1 / kap);
    y[2 * ncolp + i] = (T)i1;
}

// pass 1: thread (column, segment) — F (forward, to the last valid row), B (backward, from the start)
template <typename T>
__global__ void __launch_bounds__(256) k_imp_ysum(const ImpSArgs a) {
    const int64_t ci = blockIdx.x * 32 + threadIdx.x;   // column index 0.. (global column ci + 1)
    const int sg = blockIdx.y * 8 + threadIdx.y;
    const int b = blockIdx.z;
    if (ci >= a.nx - 2 || sg >= a.nseg) return;
    const T rho = static_cast<const T*>(a.ycol)[b * 4 * a.ncolp + ci];
    const int j0 = 1 + sg * IMPS_SEG;
    const int nv = min(IMPS_SEG, a.m - j0 + 1);
    const T* zq = static_cast<const T*>(a.z) + b * a.mstride + (ci + 1) + int64_t(1 + j0) * a.pitch;
    T zz[IMPS_SEG];
#pragma unroll
    for (int k = 0; k < IMPS_SEG; ++k) zz[k] = (k < nv) ? zq[int64_t(k) * a.pitch] : (T)0;
    T F = (T)0, Bs = (T)0, pw = (T)1;
#pragma unroll
    for (int k = 0; k < IMPS_SEG; ++k) {
        if (k < nv) {
            F = fmaT(rho, F, zz[k]);
            Bs = fmaT(pw, zz[k], Bs);
            pw = pw * rho;
        }
    }
    static_cast<T*>(a.cF)[(b * int64_t(a.nseg) + sg) * a.ncolp + ci] = F;
    static_cast<T*>(a.cB)[(b * int64_t(a.nseg) + sg) * a.ncolp + ci] = Bs;
}

// pass 2: scans over the segments of each column (in place: F → L_in, B → S_below) and the
// column-global constants βz₁, A₂'.  CTA = 32 columns × 32 groups; group g owns segments
// [g·G, (g+1)·G): local scans, carries across the groups through shared memory, re-walk.
constexpr int IMPS_GROUPS = 32;
template <typename T, int GMAX>
__global__ void __launch_bounds__(1024) k_imp_yscan(const ImpSArgs a) {
    __shared__ T sF[IMPS_GROUPS][33], sB[IMPS_GROUPS][33], sP[IMPS_GROUPS][33];
    __shared__ T sLm[32], sA1[32];
    const int tx = threadIdx.x, grp = threadIdx.y;
    const int64_t ci = blockIdx.x * 32 + tx;
    const int b = blockIdx.y;
    const bool ok = ci < a.nx - 2;
    const int G = (a.nseg + IMPS_GROUPS - 1) / IMPS_GROUPS;   // segments per group (≤ GMAX)
    const T* y = static_cast<const T*>(a.ycol) + b * 4 * a.ncolp;
    const T rho = ok ? y[ci] : (T)0;
    const T i1 = ok ? y[2 * a.ncolp + ci] : (T)1;
    T* F = static_cast<T*>(a.cF) + b * int64_t(a.nseg) * a.ncolp + ci;
    T* Bv = static_cast<T*>(a.cB) + b * int64_t(a.nseg) * a.ncolp + ci;
    const T rS = powi_T(rho, IMPS_SEG);
    const int nlast = a.m - (a.nseg - 1) * IMPS_SEG;
    const T rL = powi_T(rho, nlast);
    const int g0 = grp * G;
    T f[GMAX], bb[GMAX];
    T Lloc = (T)0, P = (T)1;
#pragma unroll
    for (int k = 0; k < GMAX; ++k) {
        const int sg = g0 + k;
        const bool v = ok && k < G && sg < a.nseg;
        f[k] = v ? F[int64_t(sg) * a.ncolp] : (T)0;
        bb[k] = v ? Bv[int64_t(sg) * a.ncolp] : (T)0;
        if (v) {
            const T fac = (sg == a.nseg - 1) ? rL : rS;
            Lloc = fmaT(fac, Lloc, f[k]);
            P = P * fac;
        }
    }
    T Sloc = (T)0;
#pragma unroll
    for (int k = GMAX - 1; k >= 0; --k) {
        const int sg = g0 + k;
        if (ok && k < G && sg < a.nseg) Sloc = fmaT((sg == a.nseg - 1) ? rL : rS, Sloc, bb[k]);
    }
    sF[grp][tx] = Lloc;
    sB[grp][tx] = Sloc;
    sP[grp][tx] = P;
    __syncthreads();
    T L = (T)0;
    for (int g = 0; g < grp; ++g) L = fmaT(sP[g][tx], L, sF[g][tx]);
    T S = (T)0;
    for (int g = IMPS_GROUPS - 1; g > grp; --g) S = fmaT(sP[g][tx], S, sB[g][tx]);
    if (grp == IMPS_GROUPS - 1) sLm[tx] = fmaT(P, L, Lloc);   // L_m: everything composed
    if (grp == 0) sA1[tx] = fmaT(P, S, Sloc);                  // A₁
    // re-walk with the true carries
#pragma unroll
    for (int k = 0; k < GMAX; ++k) {
        const int sg = g0 + k;
        if (ok && k < G && sg < a.nseg) {
            F[int64_t(sg) * a.ncolp] = L;
            L = fmaT((sg == a.nseg - 1) ? rL : rS, L, f[k]);
        }
    }
#pragma unroll
    for (int k = GMAX - 1; k >= 0; --k) {
        const int sg = g0 + k;
        if (ok && k < G && sg < a.nseg) {
            Bv[int64_t(sg) * a.ncolp] = S;
            S = fmaT((sg == a.nseg - 1) ? rL : rS, S, bb[k]);
        }
    }
    __syncthreads();
    if (grp == 0 && ok) {
        const T Lm = sLm[tx], A1 = sA1[tx];
        const T A2 = rho * Lm;
        const T rhom = powi_T(rho, a.m);
        const T z1 = (A1 - rhom * A2) * i1;
        const T rr = rho * rho;
        const T beta = rr / ((T)1 + rr * (((T)1 - rhom * rhom) * i1));
        const T bz1 = beta * z1;
        T* cc = static_cast<T*>(a.ccon) + b * 2 * a.ncolp;
        cc[ci] = bz1;
        cc[a.ncolp + ci] = A2 - bz1 * rhom;
    }
}

// pass 3: thread (column, segment) — u^{n+1}_j = K·(L_j + R_j − βz₁ρ^{j−1} − ρ^{m+1−j}A₂') ∓ prev_j
template <typename T, int MODE>
__global__ void __launch_bounds__(256) k_imp_yfin(const ImpSArgs a) {
    const int64_t ci = blockIdx.x * 32 + threadIdx.x;
    const int sg = blockIdx.y * 8 + threadIdx.y;
    const int b = blockIdx.z;
    if (ci >= a.nx - 2 || sg >= a.nseg) return;
    const int j0 = 1 + sg * IMPS_SEG;
    const int nv = min(IMPS_SEG, a.m - j0 + 1);
    const T* zq = static_cast<const T*>(a.z) + b * a.mstride + (ci + 1) + int64_t(1 + j0) * a.pitch;
    T* pq = static_cast<T*>(a.prev) + b * a.mstride + (ci + 1) + int64_t(1 + j0) * a.pitch;
    T zz[IMPS_SEG], w[IMPS_SEG];
#pragma unroll
    for (int k = 0; k < IMPS_SEG; ++k) {
        zz[k] = (k < nv) ? zq[int64_t(k) * a.pitch] : (T)0;
        w[k] = (k < nv) ? pq[int64_t(k) * a.pitch] : (T)0;
    }
    const T* y = static_cast<const T*>(a.ycol) + b * 4 * a.ncolp;
    const T rho = y[ci], K = y[a.ncolp + ci];
    const T* cc = static_cast<const T*>(a.ccon) + b * 2 * a.ncolp;
    const T bz1 = cc[ci], A2p = cc[a.ncolp + ci];
    T L = static_cast<const T*>(a.cF)[(b * int64_t(a.nseg) + sg) * a.ncolp + ci];
    T R = rho * static_cast<const T*>(a.cB)[(b * int64_t(a.nseg) + sg) * a.ncolp + ci];
    T pu = powi_T(rho, j0 - 1);
    T pd = powi_T(rho, a.m + 1 - (j0 + nv - 1));
    const T dtT = (T)a.dt;
#pragma unroll
    for (int k = 0; k < IMPS_SEG; ++k) {
        if (k < nv) {
            L = fmaT(rho, L, zz[k]);
            const T lc = K * fmaT(-bz1, pu, L);
            w[k] = (MODE == 0) ? (lc - w[k]) : fmaT(dtT, w[k], lc);
            pu = pu * rho;
        }
    }
#pragma unroll
    for (int k = IMPS_SEG - 1; k >= 0; --k) {
        if (k < nv) {
            pq[int64_t(k) * a.pitch] = fmaT(K, fmaT(-pd, A2p, R), w[k]);
            pd = pd * rho;
            R = rho * (zz[k] + R);
        }
    }
}

// ------------------------------------------------------------------------------------------
// Peer halos (peer mode): ghost rows are written by the producing rank straight
// into its neighbours' buffers through mapped peer pointers (NVLink), instead of NCCL messages.
// k_push_rows copies rows that are already computed (start-up level, initial state, remainder
// levels); the temporally blocked stencil pushes its boundary rows itself (TbArgs::pu_* / pd_*).
// k_peer_signal publishes "epoch e done" into the neighbours' mailboxes after a fence;
// k_peer_wait makes the receiving stream wait for its local mailbox.
// ------------------------------------------------------------------------------------------
template <typename T>
struct PushArgs {
    const T* src;      // this slab's buffer (view: storage row 1 = first owned row)
    T* pu;             // upper neighbour's buffer, shifted: this slab's row r ↦ its row r + ny_up (or null)
    T* pd;             // lower neighbour's buffer, shifted: row r ↦ its row r − ny_local (or null)
    int64_t pitch, mstride, pu_mstride, pd_mstride;
    int64_t nx, ny_local;
    int32_t nrows, batch;
};

template <typename T>
__global__ void k_push_rows(const PushArgs<T> a) {
    const int64_t per = int64_t(a.nrows) * a.nx;                 // elements per direction and member
    const int64_t total = per * 2 * a.batch;
    for (int64_t e = blockIdx.x * int64_t(blockDim.x) + threadIdx.x; e < total; e += int64_t(gridDim.x) * blockDim.x) {
        const int64_t i = e % a.nx;
        const int64_t rest = e / a.nx;
        const int64_t k = rest % a.nrows;
        const int64_t dirb = rest / a.nrows;
        const int dir = int(dirb & 1);
        const int64_t b = dirb >> 1;
        if (dir == 0) {
            if (!a.pu) continue;
            const int64_t r = 1 + k;                                  // first owned rows go up
            a.pu[b * a.pu_mstride + r * a.pitch + i] = a.src[b * a.mstride + r * a.pitch + i];
        } else {
            if (!a.pd) continue;
            const int64_t r = a.ny_local - a.nrows + 1 + k;           // last owned rows go down
            a.pd[b * a.pd_mstride + r * a.pitch + i] = a.src[b * a.mstride + r * a.pitch + i];
        }
    }
}

// Wait until the mailbox slots of the existing neighbours reach `target` (acquire), bounded:
// after ~20 s the error word is set and the kernel returns (the host reports it).  On one GPU the
// ranks of a process share one stream and are issued epoch by epoch, so the wait is always
// already satisfied there; across GPUs it is the rank's own stream that waits.
__global__ void k_peer_wait(const unsigned int* mbox, int has_up, int has_dn, unsigned int target, unsigned int* err) {
    if (threadIdx.x != 0) return;
    unsigned long long t0;
    asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t0));
    for (int side = 0; side < 2; ++side) {
        if (!(side == 0 ? has_up : has_dn)) continue;
        for (;;) {
            unsigned int v;
            asm volatile("ld.acquire.sys.global.u32 %0, [%1];" : "=r"(v) : "l"(mbox + side) : "memory");
            if (int(v - target) >= 0) break;
            unsigned long long t;
            asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
            if (t - t0 > 20000000000ull) {
                atomicExch(err, 1u);
                return;
            }
            __nanosleep(256);
        }
    }
}

__global__ void k_peer_signal(unsigned int* up_slot, unsigned int* dn_slot, unsigned int epoch) {
    if (threadIdx.x == 0) {
        __threadfence_system();
        if (up_slot) asm volatile("st.release.sys.global.u32 [%0], %1;" ::"l"(up_slot), "r"(epoch) : "memory");
        if (dn_slot) asm volatile("st.release.sys.global.u32 [%0], %1;" ::"l"(dn_slot), "r"(epoch) : "memory");
    }
}

// ------------------------------------------------------------------------------------------
// plumbing kernels
// ------------------------------------------------------------------------------------------
// Force the Dirichlet nodes of the slab (global rows 0 / ny−1, columns 0 / nx−1) and the padding
// columns to +0 (R10).
template <typename T>
__global__ void k_zero_boundary(T* __restrict__ u, int dim, int64_t nx, int64_t ny, int64_t r0, int64_t ny_local,
                                int64_t pitch, int64_t mstride) {
    const int b = blockIdx.y;
    T* ub = u + b * mstride;
    const int64_t rows = (dim == 1) ? 1 : ny_local;
    const int64_t total = rows * pitch;
    for (int64_t k = blockIdx.x * int64_t(blockDim.x) + threadIdx.x; k < total; k += int64_t(gridDim.x) * blockDim.x) {
        const int64_t i = k % pitch;
        const int64_t s = (dim == 1) ? 0 : 1 + k / pitch;
        const int64_t g = (dim == 1) ? 0 : r0 + s - 1;
        const bool bnd = (i == 0) || (i >= nx - 1) || (dim == 2 && (g == 0 || g == ny - 1));
        if (bnd) ub[s * pitch + i] = (T)0;
    }
}

// ------------------------------------------------------------------------------------------
// S5 fused into the temporally blocked pass (EN variant of k_step2d_tb): out[b] = w · Σ of member b's
// item partials (the node form of the energy, R30) over the pass's launches (segments: offset,
// partials per member; a split slab pass has two), fixed order (one warp per member).
// ------------------------------------------------------------------------------------------
__global__ void k_tb_energy_final(const double* __restrict__ part, int nseg, int64_t off0, int64_t pm0, int64_t off1,
                                  int64_t pm1, double w, double* __restrict__ out) {
    const int b = blockIdx.x;
    double v = 0.0;
    for (int sg = 0; sg < nseg; ++sg) {
        const int64_t off = sg ? off1 : off0, pm = sg ? pm1 : pm0;
        for (int64_t k = threadIdx.x; k < pm; k += 32) v += part[off + b * pm + k];
    }
    v = warp_sum(v);
    if (threadIdx.x == 0) out[b] = w * v;
}

// ------------------------------------------------------------------------------------------
// Measurement: the non-contracted add/multiply throughput the stencil's arithmetic runs on (the
// ALU roof of bench.py's roofline, measured instead of derived).  Eight independent chains per
// thread of (x + b)·a − b — two adds to one multiply, the stencil's mix — with a = 1 and b passed
// at run time, so nothing folds; 2048 threads per SM.
// ------------------------------------------------------------------------------------------
template <typename T>
__global__ void __launch_bounds__(256) k_alu_probe(T* __restrict__ out, int iters, T a, T b) {
    T x[8];
#pragma unroll
    for (int i = 0; i < 8; ++i) x[i] = T(threadIdx.x + i);
    for (int it = 0; it < iters; ++it) {
#pragma unroll
        for (int i = 0; i < 8; ++i) x[i] = r_add(x[i], b);
#pragma unroll
        for (int i = 0; i < 8; ++i) x[i] = r_mul(x[i], a);
#pragma unroll
        for (int i = 0; i < 8; ++i) x[i] = r_sub(x[i], b);
    }
    T acc = x[0];
#pragma unroll
    for (int i = 1; i < 8; ++i) acc = r_add(acc, x[i]);
    if (acc == T(-1.2345)) out[threadIdx.x] = acc;   // never true: keeps the chains alive
}

#endif  // TSW_TB_UNIT

}  // namespace tsw
