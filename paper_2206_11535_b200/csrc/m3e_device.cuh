// m3e_device.cuh -- per-frame device math of the Mu3e online event selection
// (PAPER.md = arXiv 2206.11535).  Selection cuts and the triplet fit run in fp32
// (one lane per combination / per candidate); the rarely executed vertex stage
// runs in fp64.  This file shares nothing with oracle/ (the CPU reference); the
// readings R<n> it follows are listed in DESIGN.md.
#pragma once
#include <cstdint>
#include <cuda_runtime.h>

#include "m3e.h"

// fp32 fit math is also compiled for the host (tools/fit_numerics.cu) to study
// its rounding against the oracle without a GPU
#define M3E_HD __host__ __device__ __forceinline__
// fit_triplet / arc_phi: inlined (their Triplet results then stay in
// registers instead of the local-memory stack; measured -8% filter kernel time
// once the selection moved to its own kernel); M3E_FIT_NOINLINE builds one
// out-of-line copy instead (smaller code)
#if defined(__CUDA_ARCH__) && defined(M3E_FIT_NOINLINE)
#define M3E_HD_CALL __host__ __device__ __noinline__
#elif defined(__CUDA_ARCH__)
#define M3E_HD_CALL __host__ __device__ __forceinline__
#else
#define M3E_HD_CALL __host__ __device__ inline
#endif

#ifndef M3E_NEWTON_IT_FINAL
#define M3E_NEWTON_IT_FINAL 1   // Newton steps for the track parameters' arc (R11)
#endif
#ifndef M3E_NEWTON_IT
#define M3E_NEWTON_IT 1   // Newton steps of arc_phi (host study, tools/fit_numerics_study.py: 1, 2, 3 give
                          // identical decisions, layer-3 hits and deviations on 140k candidates)
#endif

namespace m3e {

constexpr float kInfF = __builtin_huge_valf();
constexpr float kPiF = 3.14159265358979323846f;
constexpr double kPi = 3.14159265358979323846;
constexpr double kMuMass = 105.6583755;   // MeV (PDG), m_mu c^2 of Eq. 1
constexpr double kEMass = 0.51099895;     // MeV (PDG)
constexpr double kPtConv = 0.299792458;   // MeV/c per (T mm)
constexpr int kMaxLayerHits = 1024;       // 10-bit candidate index fields

// Compact fp32 primitives for the fit (code size matters: every warp of an SM
// can be in a different stage, so the hot code must stay in the I-cache).
// rcp: one MUFU.RCP (rcp.approx.ftz, <= 1 ulp): the fit is compared at 1e-4.
M3E_HD float rcp(float x) {
#ifdef __CUDA_ARCH__
    float r;
    asm("rcp.approx.ftz.f32 %0, %1;" : "=f"(r) : "f"(x));
    return r;
#else
    return 1.0f / x;
#endif
}
// sqrt: one MUFU.SQRT (sqrt.approx.ftz, ~1 ulp) instead of the IEEE-rounded
// sequence with its slow-path branch: the fit is compared at 1e-4 and the
// Selection Cuts' decisions at 1e-5 relative of a threshold
M3E_HD float fsqrt(float x) {
#ifdef __CUDA_ARCH__
    float r;
    asm("sqrt.approx.ftz.f32 %0, %1;" : "=f"(r) : "f"(x));
    return r;
#else
    return sqrtf(x);
#endif
}
// Packed fp32 pairs: sm_100 issues FFMA2 / FMUL2 / FADD2 (two fp32 lanes per
// instruction); the fit evaluates its two arcs side by side with them.  Per
// component the numerics are fmaf / fmul / fadd (round to nearest).  The host
// build (numerics studies) uses the scalar forms.
#ifndef M3E_PACKED
#define M3E_PACKED 1
#endif
M3E_HD float2 f2(float a, float b) { return make_float2(a, b); }
M3E_HD float2 f2s(float a) { return make_float2(a, a); }
M3E_HD float2 mul2(float2 a, float2 b) {
#if defined(__CUDA_ARCH__) && __CUDA_ARCH__ >= 1000 && M3E_PACKED
    return __fmul2_rn(a, b);
#else
    return make_float2(a.x * b.x, a.y * b.y);
#endif
}
M3E_HD float2 fma2(float2 a, float2 b, float2 c) {
#if defined(__CUDA_ARCH__) && __CUDA_ARCH__ >= 1000 && M3E_PACKED
    return __ffma2_rn(a, b, c);
#else
    return make_float2(fmaf(a.x, b.x, c.x), fmaf(a.y, b.y, c.y));
#endif
}
M3E_HD float2 add2(float2 a, float2 b) {
#if defined(__CUDA_ARCH__) && __CUDA_ARCH__ >= 1000 && M3E_PACKED
    return __fadd2_rn(a, b);
#else
    return make_float2(a.x + b.x, a.y + b.y);
#endif
}
M3E_HD float2 sqrt2(float2 a) { return make_float2(fsqrt(a.x), fsqrt(a.y)); }
// 1/sqrt: one MUFU.RSQ (rsqrt.approx.ftz, ~1 ulp) where a square root is only divided by
M3E_HD float frsqrt(float x) {
#ifdef __CUDA_ARCH__
    float r;
    asm("rsqrt.approx.ftz.f32 %0, %1;" : "=f"(r) : "f"(x));
    return r;
#else
    return 1.0f / sqrtf(x);
#endif
}
M3E_HD float2 rsqrt2(float2 a) { return make_float2(frsqrt(a.x), frsqrt(a.y)); }
M3E_HD float2 rcp2(float2 a) { return make_float2(rcp(a.x), rcp(a.y)); }

#ifndef M3E_FAST_TRIG
#define M3E_FAST_TRIG 1   // 0: CUDA asinf / atan2f in the fit
#endif
// asin of 0 <= x <= 1: odd minimax polynomial on [0, 1/2] (Cephes asinf
// coefficients, ~1 ulp), asin x = pi/2 - 2 asin(sqrt((1 - x)/2)) above; branch-free
M3E_HD float fasin(float x) {
#if M3E_FAST_TRIG
    const bool big = x > 0.5f;
    const float z = big ? 0.5f * (1.0f - x) : x * x;
    const float t = big ? fsqrt(z) : x;
    const float p = ((((4.2163199048e-2f * z + 2.4181311049e-2f) * z + 4.5470025998e-2f) * z + 7.4953002686e-2f) * z +
                     1.6666752422e-1f) * z * t + t;
    return big ? 1.57079632679f - 2.0f * p : p;
#else
    return asinf(x);
#endif
}
// fasin of a pair (0 <= x <= 1), the polynomial in FFMA2
M3E_HD float2 fasin2(float2 x) {
#if M3E_FAST_TRIG
    const bool bx = x.x > 0.5f, by = x.y > 0.5f;
    const float2 z = f2(bx ? 0.5f * (1.0f - x.x) : x.x * x.x, by ? 0.5f * (1.0f - x.y) : x.y * x.y);
    const float2 t = f2(bx ? fsqrt(z.x) : x.x, by ? fsqrt(z.y) : x.y);
    float2 p = fma2(f2s(4.2163199048e-2f), z, f2s(2.4181311049e-2f));
    p = fma2(p, z, f2s(4.5470025998e-2f));
    p = fma2(p, z, f2s(7.4953002686e-2f));
    p = fma2(p, z, f2s(1.6666752422e-1f));
    p = fma2(mul2(p, z), t, t);
    return f2(bx ? 1.57079632679f - 2.0f * p.x : p.x, by ? 1.57079632679f - 2.0f * p.y : p.y);
#else
    return make_float2(asinf(x.x), asinf(x.y));
#endif
}
// atan2: octant reduction to [0, 1], then tan(pi/8) reduction and the Cephes atanf
// polynomial (~2 ulp); atan2(0, 0) = 0; branch-free
M3E_HD float fatan2(float y, float x) {
#if M3E_FAST_TRIG
    const float ax = fabsf(x), ay = fabsf(y);
    const float mx = fmaxf(ax, ay), mn = fminf(ax, ay);
    // t = mn / mx; above tan(pi/8) the reduced argument (t - 1) / (t + 1) =
    // (mn - mx) / (mn + mx): one reciprocal either way
    const bool r = mn > 0.41421356237f * mx;
    const float tt = mx > 0.0f ? (r ? mn - mx : mn) * rcp(r ? mn + mx : mx) : 0.0f;
    const float z = tt * tt;
    float a = (((8.05374449538e-2f * z - 1.38776856032e-1f) * z + 1.99777106478e-1f) * z - 3.33329491539e-1f) * z * tt + tt;
    a = r ? a + 0.78539816340f : a;
    a = ay > ax ? 1.57079632679f - a : a;
    a = x < 0.0f ? 3.14159265359f - a : a;
    return copysignf(a, y);
#else
    return atan2f(y, x);
#endif
}
// sin / cos of 0 <= x <= pi/2 by Taylor polynomials of degree 11 / 12
// (truncation < 6e-8 absolute on the interval; no range reduction needed).
M3E_HD void sincos_half(float x, float& s, float& c) {
    const float x2 = x * x;
    s = x * (1.0f + x2 * (-1.6666667e-1f + x2 * (8.3333333e-3f + x2 * (-1.9841270e-4f +
                                                                           x2 * (2.7557319e-6f + x2 * -2.5052108e-8f)))));
    c = 1.0f + x2 * (-0.5f + x2 * (4.1666667e-2f + x2 * (-1.3888889e-3f + x2 * (2.4801587e-5f +
                                                                              x2 * (-2.7557319e-7f + x2 * 2.0876757e-9f)))));
}

// cos of the transverse angle between two hits, Eq. 4: (xa xb + ya yb) / (ra rb),
// with a pinned operation order (one product, one fma, one product; no
// contraction left to the compiler), so that every walk of the Selection Cuts,
// scalar or packed fp32 (cos_sep2), takes identical decisions
M3E_HD float cos_sep(float xa, float ya, float xb, float yb, float inv) {
#ifdef __CUDA_ARCH__
    return __fmul_rn(__fmaf_rn(xa, xb, __fmul_rn(ya, yb)), inv);
#else
    return fmaf(xa, xb, ya * yb) * inv;
#endif
}
#if !defined(__CUDA_ARCH__) || __CUDA_ARCH__ >= 1000
// two hits b against one hit a (sm_100 FMUL2 / FFMA2; per component = cos_sep)
__device__ __forceinline__ float2 cos_sep2(float xa, float ya, float2 xb, float2 yb, float inv) {
    return __fmul2_rn(__ffma2_rn(make_float2(xa, xa), xb, __fmul2_rn(make_float2(ya, ya), yb)), make_float2(inv, inv));
}
#endif

// Kernel-side parameters, derived once on the host from m3e_params.
struct DevParams {
    float R[4];                 // layer radii
    float inv_dr01, inv_dr12;   // 1/(R1-R0), 1/(R2-R1)         (Eq. 2)
    float inv_r0r1, inv_r1r2;   // 1/(R0 R1), 1/(R1 R2)         (Eq. 4)
    float dl_max, c01_min, c12_min, rt_min, rt_max;
    float rt_min2, rt_max2;   // squared r_t window (selection kernel: no square roots)
    float chl;                  // sigma_MS = chl * k  (Highland at p = ptb / k, R7)
    float chi2_max;
    float R3sq;                 // layer-3 radius squared
    int cuts_max, max_tracks, max_combs;
    // vertex stage (fp64)
    double ptb;                 // kPtConv * B: p = ptb / k
    double chl_d;
    double e_window, rlim, sig_pix2, chi2v_max, tdist_max, ptot_max, target_r, target_half;
};

// Delta-lambda (Eq. 2-3) of (i0, i1, i2) as z2 / dr12 - u(i0, i1) with the pair term
//   u = z1 (1/dr12 + 1/dr01) - z0 / dr01 = z1 / dr12 + (z1 - z0) / dr01,
// both with a pinned operation order so that every walk of the Selection Cuts
// (per frame, flat, pair-factorised, mask-factorised) takes identical decisions:
// pass iff |fma(z2, 1/dr12, -u)| <= dl_max
M3E_HD float pair_u(const DevParams& P, float z0, float z1) {
#ifdef __CUDA_ARCH__
    return __fmaf_rn(z1, P.inv_dr12, __fmul_rn(__fsub_rn(z1, z0), P.inv_dr01));
#else
    return fmaf(z1, P.inv_dr12, (z1 - z0) * P.inv_dr01);
#endif
}

struct Frame {                  // one frame's hits, pointers to its first hit
    const float* x;
    const float* y;
    const float* z;
    int s[4];                   // layer starts relative to the frame's first hit
    int n[4];                   // hits per layer
};

M3E_HD float3 hit(const Frame& F, int layer, int i) {
    int g = F.s[layer] + i;
    return make_float3(F.x[g], F.y[g], F.z[g]);
}

// ---------------------------------------------------------------- Eq. 5 ----
// r_tc = d01 d12 d20 / (2 [(h0 - h1) x (h2 - h1)]_z); > 0 clockwise (R5);
// collinear -> +inf.
// transverse chord lengths (d01, d12) of the two arcs h0 -> h1, h1 -> h2, rounded as
// fma(dx, dx, dy dy) (the fit's own order)
M3E_HD float2 chords(float3 h0, float3 h1, float3 h2) {
    const float2 dx = f2(h1.x - h0.x, h2.x - h1.x), dy = f2(h1.y - h0.y, h2.y - h1.y);
    return sqrt2(fma2(dx, dx, mul2(dy, dy)));
}
// r_tc (Eq. 5) with the chords (d01, d12) = chords(h0, h1, h2) already known (the
// fit reuses them for its arcs, the extension and the track parameters)
M3E_HD float circle_radius_d(float3 h0, float3 h1, float3 h2, float2 d) {
    const float ax = h0.x - h1.x, ay = h0.y - h1.y, bx = h2.x - h1.x, by = h2.y - h1.y;
    const float cz = ax * by - ay * bx;
    if (cz == 0.0f) return kInfF;
    const float cx = h2.x - h0.x, cy = h2.y - h0.y;
    const float d20 = fsqrt(cx * cx + cy * cy);
    return d.x * d.y * d20 * rcp(2.0f * cz);
}
M3E_HD float circle_radius(float3 h0, float3 h1, float3 h2) { return circle_radius_d(h0, h1, h2, chords(h0, h1, h2)); }

// ------------------------------------------------------- Selection Cuts ----
// Alg. 2 tests: Delta-lambda (Eq. 2-3) first, then Phi_01, Phi_12 (Eq. 4) and
// r_tc (Eq. 5).  The survivor set is the AND of the four tests, so evaluating
// them in two passes (below) does not change it.
__device__ __forceinline__ bool pass_dlambda(const DevParams& P, const Frame& F, int i0, int i1, int i2) {
    const float z0 = F.z[F.s[0] + i0], z1 = F.z[F.s[1] + i1], z2 = F.z[F.s[2] + i2];
    const float dl = (z2 - z1) * P.inv_dr12 - (z1 - z0) * P.inv_dr01;
    return fabsf(dl) <= P.dl_max;
}
__device__ __forceinline__ bool pass_rest(const DevParams& P, const Frame& F, int i0, int i1, int i2, float& rt) {
    const int g0 = F.s[0] + i0, g1 = F.s[1] + i1, g2 = F.s[2] + i2;
    const float x0 = F.x[g0], y0 = F.y[g0], x1 = F.x[g1], y1 = F.y[g1];
    if (!(cos_sep(x0, y0, x1, y1, P.inv_r0r1) >= P.c01_min)) return false;
    const float x2 = F.x[g2], y2 = F.y[g2];
    if (!(cos_sep(x1, y1, x2, y2, P.inv_r1r2) >= P.c12_min)) return false;
    rt = circle_radius(make_float3(x0, y0, 0.0f), make_float3(x1, y1, 0.0f), make_float3(x2, y2, 0.0f));
    const float ar = fabsf(rt);
    return ar >= P.rt_min && ar <= P.rt_max;
}

// r_tc window of Eq. 5 (the last of the Selection Cuts)
__device__ __forceinline__ bool pass_rtc(const DevParams& P, const Frame& F, int i0, int i1, int i2, float& rt) {
    const int g0 = F.s[0] + i0, g1 = F.s[1] + i1, g2 = F.s[2] + i2;
    rt = circle_radius(make_float3(F.x[g0], F.y[g0], 0.0f), make_float3(F.x[g1], F.y[g1], 0.0f),
                       make_float3(F.x[g2], F.y[g2], 0.0f));
    const float ar = fabsf(rt);
    return ar >= P.rt_min && ar <= P.rt_max;
}

// the same window without r_tc itself: r_tc^2 = d01^2 d12^2 d20^2 / (2 cz)^2
// (collinear, cz = 0: fails, as r_tc = inf does)
__device__ __forceinline__ bool pass_rtc_sq(const DevParams& P, const Frame& F, int i0, int i1, int i2) {
    const int g0 = F.s[0] + i0, g1 = F.s[1] + i1, g2 = F.s[2] + i2;
    const float x1 = F.x[g1], y1 = F.y[g1];
    const float ax = F.x[g0] - x1, ay = F.y[g0] - y1, bx = F.x[g2] - x1, by = F.y[g2] - y1;
    const float cx = bx - ax, cy = by - ay;
    const float cz = ax * by - ay * bx;
    const float num = (ax * ax + ay * ay) * (bx * bx + by * by) * (cx * cx + cy * cy);
    const float den = 4.0f * cz * cz;
    return cz != 0.0f && num >= den * P.rt_min2 && num <= den * P.rt_max2;
}

// Warp-cooperative Selection Cuts of one frame, in the row-major (i0, i1, i2)
// order of Alg. 2.  The cuts are factorised by the hits they depend on (Eq. 2-5):
// Phi_01 by (i0, i1) alone, so
//   1. the (i0, i1) pairs are tested for Phi_01, 32 per step, and the survivors
//      (~22 %) appended with ballot + popc to the pair list `pl` (shared memory);
//   2. the first K <= 32 listed pairs are expanded against every layer-2 hit,
//      32 (k, i2) combinations per step in row-major order, and tested for
//      Delta-lambda and Phi_12; survivors (~11 %) go to the FIFO `q`;
//   3. each full 32 of the FIFO is tested for r_tc on all 32 lanes and the final
//      survivors compacted again with ballot + popc,
// so the stored candidates keep the enumeration order and the set is exactly the
// conjunction of the four cuts.  Stops once more than cuts_max survive (R3).
// emit(pos, packed, rt) is called for pos < cuts_max (rt = r_tc if kRt, else 0:
// the split path's fit kernel recomputes it).  Returns min(#survivors,
// cuts_max + 1) (warp-uniform).
template <bool kRt, class Emit>
__device__ __forceinline__ int select_frame_warp(const DevParams& P, const Frame& F, uint32_t* q, uint2* pl,
                                                 Emit emit) {
    const int lane = threadIdx.x & 31;
    const int n0 = F.n[0], n1 = F.n[1], n2 = F.n[2];
    const int np = n0 * n1;
    if (np == 0 || n2 == 0) return 0;
    const unsigned lt_mask = (1u << lane) - 1u;
    // mixed-radix digits: quotients of x by n as floor((x + 0.5) / n), >= 0.5/n
    // away from an integer for the x < 2^15 used here, far above the error of rcp
    const float in1 = rcp((float)n1), in2 = rcp((float)n2);
    int j0 = (int)(((float)lane + 0.5f) * in1), j1 = lane - j0 * n1;   // lane's first pair
    const int a1 = (int)(32.5f * in1), b1 = 32 - a1 * n1;                // step of 32 pairs
    int count = 0, qn = 0, pn = 0, pnext = 0;
    // r_tc for q[0..n) (n <= 32); true once the frame overflows
    auto drain = [&](int n) -> bool {   // branch-free: lanes >= n test a clamped entry
        float rt = 0.0f;
        const uint32_t pk = q[min(lane, n - 1)];
        bool pass;
        if constexpr (kRt) pass = pass_rtc(P, F, pk & 1023u, (pk >> 10) & 1023u, (pk >> 20) & 1023u, rt);
        else pass = pass_rtc_sq(P, F, pk & 1023u, (pk >> 10) & 1023u, (pk >> 20) & 1023u);
        pass = pass && lane < n;
        const unsigned m = __ballot_sync(0xffffffffu, pass);
        const int pos = count + __popc(m & lt_mask);
        if (pass && pos < P.cuts_max) emit(pos, pk, rt);
        count += __popc(m);
        return count > P.cuts_max;
    };
    for (;;) {
        // 1. refill the pair list to >= 32 Phi_01 survivors (or all pairs)
        while (pn < 32 && pnext < np) {
            // branch-free: lanes past the last pair test a clamped (valid) one
            const int g0 = F.s[0] + min(j0, n0 - 1), g1 = F.s[1] + j1;
            const bool pass = (j0 < n0) & (cos_sep(F.x[g0], F.y[g0], F.x[g1], F.y[g1], P.inv_r0r1) >= P.c01_min);
            const unsigned m = __ballot_sync(0xffffffffu, pass);
            // Delta-lambda = z2 / dr12 - u(i0, i1), u = z1 (1/dr12 + 1/dr01) - z0 / dr01
            const float u = pair_u(P, F.z[g0], F.z[g1]);
            if (pass) pl[pn + __popc(m & lt_mask)] = make_uint2((uint32_t)j0 | ((uint32_t)j1 << 10), __float_as_uint(u));
            pn += __popc(m);
            pnext += 32;
            j1 += b1;
            if (j1 >= n1) { j1 -= n1; ++j0; }
            j0 += a1;
        }
        if (pn == 0) break;
        __syncwarp();
        // 2. expand the first K listed pairs against layer 2
        const int K = min(pn, 32), nk = K * n2;
        for (int cb = 0; cb < nk; cb += 32) {
            // branch-free: lanes past the end evaluate a clamped (valid) combination
            const int c = min(cb + lane, nk - 1);
            const int k = (int)(((float)c + 0.5f) * in2), i2 = c - k * n2;
            const uint2 pe = pl[k];
            const uint32_t pk = pe.x | ((uint32_t)i2 << 20);
            const int g1 = F.s[1] + (int)(pe.x >> 10), g2 = F.s[2] + i2;
            const float dl = fmaf(F.z[g2], P.inv_dr12, -__uint_as_float(pe.y));
            const float c12 = cos_sep(F.x[g1], F.y[g1], F.x[g2], F.y[g2], P.inv_r1r2);
            const bool pass = (cb + lane < nk) & (fabsf(dl) <= P.dl_max) & (c12 >= P.c12_min);
            const unsigned m = __ballot_sync(0xffffffffu, pass);
            if (pass) q[qn + __popc(m & lt_mask)] = pk;
            qn += __popc(m);
            if (qn >= 32) {
                __syncwarp();
                if (drain(32)) return P.cuts_max + 1;
                const uint32_t v = lane < qn - 32 ? q[32 + lane] : 0u;
                __syncwarp();
                if (lane < qn - 32) q[lane] = v;
                qn -= 32;
            }
            __syncwarp();
        }
        // drop the K expanded pairs
        const uint2 v = lane < pn - K ? pl[K + lane] : make_uint2(0u, 0u);
        __syncwarp();
        if (lane < pn - K) pl[lane] = v;
        pn -= K;
        __syncwarp();
    }
    __syncwarp();
    if (qn > 0 && drain(qn)) return P.cuts_max + 1;
    return count;
}

// Where a selected candidate goes: flat index base + pos; below `split` into
// the shared-memory array (s*), else into the global array (g*).
struct CandSink {
    uint32_t* si;
    float* sr;
    uint32_t* gi;
    float* gr;
    uint32_t base, split;
    __device__ __forceinline__ void put(int pos, uint32_t packed, float rt) const {
        const uint32_t fi = base + (uint32_t)pos;
        if (fi < split) { si[fi] = packed; sr[fi] = rt; }
        else { gi[fi] = packed; gr[fi] = rt; }
    }
};

__device__ __forceinline__ bool pass_rt(const DevParams& P, const Frame& F, int i0, int i1, int i2, float& rt) {
    const int g0 = F.s[0] + i0, g1 = F.s[1] + i1, g2 = F.s[2] + i2;
    rt = circle_radius(make_float3(F.x[g0], F.y[g0], 0.0f), make_float3(F.x[g1], F.y[g1], 0.0f),
                       make_float3(F.x[g2], F.y[g2], 0.0f));
    const float ar = fabsf(rt);
    return ar >= P.rt_min && ar <= P.rt_max;
}

// ballot-compact the pairs (ia in layer la, ib in layer lb) passing cos Phi >= cmin
// in row-major order (ia outer), with t = u(ia, ib) (kU: layers 0, 1) or z_b
// (layers 1, 2); returns the count (> cap: overflow, lists incomplete)
template <bool kU>
__device__ __forceinline__ int pair_list(const DevParams& P, const Frame& F, int la, int lb, float inv_rr, float cmin,
                                         uint32_t* lst, float* tv, int cap) {
    const int lane = threadIdx.x & 31;
    const unsigned lt_mask = (1u << lane) - 1u;
    const int na = F.n[la], nb = F.n[lb];
    const int tot = na * nb;
    const float inb = rcp((float)nb);   // quotients of x < 64 by nb, as in select_frame_warp
    int ia = (int)(((float)lane + 0.5f) * inb), ib = lane - ia * nb;
    const int sa = (int)(32.5f * inb), sb = 32 - sa * nb;
    int cnt = 0;
    for (int base = 0; base < tot; base += 32) {
        bool pass = false;
        float t = 0.0f;
        if (ia < na) {
            const int ga = F.s[la] + ia, gb = F.s[lb] + ib;
            pass = cos_sep(F.x[ga], F.y[ga], F.x[gb], F.y[gb], inv_rr) >= cmin;
            t = kU ? pair_u(P, F.z[ga], F.z[gb]) : F.z[gb];
        }
        const unsigned m = __ballot_sync(0xffffffffu, pass);
        const int pos = cnt + __popc(m & lt_mask);
        if (pass && pos < cap) {
            lst[pos] = (uint32_t)ia | ((uint32_t)ib << 10);
            tv[pos] = t;
        }
        cnt += __popc(m);
        if (cnt > cap) return cnt;
        ib += sb;
        if (ib >= nb) { ib -= nb; ++ia; }
        ia += sa;
    }
    return cnt;
}

// Selection Cuts of a big frame (phase-II occupancy), pair-factorised: Phi_01
// depends only on (i0, i1), Phi_12 only on (i1, i2), and Delta-lambda =
// t12(i1, i2) - t01(i0, i1) (Eq. 2-4).  1. list the (i0, i1) pairs passing Phi_01,
// row-major, with t01; 2. list the (i1, i2) pairs passing Phi_12 (grouped by i1)
// with t12; 3. enumerate list-1 entries x their i1's group of list 2 in row-major
// (i0, i1, i2) order, test Delta-lambda, push survivors to the FIFO and test r_tc
// on full warps (same survivor set and order as select_frame_warp, R3 overflow).
// Returns -1 if a list exceeds kPairCapG (caller falls back to select_frame_warp).
// Out of line: phase-I frames never take it, so its code stays out of the I-cache.
static __device__ __noinline__ int select_frame_big(const DevParams* __restrict__ Pp, const Frame& Fin, uint32_t* q,
                                                    uint32_t* X, const CandSink& sink_in, int cap) {
    const DevParams& P = *Pp;
    // the frame view and the sink in registers: the caller's copies are in local
    // memory (their addresses are passed), and the list stores below could alias
    // them, forcing a reload of every field on every access
    const Frame F = Fin;
    const CandSink sink = sink_in;
    const int lane = threadIdx.x & 31;
    const unsigned lt_mask = (1u << lane) - 1u;
    const int n1 = F.n[1];
    uint32_t* l01 = X;
    float* u01 = reinterpret_cast<float*>(X + cap);    // u(i0, i1) of list 1
    uint32_t* l12 = X + 2 * cap;
    float* z12 = reinterpret_cast<float*>(X + 3 * cap);   // z2 of list 2
    uint32_t* off12 = X + 4 * cap;                 // n1 + 1 entries
    uint32_t* wpre = off12 + (kMaxLayerHits + 2);  // cap + 1 entries
    const int c01 = pair_list<true>(P, F, 0, 1, P.inv_r0r1, P.c01_min, l01, u01, cap);
    if (c01 > cap) return -1;
    const int c12 = pair_list<false>(P, F, 1, 2, P.inv_r1r2, P.c12_min, l12, z12, cap);
    if (c12 > cap) return -1;
    __syncwarp();
    for (int i1 = lane; i1 <= n1; i1 += 32) {      // off12[i1] = lower bound of i1 in list 2
        int lo = 0, hi = c12;
        while (lo < hi) {
            const int mid = (lo + hi) >> 1;
            if ((int)(l12[mid] & 1023u) < i1) lo = mid + 1; else hi = mid;
        }
        off12[i1] = (uint32_t)lo;
    }
    __syncwarp();
    uint32_t run = 0;                               // work prefix over list 1
    for (int b0 = 0; b0 < c01; b0 += 32) {
        const int p = b0 + lane;
        uint32_t w = 0;
        if (p < c01) {
            const int i1 = (l01[p] >> 10) & 1023u;
            w = off12[i1 + 1] - off12[i1];
        }
        uint32_t inc = w;
#pragma unroll
        for (int o = 1; o < 32; o <<= 1) {
            const uint32_t t = __shfl_up_sync(0xffffffffu, inc, o);
            if (lane >= o) inc += t;
        }
        if (p < c01) wpre[p] = run + inc - w;
        run += __shfl_sync(0xffffffffu, inc, 31);
    }
    __syncwarp();
    const long long Wk = run;
    int count = 0, qn = 0;
    auto drain = [&](int n) -> bool {
        float rt = 0.0f;
        uint32_t pk = 0;
        bool pass = false;
        if (lane < n) {
            pk = q[lane];
            pass = pass_rt(P, F, pk & 1023u, (pk >> 10) & 1023u, (pk >> 20) & 1023u, rt);
        }
        const unsigned m = __ballot_sync(0xffffffffu, pass);
        const int pos = count + __popc(m & lt_mask);
        if (pass && pos < P.cuts_max) sink.put(pos, pk, rt);
        count += __popc(m);
        return count > P.cuts_max;
    };
    int lo = 0;   // this lane's list-1 entry, advanced monotonically (e grows by 32 per step)
    for (long long base = 0; base < Wk; base += 32) {
        const long long e = base + lane;
        bool pass = false;
        uint32_t pk = 0;
        if (e < Wk) {
            // list-1 entry: largest p with wpre[p] <= e (wpre non-decreasing)
            while (lo + 1 < c01 && (long long)wpre[lo + 1] <= e) ++lo;
            const uint32_t a = l01[lo];
            const int i1 = (a >> 10) & 1023u;
            const int k = (int)off12[i1] + (int)(e - (long long)wpre[lo]);
            const int i2 = (l12[k] >> 10) & 1023u;
            pass = fabsf(fmaf(z12[k], P.inv_dr12, -u01[lo])) <= P.dl_max;
            pk = (a & 1023u) | ((uint32_t)i1 << 10) | ((uint32_t)i2 << 20);
        }
        const unsigned m = __ballot_sync(0xffffffffu, pass);
        if (pass) q[qn + __popc(m & lt_mask)] = pk;
        qn += __popc(m);
        if (qn >= 32) {
            __syncwarp();
            if (drain(32)) return P.cuts_max + 1;
            const uint32_t v = lane < qn - 32 ? q[32 + lane] : 0u;
            __syncwarp();
            if (lane < qn - 32) q[lane] = v;
            qn -= 32;
            __syncwarp();
        }
    }
    __syncwarp();
    if (qn > 0 && drain(qn)) return P.cuts_max + 1;
    return count;
}

// ------------------------------------------------------------ Triplet Fit ----
// Single-triplet fit (Sec. IV-B-1, Eq. 6, readings R6-R8).  Each arc's bending
// angle Phi and polar angle theta are linearised in the 3D curvature k around
// the arc's circle solution (radius r_tc of Eq. 5) with analytic derivatives of
//   1/k^2 = d^2 / (4 sin^2(Phi/2)) + z^2 / Phi^2 ,   cos theta = z k / Phi.
// Around k_ref = (k_C01 + k_C12)/2, delta = k - k_ref:
//   Phi_MS(delta)   = al_phi + b_phi delta,  Theta_MS(delta) = al_th + b_th delta
// and chi2 = Phi_MS^2 w_phi + Theta_MS^2 w_th is minimised in closed form.
struct Triplet {
    int q;                       // +1 clockwise (e+), -1
    float kref, al_phi, b_phi, al_th, b_th, w_phi, w_th;
    float khat;                  // |kappa_t|
    float A;                     // 1 / sigma^2_kappa,t = b_phi^2 w_phi + b_th^2 w_th (Eq. 8 weight)
    // arc data kept for the extensions
    float phc[2], kc[2], dphi[2];
};

// d = the transverse chords (d01, d12) of the two arcs (chords())
M3E_HD_CALL bool fit_triplet(const DevParams& P, float3 h0, float3 h1, float3 h2, float rtc, float2 d,
                                            Triplet& T) {
    if (!(fabsf(rtc) < kInfF)) return false;
    T.q = rtc > 0.0f ? 1 : -1;
    const float r = fabsf(rtc);
    const float ir = rcp(r);
    // the two arcs h0 -> h1 (.x) and h1 -> h2 (.y) side by side (packed fp32)
    const float2 z = f2(h1.z - h0.z, h2.z - h1.z);
    float2 sv = mul2(d, f2s(0.5f * ir));
    sv = f2(fminf(sv.x, 1.0f), fminf(sv.y, 1.0f));
    const float2 phc = mul2(f2s(2.0f), fasin2(sv));
    const float2 rphc = mul2(f2s(r), phc);
    const float2 z2 = mul2(z, z);
    const float2 iden = rsqrt2(fma2(rphc, rphc, z2));
    const float2 kc = mul2(phc, iden);
    const float2 cthv = mul2(z, iden), sthv = mul2(rphc, iden);
    const float2 cs2 = fma2(make_float2(-sv.x, -sv.y), sv, f2s(1.0f));
    const float2 ch = sqrt2(f2(fmaxf(0.0f, cs2.x), fmaxf(0.0f, cs2.y)));   // cos(Phi_C / 2)
    // dPhi/dk = (2/k^3) / (d^2 cos(Phi/2) / (4 sin^3(Phi/2)) + 2 z^2/Phi^3), sin(Phi_C/2) = d/(2r)
    const float2 iphc = rcp2(phc), ikc = rcp2(kc);
    const float2 iphc2 = mul2(iphc, iphc);
    const float2 dd = fma2(mul2(f2s(2.0f), z2), mul2(iphc2, iphc), mul2(mul2(f2s(r * r), ch), rcp2(sv)));
    const float2 dphi = mul2(mul2(mul2(f2s(2.0f), ikc), mul2(ikc, ikc)), rcp2(dd));
    // dtheta/dk = -z (Phi - k Phi') / (Phi^2 sin theta)
    const float2 dth = mul2(mul2(make_float2(-z.x, -z.y), fma2(make_float2(-kc.x, -kc.y), dphi, phc)),
                            mul2(iphc2, rcp2(sthv)));
    const float sth0 = sthv.x;
    T.phc[0] = phc.x; T.phc[1] = phc.y;
    T.kc[0] = kc.x; T.kc[1] = kc.y;
    T.dphi[0] = dphi.x; T.dphi[1] = dphi.y;
    const float dk = T.kc[1] - T.kc[0];
    T.kref = 0.5f * (T.kc[0] + T.kc[1]);
    T.b_phi = 0.5f * T.q * (T.dphi[0] + T.dphi[1]);
    T.al_phi = 0.25f * T.q * dk * (T.dphi[0] - T.dphi[1]);
    T.b_th = dth.y - dth.x;
    // theta_12 - theta_01 (both in (0, pi)) with one atan2
    const float dtheta = fatan2(sthv.y * cthv.x - cthv.y * sthv.x, cthv.y * cthv.x + sthv.y * sthv.x);
    T.al_th = dtheta - 0.5f * dk * (dth.y + dth.x);
    const float sig = P.chl * T.kref;
    T.w_th = rcp(sig * sig);
    T.w_phi = sth0 * sth0 * T.w_th;
    const float A = T.b_phi * T.b_phi * T.w_phi + T.b_th * T.b_th * T.w_th;
    if (!(A > 0.0f)) return false;
    const float B = T.al_phi * T.b_phi * T.w_phi + T.al_th * T.b_th * T.w_th;
    T.A = A;
    T.khat = T.kref - B * rcp(A);
    return true;
}

// chi2_t (Eq. 6, linearised) at signed global curvature kappa (Eq. 7)
M3E_HD float triplet_chi2(const Triplet& T, float kappa) {
    const float del = T.q * kappa - T.kref;
    const float fp = T.al_phi + T.b_phi * del, ft = T.al_th + T.b_th * del;
    return fp * fp * T.w_phi + ft * ft * T.w_th;
}

// exact short-arc bending angle: root of d^2/(4 sin^2(Phi/2)) + z^2/Phi^2 = 1/k^2
// on (0, pi] by Newton from `start` (the linearised value).  false if no short arc
// of curvature k joins the hits (1/k^2 < d^2/4 + z^2/pi^2).
template <int kIt = M3E_NEWTON_IT>
M3E_HD_CALL bool arc_phi(float d, float z, float k, float start, float& phi) {
    if (!(k > 0.0f)) return false;
    const float ik = rcp(k);
    const float R2 = ik * ik;
    const float d2 = 0.25f * d * d, z2 = z * z;
    if (R2 < d2 + z2 * (1.0f / (kPiF * kPiF))) return false;
    float p = fminf(fmaxf(start, 1e-6f), kPiF);
#pragma unroll 1
    for (int it = 0; it < kIt; ++it) {   // quadratic convergence from the linearised start
        float sh, ch;
        sincos_half(0.5f * p, sh, ch);
        const float is = rcp(sh), ip = rcp(p);
        const float is2 = is * is, ip2 = ip * ip;
        const float f = d2 * is2 + z2 * ip2 - R2;
        const float fp = -d2 * ch * is2 * is - 2.0f * z2 * ip2 * ip;
        p = fminf(fmaxf(p - f * rcp(fp), 1e-7f), kPiF);
    }
    phi = p;
    return true;
}

// Sec. IV-B-2 "Using this preliminary helix, the hit position in the fourth
// layer is estimated" (R9): continue the arc h1 -> h2 of curvature k past h2 to
// its first crossing of the layer-3 cylinder.
// (d = the chord h1 -> h2)
M3E_HD bool extrapolate(const DevParams& P, float3 h1, float3 h2, float d, const Triplet& T, float3& out) {
    const float k = T.khat;
    const float dx = h2.x - h1.x, dy = h2.y - h1.y, z = h2.z - h1.z;
    float phi;
    if (!arc_phi(d, z, k, T.phc[1] + T.dphi[1] * (k - T.kc[1]), phi)) return false;
    const float ik = rcp(k);
    const float cth = fminf(fmaxf(z * k * rcp(phi), -1.0f), 1.0f);
    const float rt = fsqrt(1.0f - cth * cth) * ik;
    // heading at h2 = chord direction turned by -q phi/2 (a clockwise arc turns by -phi)
    float sh, ch;
    sincos_half(0.5f * phi, sh, ch);
    const float id = rcp(d), ux = dx * id, uy = dy * id;
    const float ex = ux * ch + T.q * uy * sh, ey = uy * ch - T.q * ux * sh;
    // centre: clockwise (q = +1) to the right of the heading
    const float cx = h2.x + T.q * rt * ey, cy = h2.y - T.q * rt * ex;
    const float C2 = cx * cx + cy * cy;
    if (C2 == 0.0f) return false;
    // crossings of |p| = r3 and |p - c| = rt: p = a c^ +- hh n^ (no trigonometry)
    const float iC = frsqrt(C2);
    const float a = (P.R3sq - rt * rt + C2) * 0.5f * iC;
    const float hh2 = P.R3sq - a * a;
    if (hh2 < 0.0f) return false;                    // the helix never reaches layer 3
    const float hh = fsqrt(hh2);
    const float cux = cx * iC, cuy = cy * iC;
    const float ax = h2.x - cx, ay = h2.y - cy;
    // first crossing in the direction of motion: the smaller positive turning
    // angle from h2, compared on a monotone pseudo-angle of (cross, dot) in
    // (-2, 2] (no trigonometry); one atan2 for the chosen crossing's angle
    float bestp = 1e30f, bx = 0.0f, by = 0.0f, bcr = 0.0f, bdt = 0.0f;
#pragma unroll
    for (int s = -1; s <= 1; s += 2) {
        const float px = a * cux - s * hh * cuy, py = a * cuy + s * hh * cux;
        const float qx = px - cx, qy = py - cy;
        const float cr = ax * qy - ay * qx, dt = ax * qx + ay * qy;
        const float r = cr * rcp(fabsf(dt) + fabsf(cr));
        float t = -T.q * (dt >= 0.0f ? r : (cr >= 0.0f ? 2.0f - r : -2.0f - r));
        if (t < 0.0f) t += 4.0f;
        if (t > 0.0f && t < bestp) { bestp = t; bx = px; by = py; bcr = cr; bdt = dt; }
    }
    // turning angle from h2 to the crossing in the direction of motion, in (0, 2 pi)
    // (no crossing ahead, both at h2 itself: degenerate, as before 1e30)
    float best = 1e30f;
    if (bestp < 1e30f) {
        best = -T.q * fatan2(bcr, bdt);
        if (best < 0.0f) best += 2.0f * kPiF;
    }
    out = make_float3(bx, by, h2.z + cth * ik * best);
    return true;
}

// Track Reconstruction of one candidate (Sec. IV-B-2, Alg. 3, Eq. 7-8, R9-R11).
struct FitOut {
    int status;                  // 0 ok ... 6 domain, as m3e_fit_record.status
    int hit3;
    float kappa1, kappa2, var1, var2, kappa, chi2, cth01, cx, cy;
};

// h0, h1, h2 given; F supplies the frame's layer-3 hits (F.s[3], F.n[3])
// dc = chords(h0, h1, h2)
template <bool kPairs = true>
M3E_HD FitOut fit_candidate_hd(const DevParams& P, const Frame& F, float3 h0, float3 h1, float3 h2, float rtc,
                               float2 dc) {
    FitOut o;
    o.status = 0; o.hit3 = -1;
    o.kappa1 = o.kappa2 = o.var1 = o.var2 = o.kappa = o.chi2 = o.cth01 = o.cx = o.cy = 0.0f;
    Triplet T1, T2;
    if (!fit_triplet(P, h0, h1, h2, rtc, dc, T1)) { o.status = 1; return o; }
    o.kappa1 = T1.q * T1.khat;
    o.var1 = rcp(T1.A);
    float3 pred;
    if (!extrapolate(P, h1, h2, dc.y, T1, pred)) { o.status = 2; return o; }
    if (F.n[3] == 0) { o.status = 3; return o; }
    // find_closest_layer3_hit: 3D Euclidean, lowest index on ties (R10); every
    // distance rounded as (dx = x - px) dx dx, fma dy dy, fma dz dz and compared
    // in index order.  kPairs (phase-I frames, ~6 layer-3 hits that differ between
    // the lanes' frames): two hits per iteration in packed fp32, half the
    // divergent trip count; big frames (~56 hits, the same frame on every lane):
    // one hit per iteration, fewer instructions per hit
    float best = kInfF;
    int bi = 0;
    {
        const int n3 = F.n[3];
        const float* x3 = F.x + F.s[3];
        const float* y3 = F.y + F.s[3];
        const float* z3 = F.z + F.s[3];
        if constexpr (kPairs) {
            int i = 0;
            for (; i + 1 < n3; i += 2) {
                const float2 ex = add2(f2(x3[i], x3[i + 1]), f2s(-pred.x));
                const float2 ey = add2(f2(y3[i], y3[i + 1]), f2s(-pred.y));
                const float2 ez = add2(f2(z3[i], z3[i + 1]), f2s(-pred.z));
                const float2 d2 = fma2(ez, ez, fma2(ey, ey, mul2(ex, ex)));
                if (d2.x < best) { best = d2.x; bi = i; }
                if (d2.y < best) { best = d2.y; bi = i + 1; }
            }
            if (i < n3) {
                const float ex = x3[i] - pred.x, ey = y3[i] - pred.y, ez = z3[i] - pred.z;
                const float d2 = fmaf(ez, ez, fmaf(ey, ey, ex * ex));
                if (d2 < best) { best = d2; bi = i; }
            }
        } else {
            for (int i = 0; i < n3; ++i) {
                const float ex = x3[i] - pred.x, ey = y3[i] - pred.y, ez = z3[i] - pred.z;
                const float d2 = fmaf(ez, ez, fmaf(ey, ey, ex * ex));
                if (d2 < best) { best = d2; bi = i; }
            }
        }
    }
    o.hit3 = bi;
    const float3 h3 = hit(F, 3, bi);
    const float2 dc2 = f2(dc.y, fsqrt(fmaf(h3.x - h2.x, h3.x - h2.x, (h3.y - h2.y) * (h3.y - h2.y))));
    if (!fit_triplet(P, h1, h2, h3, circle_radius_d(h1, h2, h3, dc2), dc2, T2)) { o.status = 4; return o; }
    o.kappa2 = T2.q * T2.khat;
    o.var2 = rcp(T2.A);
    // Eq. 8 weighted mean, Eq. 7 global chi2
    const float w1 = T1.A, w2 = T2.A;
    const float kb = (o.kappa1 * w1 + o.kappa2 * w2) * rcp(w1 + w2);
    o.kappa = kb;
    o.chi2 = triplet_chi2(T1, kb) + triplet_chi2(T2, kb);
    if (!(o.chi2 < P.chi2_max)) { o.status = 5; return o; }
    // track parameters: polar angle of arc 01 at |kappa-bar|, transverse circle (R11)
    const float k = fabsf(kb);
    const int q = kb > 0.0f ? 1 : -1;
    const float dx = h1.x - h0.x, dy = h1.y - h0.y, z01 = h1.z - h0.z;
    const float d01 = dc.x;
    float phi01;
    if (!arc_phi<M3E_NEWTON_IT_FINAL>(d01, z01, k, T1.phc[0] + T1.dphi[0] * (k - T1.kc[0]), phi01)) {
        o.status = 6;
        return o;
    }
    const float cth = fminf(fmaxf(z01 * k * rcp(phi01), -1.0f), 1.0f);
    const float rt = fsqrt(1.0f - cth * cth) * rcp(k);
    const float off = fsqrt(fmaxf(0.0f, rt * rt - 0.25f * d01 * d01));
    const float id01 = rcp(d01);
    const float ux = dx * id01, uy = dy * id01;
    o.cth01 = cth;
    o.cx = 0.5f * (h0.x + h1.x) + q * off * uy;   // clockwise: centre right of the chord
    o.cy = 0.5f * (h0.y + h1.y) - q * off * ux;
    return o;
}

template <bool kPairs = true>
M3E_HD FitOut fit_candidate_h(const DevParams& P, const Frame& F, float3 h0, float3 h1, float3 h2, float rtc) {
    return fit_candidate_hd<kPairs>(P, F, h0, h1, h2, rtc, chords(h0, h1, h2));
}

template <bool kPairs = true>
M3E_HD FitOut fit_candidate(const DevParams& P, const Frame& F, int i0, int i1, int i2, float rtc) {
    return fit_candidate_h<kPairs>(P, F, hit(F, 0, i0), hit(F, 1, i1), hit(F, 2, i2), rtc);
}

// ------------------------------------------------------------- Vertex Fit ----
// fp64, Sec. IV-C + Alg. 4 phase 2 for one (e+, e+, e-) triple (R12-R16).
// Per track only what phase 2 reads (the energy test of phase 1 is elsewhere).
struct VTrk {
    int q;
    double cx, cy, rt;           // transverse circle (R11)
    double h0x, h0y, h0z;        // layer-0 hit
    double cthk;                 // cos(theta) / k: dz per radian of turning (Eq. 11)
    double sms;                  // sigma_MS at the track's momentum (Highland, R7)
    double pz;                   // p cos(theta)
};

__device__ __forceinline__ VTrk make_vtrk(const DevParams& P, const m3e_track& t, const Frame& F) {
    VTrk v;
    v.q = t.kappa > 0.0f ? 1 : -1;
    const double k = fabs((double)t.kappa);
    const double cth = (double)t.cos_theta01;
    const double ik = 1.0 / k;
    v.cx = (double)t.cx;
    v.cy = (double)t.cy;
    v.rt = sqrt(fmax(0.0, 1.0 - cth * cth)) * ik;
    const int g = F.s[0] + t.hit[0];
    v.h0x = (double)F.x[g];
    v.h0y = (double)F.y[g];
    v.h0z = (double)F.z[g];
    v.cthk = cth * ik;
    v.sms = P.chl_d * k;   // Highland at p (R7)
    v.pz = P.ptb * ik * cth;
    return v;
}

// circle-circle intersections; 0 or 2 points {x0,y0,x1,y1}
__device__ __forceinline__ int intersect(const VTrk& A, const VTrk& B, double o[4]) {
    const double dx = B.cx - A.cx, dy = B.cy - A.cy, D = sqrt(dx * dx + dy * dy);
    if (D == 0.0 || D > A.rt + B.rt || D < fabs(A.rt - B.rt)) return 0;
    const double iD = 1.0 / D;
    const double a = (A.rt * A.rt - B.rt * B.rt + D * D) * (0.5 * iD);
    const double h = sqrt(fmax(0.0, A.rt * A.rt - a * a));
    const double ux = dx * iD, uy = dy * iD;
    o[0] = A.cx + a * ux - h * uy; o[1] = A.cy + a * uy + h * ux;
    o[2] = A.cx + a * ux + h * uy; o[3] = A.cy + a * uy - h * ux;
    return 2;
}

__device__ __forceinline__ double seg_dist(double px, double py, double ax, double ay, double bx, double by) {
    const double vx = bx - ax, vy = by - ay;
    double t = ((px - ax) * vx + (py - ay) * vy) / (vx * vx + vy * vy);
    t = fmin(fmax(t, 0.0), 1.0);
    const double ex = px - ax - t * vx, ey = py - ay - t * vy;
    return sqrt(ex * ex + ey * ey);
}

// distance to the double hollow-cone target surface (R14)
__device__ __forceinline__ double target_distance(const DevParams& P, double x, double y, double z) {
    const double rho = sqrt(x * x + y * y), R = P.target_r, L = P.target_half;
    return fmin(seg_dist(rho, z, 0.0, -L, R, 0.0), seg_dist(rho, z, R, 0.0, 0.0, L));
}

struct VResult {
    int found;                   // some intersection choice produced a vertex
    int pass;
    double x, y, z, chi2, tdist, ptot;
};

// intersections of one track pair within target_r + xy_margin (Sec. IV-C), slot 0
// first; n = 0: the pair does not intersect or no intersection is near the target
struct PairPts {
    double x0, y0, x1, y1, iw0, iw1;   // points, inverse Eq. 10 variances (R13)
    int n;
};

// signed turning angle (R12) from the direction (bx, by) out of the track circle's
// centre to the layer-0 hit, in the direction of motion, in (-pi, pi]: one atan2 of
// the cross and dot products of the two radii (scale-free in (bx, by))
// out of line: one copy of the fp64 atan2 instead of nine inlined ones keeps the
// vertex kernels' code in the instruction cache (triple kernel 0.44 -> 0.36 ms)
static __device__ __noinline__ double turn_atan2(double y, double x) { return atan2(y, x); }
__device__ __forceinline__ double turn_to_h0(const VTrk& t, double bx, double by) {
    const double ax = t.h0x - t.cx, ay = t.h0y - t.cy;
    return t.q * turn_atan2(ax * by - ay * bx, ax * bx + ay * by);
}

// Eq. 10 (R13) inverse variance of an intersection point of tracks A and B
__device__ __forceinline__ double point_iw(const DevParams& P, const VTrk& A, const VTrk& B, double px, double py) {
    const double sa = A.rt * fabs(turn_to_h0(A, px - A.cx, py - A.cy));
    const double sb = B.rt * fabs(turn_to_h0(B, px - B.cx, py - B.cy));
    return 1.0 / (0.5 * (A.sms * A.sms * sa * sa + B.sms * B.sms * sb * sb) + P.sig_pix2);
}

__device__ __forceinline__ void pair_points(const DevParams& P, const VTrk& A, const VTrk& B, PairPts& o) {
    o.n = 0;
    const double dx = B.cx - A.cx, dy = B.cy - A.cy, D = sqrt(dx * dx + dy * dy);
    if (D == 0.0 || D > A.rt + B.rt || D < fabs(A.rt - B.rt)) return;   // "the track triplet is skipped"
    const double iD = 1.0 / D;
    const double a = (A.rt * A.rt - B.rt * B.rt + D * D) * (0.5 * iD);
    const double h = sqrt(fmax(0.0, A.rt * A.rt - a * a));
    const double ux = dx * iD, uy = dy * iD;
    const double ax0 = A.cx + a * ux - h * uy, ay0 = A.cy + a * uy + h * ux;
    const double ax1 = A.cx + a * ux + h * uy, ay1 = A.cy + a * uy - h * ux;
    const bool k0 = sqrt(ax0 * ax0 + ay0 * ay0) <= P.rlim, k1 = sqrt(ax1 * ax1 + ay1 * ay1) <= P.rlim;
    o.x0 = k0 ? ax0 : ax1;
    o.y0 = k0 ? ay0 : ay1;
    o.x1 = ax1;
    o.y1 = ay1;
    o.n = (int)k0 + (int)k1;
    // Eq. 10 of each kept point, once (the choice loop combines them up to 2^3 ways);
    // the second point is rarely near the target
    o.iw0 = o.n ? point_iw(P, A, B, o.x0, o.y0) : 0.0;
    o.iw1 = o.n == 2 ? point_iw(P, A, B, o.x1, o.y1) : 0.0;
}

// Alg. 4 phase 2 for one (e+, e+, e-) triple, inline: every array a named
// register (choices selected by value), so that a kernel running one triple per
// thread keeps it out of local memory
__device__ __forceinline__ VResult vertex_triple_inl(const DevParams& P, const VTrk& T0, const VTrk& T1,
                                                     const VTrk& T2) {
    VResult best;
    best.found = 0; best.pass = 0;
    best.x = best.y = best.z = best.tdist = best.ptot = 0.0;
    best.chi2 = 1e300;
    PairPts Q0, Q1, Q2;   // pairs (0,1), (0,2), (1,2)
    pair_points(P, T0, T1, Q0);
    if (Q0.n == 0) return best;
    pair_points(P, T0, T2, Q1);
    if (Q1.n == 0) return best;
    pair_points(P, T1, T2, Q2);
    if (Q2.n == 0) return best;
#pragma unroll 1
    for (int c = 0; c < 8; ++c) {   // (s0, s1, s2) in the oracle's nested order, s2 fastest
        const int s0 = c >> 2, s1 = (c >> 1) & 1, s2 = c & 1;
        if (s0 >= Q0.n || s1 >= Q1.n || s2 >= Q2.n) continue;
        const double p0x = s0 ? Q0.x1 : Q0.x0, p0y = s0 ? Q0.y1 : Q0.y0, w0 = s0 ? Q0.iw1 : Q0.iw0;
        const double p1x = s1 ? Q1.x1 : Q1.x0, p1y = s1 ? Q1.y1 : Q1.y0, w1 = s1 ? Q1.iw1 : Q1.iw0;
        const double p2x = s2 ? Q2.x1 : Q2.x0, p2y = s2 ? Q2.y1 : Q2.y0, w2 = s2 ? Q2.iw1 : Q2.iw0;
        // Eq. 9: weighted mean of the three points
        const double iws = 1.0 / (w0 + w1 + w2);
        const double mx = (p0x * w0 + p1x * w1 + p2x * w2) * iws, my = (p0y * w0 + p1y * w1 + p2y * w2) * iws;
        double pcx[3], pcy[3], pcz[3], isg[3], mz = 0.0, wz = 0.0;
        bool bad = false;
#pragma unroll
        for (int t = 0; t < 3; ++t) {   // Fig. 6, Eq. 11: point of closest approach to (mx, my)
            const VTrk& A = t == 0 ? T0 : (t == 1 ? T1 : T2);
            const double dx = mx - A.cx, dy = my - A.cy, dn = sqrt(dx * dx + dy * dy);
            bad |= dn == 0.0;
            const double s = A.rt / dn;
            pcx[t] = A.cx + dx * s;
            pcy[t] = A.cy + dy * s;
            const double dphi = turn_to_h0(A, dx, dy);
            pcz[t] = A.h0z - dphi * A.cthk;
            const double sv = A.rt * fabs(dphi);
            isg[t] = 1.0 / (A.sms * A.sms * sv * sv + P.sig_pix2);
            mz += pcz[t] * isg[t];
            wz += isg[t];
        }
        if (bad) continue;
        mz /= wz;
        double chi = 0.0;   // Eq. 12 (R15)
#pragma unroll
        for (int t = 0; t < 3; ++t) {
            const double ex = pcx[t] - mx, ey = pcy[t] - my, ez = pcz[t] - mz;
            chi += (ex * ex + ey * ey + ez * ez) * isg[t];
        }
        if (chi < best.chi2) {
            best.found = 1;
            best.chi2 = chi;
            best.x = mx; best.y = my; best.z = mz;
            // momentum at the pca: p_t q (sin ph, -cos ph), ph the angle of pca - c, with
            // p_t = p sin(theta) = ptb rt (R11: rt = sin(theta) / k) and (cos ph, sin ph) =
            // (pca - c) / rt: q ptb (pcy - cy, cx - pcx)
            double px = 0.0, py = 0.0, pz = 0.0;
#pragma unroll
            for (int t = 0; t < 3; ++t) {
                const VTrk& A = t == 0 ? T0 : (t == 1 ? T1 : T2);
                const double f = A.q * P.ptb;
                px += f * (pcy[t] - A.cy);
                py -= f * (pcx[t] - A.cx);
                pz += A.pz;
            }
            best.ptot = sqrt(px * px + py * py + pz * pz);
        }
    }
    if (best.found) {
        best.tdist = target_distance(P, best.x, best.y, best.z);
        best.pass = best.chi2 <= P.chi2v_max && best.tdist <= P.tdist_max && best.ptot <= P.ptot_max;
    }
    return best;
}

}  // namespace m3e
