// m3e_kernels.cu -- the persistent filter kernel of the Mu3e online event selection.
//
// One CTA (256 threads, 8 warps) processes a batch of consecutive frames at a
// time (Alg. 1 "Distribute frames over CUDA blocks", re-blocked for
// B200: a batch instead of one frame, so the fit stage runs one lane per
// candidate over the whole batch instead of one thread per candidate of one
// frame).  Per batch:
//   load   the batch's offsets and hits (SoA x/y/z) into shared memory with
//          cp.async.bulk (TMA bulk copies) completing on an mbarrier,
//          double-buffered: the next batch's copies are in flight while this
//          batch computes;
//   S      Selection Cuts, one warp per frame, ballot/popc compaction (Alg. 2);
//   F      triplet fit + layer-3 extension, one lane per candidate (Alg. 3);
//   T      per-frame track compaction (ballot/popc), charge split;
//   V      vertex selection in fp64, one warp per frame with e+e+e- (Alg. 4);
//   O      decoupled look-back prefix over (tracks, kept frames, kept hits) so
//          every output is written in frame order; the packer copies the kept
//          frames' hits (Sec. V-A), tracks and vertices out.
// Batches are handed out by an atomic ticket, so the look-back only ever waits
// on batches held by running CTAs.  The same kernel with a compile-time MODE
// runs one stage on fixed per-frame slots (stage-isolated parity tests).
#include <cstdint>
#include <cuda_runtime.h>

#include "m3e_device.cuh"
#include "m3e_kernels.h"

namespace m3e {

// ------------------------------------------------------------ PTX helpers ----
__device__ __forceinline__ uint32_t smem_u32(const void* p) {
    return static_cast<uint32_t>(__cvta_generic_to_shared(p));
}
__device__ __forceinline__ void mbar_init(uint64_t* bar, uint32_t count) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(bar)), "r"(count) : "memory");
}
__device__ __forceinline__ void mbar_arrive_expect_tx(uint64_t* bar, uint32_t bytes) {
    asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(bar)), "r"(bytes)
                 : "memory");
}
__device__ __forceinline__ void mbar_wait(uint64_t* bar, uint32_t parity) {
    asm volatile(
        "{\n"
        ".reg .pred p;\n"
        "WAIT_%=:\n"
        "mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n"
        "@!p bra WAIT_%=;\n"
        "}\n" ::"r"(smem_u32(bar)),
        "r"(parity)
        : "memory");
}
// TMA bulk copy global -> shared, completion counted on the mbarrier (SASS UBLKCP)
__device__ __forceinline__ void bulk_g2s(void* dst, const void* src, uint32_t bytes, uint64_t* bar) {
    asm volatile(
        "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(
            smem_u32(dst)),
        "l"(src), "r"(bytes), "r"(smem_u32(bar))
        : "memory");
}
__device__ __forceinline__ void fence_proxy_async() { asm volatile("fence.proxy.async.shared::cta;" ::: "memory"); }
__device__ __forceinline__ void fence_mbar_init() {
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
}
__device__ __forceinline__ void st_volatile_v4(uint4* p, uint4 v) {
    asm volatile("st.volatile.global.v4.u32 [%0], {%1, %2, %3, %4};" ::"l"(p), "r"(v.x), "r"(v.y), "r"(v.z),
                 "r"(v.w)
                 : "memory");
}
__device__ __forceinline__ uint4 ld_volatile_v4(const uint4* p) {
    uint4 v;
    asm volatile("ld.volatile.global.v4.u32 {%0, %1, %2, %3}, [%4];"
                 : "=r"(v.x), "=r"(v.y), "=r"(v.z), "=r"(v.w)
                 : "l"(p)
                 : "memory");
    return v;
}
__device__ __forceinline__ uint32_t warp_sum(uint32_t v) {
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
    return v;
}

// ----------------------------------------------------------- shared state ----
// per-frame results of one batch; two copies, because a batch's outputs are
// written only after the CTA has computed its next batch (deferred look-back)
struct BatchState {
    int nstored[kFB], ncand[kFB], ntrk[kFB], nneg[kFB], ncomb[kFB], reason[kFB];
    uint32_t o_trk[kFB + 1], o_kept[kFB + 1], o_hits[kFB + 1];   // exclusive prefixes (+ total)
    uint32_t offs[4 * kFB + 4];                                // the batch's offsets (packer)
    m3e_vertex vtx[kFB];
    uint32_t batch;
    int nf;
};

struct Smem {
    float hx[2][kHCap];
    float hy[2][kHCap];
    float hz[2][kHCap];
    uint32_t offs[2][4 * kFB + 4];
    uint64_t bar[2];
    uint32_t b_batch[2], b_winlo[2], b_winhi[2];
    BatchState st[2];
    uint32_t pref[kFB + 1];                                   // candidates: exclusive prefix
    uint32_t g_trk, g_kept, g_hits;                            // finalized batch's global bases
    uint8_t vlist[kWarps][2][kMaxTracksCap];
    uint32_t vcomb[kWarps][kMaxCombsCap];
    unsigned long long s_kept[6], s_cand, s_trk, s_hits, s_vtx, s_frames;
    int s_overflow;
    DevParams P;   // copy for the out-of-line vertex routine (no address of a kernel parameter is taken)
};

size_t smem_bytes() { return sizeof(Smem); }

// view of frame j of the batch in buffer `buf`
__device__ __forceinline__ Frame frame_view(const KArgs& A, const Smem& S, int buf, int j) {
    Frame F;
    const uint32_t* o = S.offs[buf] + 4 * j;
    const uint32_t g = o[0];
#pragma unroll
    for (int l = 0; l < 4; ++l) {
        F.s[l] = (int)(o[l] - g);
        F.n[l] = (int)(o[l + 1] - o[l]);
    }
    const bool inwin = g >= S.b_winlo[buf] && o[4] <= S.b_winhi[buf];
    if (inwin) {
        const uint32_t d = g - S.b_winlo[buf];
        F.x = S.hx[buf] + d;
        F.y = S.hy[buf] + d;
        F.z = S.hz[buf] + d;
    } else {  // batch larger than the staging window: read this frame from HBM
        F.x = A.x + g;
        F.y = A.y + g;
        F.z = A.z + g;
    }
    return F;
}

// thread 0: claim batch b into buffer buf and start its bulk copies
__device__ __forceinline__ void issue_load(const KArgs& A, Smem& S, int buf, uint32_t b) {
    S.b_batch[buf] = b;
    if (b >= A.nbatch) return;
    const uint32_t f0 = b * (uint32_t)A.fb;
    const uint32_t nf = min(A.F - f0, (uint32_t)A.fb);
    const uint32_t lo = A.offsets[4 * f0], hi = A.offsets[4 * (f0 + nf)];
    const uint32_t wlo = lo & ~3u;
    const uint32_t whi = min((hi + 3u) & ~3u, wlo + (uint32_t)kHCap);
    S.b_winlo[buf] = wlo;
    S.b_winhi[buf] = whi;
    S.offs[buf][4 * nf] = hi;
    const uint32_t hb = (whi - wlo) * 4u, ob = nf * 16u;
    fence_proxy_async();
    mbar_arrive_expect_tx(&S.bar[buf], 3u * hb + ob);
    bulk_g2s(S.offs[buf], A.offsets + 4 * (size_t)f0, ob, &S.bar[buf]);
    if (hb) {
        bulk_g2s(S.hx[buf], A.x + wlo, hb, &S.bar[buf]);
        bulk_g2s(S.hy[buf], A.y + wlo, hb, &S.bar[buf]);
        bulk_g2s(S.hz[buf], A.z + wlo, hb, &S.bar[buf]);
    }
}

// exclusive scan of v[0..n) (n <= 64) in place by one warp, v[n] = total
__device__ __forceinline__ void warp_scan64(uint32_t* v, int n) {
    const int lane = threadIdx.x & 31;
    const uint32_t a = (2 * lane < n) ? v[2 * lane] : 0u;
    const uint32_t b = (2 * lane + 1 < n) ? v[2 * lane + 1] : 0u;
    const uint32_t s = a + b;
    uint32_t inc = s;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
        const uint32_t t = __shfl_up_sync(0xffffffffu, inc, o);
        if (lane >= o) inc += t;
    }
    const uint32_t ex = inc - s;
    const uint32_t tot = __shfl_sync(0xffffffffu, inc, 31);
    __syncwarp();
    if (2 * lane < n) v[2 * lane] = ex;
    if (2 * lane + 1 < n) v[2 * lane + 1] = ex + a;
    if (lane == 0) v[n] = tot;
    __syncwarp();
}

// largest j in [0, n) with pref[j] <= e (pref non-decreasing, pref[0] = 0)
__device__ __forceinline__ int find_frame(const uint32_t* pref, int n, uint32_t e) {
    int lo = 0, hi = n - 1;
    while (lo < hi) {
        const int mid = (lo + hi + 1) >> 1;
        if (pref[mid] <= e) lo = mid; else hi = mid - 1;
    }
    return lo;
}

__device__ __forceinline__ double track_energy(const DevParams& P, float kappa) {
    const double p = P.ptb / fabs((double)kappa);
    return sqrt(p * p + kEMass * kEMass);
}

// Decoupled look-back (warp 0).  Status word of batch b = {epoch<<2 | state,
// tracks, kept frames, kept hits}; state 1 = aggregate, 2 = inclusive prefix.
// publish_aggregate() runs as soon as the batch's counts are known; resolve()
// runs one batch later (deferred), so the predecessors have normally published.
__device__ __forceinline__ void publish_aggregate(const KArgs& A, uint32_t b, uint3 agg) {
    const uint32_t tag = (A.epoch << 2) | (b == 0 ? 2u : 1u);
    if ((threadIdx.x & 31) == 0) st_volatile_v4(A.status + b, make_uint4(tag, agg.x, agg.y, agg.z));
}

__device__ __forceinline__ uint3 resolve(const KArgs& A, uint32_t b, uint3 agg) {
    const int lane = threadIdx.x & 31;
    const uint32_t tagA = (A.epoch << 2) | 1u, tagI = (A.epoch << 2) | 2u;
    uint3 ex = make_uint3(0, 0, 0);
    if (b == 0) return ex;
    int j = (int)b - 1;
    for (;;) {
        const int idx = j - lane;
        uint4 st;
        if (idx >= 0) {
            do {
                st = ld_volatile_v4(A.status + idx);
            } while (st.x != tagA && st.x != tagI);
        } else {
            st = make_uint4(tagI, 0u, 0u, 0u);  // virtual inclusive zero before batch 0
        }
        const unsigned m = __ballot_sync(0xffffffffu, st.x == tagI);
        const int k = m ? __ffs(m) - 1 : 32;  // nearest predecessor with an inclusive prefix
        const bool use = lane <= k;
        ex.x += warp_sum(use ? st.y : 0u);
        ex.y += warp_sum(use ? st.z : 0u);
        ex.z += warp_sum(use ? st.w : 0u);
        if (m) break;
        j -= 32;
    }
    if (lane == 0) st_volatile_v4(A.status + b, make_uint4(tagI, ex.x + agg.x, ex.y + agg.y, ex.z + agg.z));
    return ex;
}

// Write the outputs of a batch whose counts and prefixes are in B (all threads):
// per-frame records, the packed kept frames (Sec. V-A), vertices and tracks.
template <int MODE>
__device__ __forceinline__ void finalize_batch(const KArgs& A, Smem& S, const BatchState& B,
                                               const m3e_track* trk) {
    const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
    const int nf = B.nf;
    const uint32_t f0 = B.batch * (uint32_t)A.fb;
    if (warp == 0) {
        const uint3 ex = resolve(A, B.batch, make_uint3(B.o_trk[nf], B.o_kept[nf], B.o_hits[nf]));
        if (lane == 0) {
            S.g_trk = ex.x;
            S.g_kept = ex.y;
            S.g_hits = ex.z;
        }
    }
    __syncthreads();
    const m3e_outputs& O = A.out;
    const uint32_t g_trk = S.g_trk, g_kept = S.g_kept, g_hits = S.g_hits;
    for (int j = tid; j < nf; j += kThreads) {
        const int r = B.reason[j];
        const bool kept = r != M3E_REASON_NONE;
        const uint32_t kidx = g_kept + B.o_kept[j];
        if (O.reason) O.reason[f0 + j] = (uint8_t)r;
        if (O.frames) {
            m3e_frame_out fo;
            fo.n_cand = (uint16_t)B.ncand[j];
            fo.n_tracks = (uint16_t)B.ntrk[j];
            fo.n_combs = (uint16_t)B.ncomb[j];
            fo.reason = (uint8_t)r;
            fo.n_neg = (uint8_t)min(B.nneg[j], 255);
            fo.track_first = g_trk + B.o_trk[j];
            fo.kept_index = kept ? kidx : 0xFFFFFFFFu;
            O.frames[f0 + j] = fo;
        }
        if (kept) {
            const uint32_t hb = g_hits + B.o_hits[j];
            if (kidx < O.kept_capacity) {
                if (O.kept_frame) O.kept_frame[kidx] = f0 + j;
                if (O.kept_offsets)
                    for (int l = 0; l < 4; ++l)
                        O.kept_offsets[4 * (size_t)kidx + l] = hb + (B.offs[4 * j + l] - B.offs[4 * j]);
                if (O.vertices) {
                    m3e_vertex v;
                    if (r == M3E_REASON_VERTEX) {
                        v = B.vtx[j];
                    } else {
                        v = m3e_vertex{};
                        v.frame = 0xFFFFFFFFu;
                    }
                    O.vertices[kidx] = v;
                }
            } else {
                S.s_overflow = 1;
            }
        }
    }
    if (B.batch == A.nbatch - 1 && tid == 0 && O.kept_offsets) {  // the last batch closes the offsets
        const uint32_t K = g_kept + B.o_kept[nf];
        if (K <= O.kept_capacity) O.kept_offsets[4 * (size_t)K] = g_hits + B.o_hits[nf];
    }
    if constexpr (MODE == kModeFull) {
        const uint32_t nt = B.o_trk[nf];
        if (O.tracks) {
            for (uint32_t e = tid; e < nt; e += kThreads) {
                const int j = find_frame(B.o_trk, nf, e);
                const uint32_t dst = g_trk + e;
                if (dst < O.track_capacity) {
                    const uint4* s4 = reinterpret_cast<const uint4*>(trk + (size_t)j * A.P.max_tracks + (e - B.o_trk[j]));
                    uint4* d4 = reinterpret_cast<uint4*>(O.tracks + dst);
                    d4[0] = s4[0];
                    d4[1] = s4[1];
                } else {
                    S.s_overflow = 1;
                }
            }
        }
    }
    // packer: hits of the kept frames, verbatim, read from HBM (Sec. V-A)
    const uint32_t nh = B.o_hits[nf];
    if (O.kept_x) {
        for (uint32_t e = tid; e < nh; e += kThreads) {
            const int j = find_frame(B.o_hits, nf, e);
            const uint32_t g = B.offs[4 * j] + (e - B.o_hits[j]);
            const uint32_t dst = g_hits + e;
            if (dst < O.kept_hit_capacity) {
                O.kept_x[dst] = A.x[g];
                O.kept_y[dst] = A.y[g];
                O.kept_z[dst] = A.z[g];
            } else {
                S.s_overflow = 1;
            }
        }
    }
    if (tid == 0) {
        S.s_frames += nf;
        S.s_trk += B.o_trk[nf];
        S.s_hits += B.o_hits[nf];
        for (int j = 0; j < nf; ++j) {
            S.s_kept[B.reason[j]] += 1;
            S.s_cand += B.nstored[j];
            S.s_vtx += B.reason[j] == M3E_REASON_VERTEX;
        }
    }
}

// ------------------------------------------------------------------ kernel ----
template <int MODE>
__global__ void __launch_bounds__(kThreads, 2) filter_kernel(const KArgs A) {
    extern __shared__ __align__(16) uint8_t smem_raw[];
    Smem& S = *reinterpret_cast<Smem*>(smem_raw);
    const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
    const unsigned lt_mask = (1u << lane) - 1u;
    const DevParams& P = A.P;
    constexpr bool kOut = MODE == kModeFull || MODE == kModePack;   // ordered outputs

    if (tid == 0) {
        S.P = A.P;
        mbar_init(&S.bar[0], 1);
        mbar_init(&S.bar[1], 1);
        fence_mbar_init();
        for (int i = 0; i < 6; ++i) S.s_kept[i] = 0;
        S.s_cand = S.s_trk = S.s_hits = S.s_vtx = S.s_frames = 0;
        S.s_overflow = 0;
        issue_load(A, S, 0, atomicAdd(A.ticket, 1u));
    }
    __syncthreads();
    int buf = 0, par = 0;
    bool pending = false;   // S.st[par ^ 1] holds a computed batch whose outputs are not written yet
    uint32_t phase0 = 0u, phase1 = 0u;

    // candidate / track slots: per-CTA scratch (FULL; tracks double-buffered by
    // batch parity) or the caller's fixed slots (stage modes)
    uint32_t* cidx;
    float* crt;
    m3e_fit_record* crec;
    m3e_track* ctrk_base;
    if constexpr (MODE == kModeFull) {
        cidx = A.pool_idx + (size_t)blockIdx.x * A.pool_stride;
        crt = A.pool_rt + (size_t)blockIdx.x * A.pool_stride;
        crec = A.pool_rec + (size_t)blockIdx.x * A.pool_stride;
        ctrk_base = A.pool_trk + (size_t)blockIdx.x * 2 * A.trk_stride;
    } else {
        cidx = A.s_cand;
        crt = A.s_rt;
        crec = A.s_rec;
        ctrk_base = A.s_trk;
    }

    for (;;) {
        const uint32_t b = S.b_batch[buf];
        if (b >= A.nbatch) break;
        if (tid == 0) issue_load(A, S, buf ^ 1, atomicAdd(A.ticket, 1u));
        if (buf == 0) { mbar_wait(&S.bar[0], phase0); phase0 ^= 1u; }
        else { mbar_wait(&S.bar[1], phase1); phase1 ^= 1u; }

        BatchState& B = S.st[par];
        const uint32_t f0 = b * (uint32_t)A.fb;
        const int nf = (int)min(A.F - f0, (uint32_t)A.fb);
        const size_t cfirst = MODE == kModeFull ? 0 : (size_t)f0 * P.cuts_max;   // slot of frame 0
        const size_t tfirst = MODE == kModeFull ? 0 : (size_t)f0 * P.max_tracks;
        m3e_track* ctrk = MODE == kModeFull ? ctrk_base + (size_t)par * A.trk_stride : ctrk_base;
        if (tid == 0) {
            B.batch = b;
            B.nf = nf;
        }

        // ---------------------------------------------------- S: Selection Cuts
        if constexpr (MODE == kModeFull || MODE == kModeSelect) {
            for (int j = warp; j < nf; j += kWarps) {
                const Frame Fv = frame_view(A, S, buf, j);
                const bool inval = Fv.n[0] > kMaxLayerHits || Fv.n[1] > kMaxLayerHits ||
                                   Fv.n[2] > kMaxLayerHits || Fv.n[3] > kMaxLayerHits;
                int count = 0;
                if (!inval) {
                    uint32_t* ci = cidx + cfirst + (size_t)j * P.cuts_max;
                    float* cr = crt + cfirst + (size_t)j * P.cuts_max;
                    count = select_frame_warp(P, Fv, [&](int pos, uint32_t packed, float rt) {
                        ci[pos] = packed;
                        cr[pos] = rt;
                    });
                }
                if (lane == 0) {
                    B.ncand[j] = count;
                    const int r = inval ? M3E_REASON_INVALID
                                        : (count > P.cuts_max ? M3E_REASON_TRIPLET_OVERFLOW : M3E_REASON_NONE);
                    B.reason[j] = r;
                    B.nstored[j] = r == M3E_REASON_NONE ? count : 0;
                }
            }
        } else if constexpr (MODE == kModeFit) {
            for (int j = tid; j < nf; j += kThreads) {
                const int n = A.s_ncand[f0 + j];
                B.ncand[j] = n;
                B.reason[j] = n > P.cuts_max ? M3E_REASON_TRIPLET_OVERFLOW : M3E_REASON_NONE;
                B.nstored[j] = n > P.cuts_max ? 0 : n;
            }
        } else if constexpr (MODE == kModeVertex) {
            for (int j = tid; j < nf; j += kThreads) {
                B.ncand[j] = 0;
                B.nstored[j] = 0;
                B.reason[j] = M3E_REASON_NONE;
                B.ntrk[j] = min((int)A.s_ntrk[f0 + j], P.max_tracks);
            }
        } else {  // kModePack
            for (int j = tid; j < nf; j += kThreads) {
                B.ncand[j] = 0;
                B.nstored[j] = 0;
                B.ntrk[j] = 0;
                B.ncomb[j] = 0;
                B.nneg[j] = 0;
                B.reason[j] = A.s_reason[f0 + j];
            }
        }
        __syncthreads();

        if constexpr (MODE == kModeSelect) {
            for (int j = tid; j < nf; j += kThreads) {
                m3e_frame_out fo;
                fo.n_cand = (uint16_t)B.ncand[j];
                fo.n_tracks = 0;
                fo.n_combs = 0;
                fo.reason = (uint8_t)B.reason[j];
                fo.n_neg = 0;
                fo.track_first = (uint32_t)(tfirst + (size_t)j * P.max_tracks);
                fo.kept_index = 0xFFFFFFFFu;
                A.out.frames[f0 + j] = fo;
            }
        }

        // -------------------------------------- F: Triplet fit, one lane per candidate
        if constexpr (MODE == kModeFull || MODE == kModeFit) {
            if (warp == 0) {
                for (int j = lane; j < nf; j += 32) S.pref[j] = (uint32_t)B.nstored[j];
                __syncwarp();
                warp_scan64(S.pref, nf);
            }
            __syncthreads();
            const int total = (int)S.pref[nf];
            for (int e = tid; e < total; e += kThreads) {
                const int j = find_frame(S.pref, nf, (uint32_t)e);
                const size_t slot = cfirst + (size_t)j * P.cuts_max + (e - (int)S.pref[j]);
                const uint32_t pk = cidx[slot];
                const Frame Fv = frame_view(A, S, buf, j);
                const FitOut o = fit_candidate(P, Fv, pk & 1023u, (pk >> 10) & 1023u, (pk >> 20) & 1023u, crt[slot]);
                m3e_fit_record r;
                r.status = (uint8_t)o.status;
                r.pad = 0;
                r.hit3 = o.hit3 < 0 ? (uint16_t)0xFFFF : (uint16_t)o.hit3;
                r.kappa1 = o.kappa1;
                r.kappa2 = o.kappa2;
                r.var1 = o.var1;
                r.var2 = o.var2;
                r.kappa = o.kappa;
                r.chi2 = o.chi2;
                r.cos_theta01 = o.cth01;
                r.cx = o.cx;
                r.cy = o.cy;
                crec[slot] = r;
            }
            __syncthreads();

            // ------------------------- T: per-frame track compaction (ballot / popc)
            for (int j = warp; j < nf; j += kWarps) {
                if (B.reason[j] != M3E_REASON_NONE) {
                    if (lane == 0) { B.ntrk[j] = 0; B.nneg[j] = 0; }
                    continue;
                }
                const int n = B.nstored[j];
                const size_t cb = cfirst + (size_t)j * P.cuts_max;
                m3e_track* tj = ctrk + tfirst + (size_t)j * P.max_tracks;
                int cnt = 0, nneg = 0;
                for (int i0 = 0; i0 < n; i0 += 32) {
                    const int i = i0 + lane;
                    bool acc = false;
                    m3e_fit_record r;
                    if (i < n) {
                        r = crec[cb + i];
                        acc = r.status == 0;
                    }
                    const unsigned m = __ballot_sync(0xffffffffu, acc);
                    const int pos = cnt + __popc(m & lt_mask);
                    const bool store = acc && pos < P.max_tracks;
                    if (store) {
                        const uint32_t pk = cidx[cb + i];
                        m3e_track t;
                        t.frame = f0 + j;
                        t.hit[0] = (uint16_t)(pk & 1023u);
                        t.hit[1] = (uint16_t)((pk >> 10) & 1023u);
                        t.hit[2] = (uint16_t)((pk >> 20) & 1023u);
                        t.hit[3] = r.hit3;
                        t.kappa = r.kappa;
                        t.chi2 = r.chi2;
                        t.cos_theta01 = r.cos_theta01;
                        t.cx = r.cx;
                        t.cy = r.cy;
                        tj[pos] = t;
                    }
                    nneg += __popc(__ballot_sync(0xffffffffu, store && r.kappa < 0.0f));
                    cnt += __popc(m);
                }
                if (lane == 0) {
                    B.ntrk[j] = min(cnt, P.max_tracks + 1);
                    if (cnt > P.max_tracks) {
                        B.reason[j] = M3E_REASON_TRACK_OVERFLOW;
                        B.nneg[j] = 0;
                    } else {
                        B.nneg[j] = nneg;
                    }
                }
            }
            __syncthreads();
        }

        if constexpr (MODE == kModeFit) {
            for (int j = tid; j < nf; j += kThreads) {
                m3e_frame_out fo;
                fo.n_cand = (uint16_t)B.ncand[j];
                fo.n_tracks = (uint16_t)B.ntrk[j];
                fo.n_combs = 0;
                fo.reason = (uint8_t)B.reason[j];
                fo.n_neg = (uint8_t)min(B.nneg[j], 255);
                fo.track_first = (uint32_t)(tfirst + (size_t)j * P.max_tracks);
                fo.kept_index = 0xFFFFFFFFu;
                A.out.frames[f0 + j] = fo;
            }
        }

        // --------------------------------------------- V: vertex selection (fp64)
        if constexpr (MODE == kModeFull || MODE == kModeVertex) {
            for (int j = warp; j < nf; j += kWarps) {
                int ncomb = 0, nneg_out = 0;
                bool has_vtx = false;
                if (B.reason[j] == M3E_REASON_NONE) {
                    const int nt = min(B.ntrk[j], P.max_tracks);
                    const m3e_track* tj = ctrk + tfirst + (size_t)j * P.max_tracks;
                    // charge-sorted index lists, in track order
                    int npos = 0, nneg = 0;
                    for (int i0 = 0; i0 < nt; i0 += 32) {
                        const int i = i0 + lane;
                        const float kap = i < nt ? tj[i].kappa : 0.0f;
                        const bool ispos = i < nt && kap > 0.0f, isneg = i < nt && kap < 0.0f;
                        const unsigned mp = __ballot_sync(0xffffffffu, ispos);
                        const unsigned mn = __ballot_sync(0xffffffffu, isneg);
                        if (ispos) S.vlist[warp][0][npos + __popc(mp & lt_mask)] = (uint8_t)i;
                        if (isneg) S.vlist[warp][1][nneg + __popc(mn & lt_mask)] = (uint8_t)i;
                        npos += __popc(mp);
                        nneg += __popc(mn);
                    }
                    __syncwarp();
                    nneg_out = nneg;
                    if (npos >= 2 && nneg >= 1) {
                        const Frame Fv = frame_view(A, S, buf, j);
                        // Alg. 4 phase 1: energy test over (a < b, e) in row-major order
                        const int tot = npos * npos * nneg;
                        for (int base = 0; base < tot; base += 32) {
                            const int t = base + lane;
                            bool pass = false;
                            uint32_t code = 0;
                            if (t < tot) {
                                const int ia = t / (npos * nneg), rem = t - ia * npos * nneg;
                                const int ib = rem / nneg, ie = rem - ib * nneg;
                                if (ia < ib) {
                                    const int a = S.vlist[warp][0][ia], bb = S.vlist[warp][0][ib],
                                              e = S.vlist[warp][1][ie];
                                    const double dE = track_energy(P, tj[a].kappa) + track_energy(P, tj[bb].kappa) +
                                                      track_energy(P, tj[e].kappa) - kMuMass;
                                    pass = fabs(dE) <= P.e_window;
                                    code = (uint32_t)a | ((uint32_t)bb << 8) | ((uint32_t)e << 16);
                                }
                            }
                            const unsigned m = __ballot_sync(0xffffffffu, pass);
                            const int pos = ncomb + __popc(m & lt_mask);
                            if (pass && pos < P.max_combs) S.vcomb[warp][pos] = code;
                            ncomb += __popc(m);
                            if (ncomb > P.max_combs) break;
                        }
                        __syncwarp();
                        if (ncomb > P.max_combs) {
                            ncomb = P.max_combs + 1;
                        } else {
                            // Alg. 4 phase 2: one lane per stored triple
                            double bchi = 1e300;
                            int bidx = 0x7fffffff;
                            VResult bres;
                            bres.pass = 0;
                            for (int c = lane; c < ncomb; c += 32) {
                                const uint32_t code = S.vcomb[warp][c];
                                VTrk T[3];
                                T[0] = make_vtrk(P, tj[code & 255u], Fv);
                                T[1] = make_vtrk(P, tj[(code >> 8) & 255u], Fv);
                                T[2] = make_vtrk(P, tj[(code >> 16) & 255u], Fv);
                                const VResult r = vertex_triple(&S.P, T);
                                if (r.pass && r.chi2 < bchi) { bchi = r.chi2; bidx = c; bres = r; }
                            }
                            // lowest chi2 among passing triples, earliest on ties
                            double wchi = bchi;
                            int widx = bidx;
#pragma unroll
                            for (int o = 16; o > 0; o >>= 1) {
                                const double oc = __shfl_xor_sync(0xffffffffu, wchi, o);
                                const int oi = __shfl_xor_sync(0xffffffffu, widx, o);
                                if (oc < wchi || (oc == wchi && oi < widx)) { wchi = oc; widx = oi; }
                            }
                            if (widx != 0x7fffffff) {
                                has_vtx = true;
                                if (bidx == widx) {
                                    const uint32_t code = S.vcomb[warp][widx];
                                    m3e_vertex v;
                                    v.frame = f0 + j;
                                    v.track[0] = (uint16_t)(code & 255u);
                                    v.track[1] = (uint16_t)((code >> 8) & 255u);
                                    v.track[2] = (uint16_t)((code >> 16) & 255u);
                                    v.pad = 0;
                                    v.pad2 = 0;
                                    v.x = bres.x; v.y = bres.y; v.z = bres.z;
                                    v.chi2 = bres.chi2;
                                    v.target_dist = (float)bres.tdist;
                                    v.p_total = (float)bres.ptot;
                                    B.vtx[j] = v;
                                }
                            }
                        }
                    }
                    if (lane == 0) {
                        B.ncomb[j] = ncomb;
                        B.nneg[j] = nneg_out;
                        if (ncomb > P.max_combs) B.reason[j] = M3E_REASON_COMB_OVERFLOW;
                        else if (has_vtx) B.reason[j] = M3E_REASON_VERTEX;
                    }
                } else if (lane == 0) {
                    B.ncomb[j] = 0;
                }
                __syncwarp();
            }
            __syncthreads();
        }

        if constexpr (MODE == kModeVertex) {
            for (int j = tid; j < nf; j += kThreads) {
                m3e_frame_out fo;
                fo.n_cand = 0;
                fo.n_tracks = (uint16_t)B.ntrk[j];
                fo.n_combs = (uint16_t)B.ncomb[j];
                fo.reason = (uint8_t)B.reason[j];
                fo.n_neg = (uint8_t)min(B.nneg[j], 255);
                fo.track_first = (uint32_t)(tfirst + (size_t)j * P.max_tracks);
                fo.kept_index = 0xFFFFFFFFu;
                A.out.frames[f0 + j] = fo;
                if (B.reason[j] == M3E_REASON_VERTEX && A.s_vtx) A.s_vtx[f0 + j] = B.vtx[j];
            }
        }

        // ------------------------ O: counts, aggregate now, outputs one batch later
        if constexpr (kOut) {
            for (int j = tid; j < nf; j += kThreads) {
                const int r = B.reason[j];
                const bool kept = r != M3E_REASON_NONE;
                const bool has_tracks = r == M3E_REASON_NONE || r == M3E_REASON_TRACK_OVERFLOW ||
                                        r == M3E_REASON_COMB_OVERFLOW || r == M3E_REASON_VERTEX;
                B.o_trk[j] = (MODE == kModeFull && has_tracks) ? (uint32_t)min(B.ntrk[j], P.max_tracks) : 0u;
                B.o_kept[j] = kept ? 1u : 0u;
                B.o_hits[j] = kept ? (S.offs[buf][4 * j + 4] - S.offs[buf][4 * j]) : 0u;
            }
            for (int i = tid; i <= 4 * nf; i += kThreads) B.offs[i] = S.offs[buf][i];
            __syncthreads();
            if (warp == 0) {
                warp_scan64(B.o_trk, nf);
                warp_scan64(B.o_kept, nf);
                warp_scan64(B.o_hits, nf);
                publish_aggregate(A, b, make_uint3(B.o_trk[nf], B.o_kept[nf], B.o_hits[nf]));
            }
            // the previous batch's predecessors have had a whole batch of time to publish
            if (pending) {
                __syncthreads();
                finalize_batch<MODE>(A, S, S.st[par ^ 1],
                                     MODE == kModeFull ? ctrk_base + (size_t)(par ^ 1) * A.trk_stride : nullptr);
            }
            pending = true;
            par ^= 1;
        }
        __syncthreads();
        buf ^= 1;
    }

    if constexpr (kOut) {
        if (pending) {
            __syncthreads();
            finalize_batch<MODE>(A, S, S.st[par ^ 1],
                                 MODE == kModeFull ? ctrk_base + (size_t)(par ^ 1) * A.trk_stride : nullptr);
        }
        __syncthreads();
        if (tid == 0 && A.out.summary) {
            m3e_summary* sm = A.out.summary;
            atomicAdd((unsigned long long*)&sm->frames, S.s_frames);
            for (int i = 0; i < 6; ++i)
                if (S.s_kept[i]) atomicAdd((unsigned long long*)&sm->kept_by_reason[i], S.s_kept[i]);
            atomicAdd((unsigned long long*)&sm->candidates, S.s_cand);
            atomicAdd((unsigned long long*)&sm->tracks, S.s_trk);
            atomicAdd((unsigned long long*)&sm->kept_hits, S.s_hits);
            atomicAdd((unsigned long long*)&sm->vertices, S.s_vtx);
            if (S.s_overflow) atomicExch((unsigned long long*)&sm->overflow, 1ull);
        }
    }
}

template <int MODE>
static cudaError_t launch_mode(const KArgs& a, int grid, cudaStream_t s) {
    const size_t smem = smem_bytes();
    cudaError_t e = cudaFuncSetAttribute(filter_kernel<MODE>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    if (e != cudaSuccess) return e;
    filter_kernel<MODE><<<grid, kThreads, smem, s>>>(a);
    return cudaGetLastError();
}

cudaError_t launch_filter(int mode, const KArgs& a, int grid, cudaStream_t s) {
    switch (mode) {
        case kModeFull: return launch_mode<kModeFull>(a, grid, s);
        case kModeSelect: return launch_mode<kModeSelect>(a, grid, s);
        case kModeFit: return launch_mode<kModeFit>(a, grid, s);
        case kModeVertex: return launch_mode<kModeVertex>(a, grid, s);
        case kModePack: return launch_mode<kModePack>(a, grid, s);
    }
    return cudaErrorInvalidValue;
}

int blocks_per_sm(int mode) {
    int n = 0;
    const size_t smem = smem_bytes();
    cudaError_t e = cudaErrorInvalidValue;
    switch (mode) {
        case kModeFull:
            cudaFuncSetAttribute(filter_kernel<kModeFull>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
            e = cudaOccupancyMaxActiveBlocksPerMultiprocessor(&n, filter_kernel<kModeFull>, kThreads, smem);
            break;
        default:
            n = 1;
            e = cudaSuccess;
    }
    return e == cudaSuccess && n > 0 ? n : 1;
}

}  // namespace m3e
