// m3e_kernels.cu -- the persistent filter kernel of the Mu3e online event selection.
//
// Every warp is an independent pipeline (no CTA-wide barriers): it claims a
// warp-batch of consecutive frames with an atomic ticket (Alg. 1
// "Distribute frames over CUDA blocks", re-blocked to warps so that uneven
// frames never stall other warps at a barrier) and, per warp-batch:
//   load   offsets + hits (SoA x/y/z) -> shared memory with cp.async.bulk (TMA
//          bulk copies) on the warp's mbarrier, double-buffered: the next
//          warp-batch is in flight while this one computes;
//   S      Selection Cuts per frame (Alg. 2), two-level ballot/popc compaction;
//   F      triplet fit + layer-3 extension (Alg. 3), one lane per candidate
//          across all frames of the warp-batch;
//   T      per-frame track compaction (ballot/popc), charge split;
//   V      vertex selection in fp64 (Alg. 4) for frames with e+ e+ e-;
//   O      per-frame records are written in place; the warp-batch's tracks and
//          kept-frame records are staged at offsets reserved with one atomic
//          per warp-batch, so no warp ever waits for another.
// The pack kernel (second launch) then scans the per-warp-batch counts with a
// decoupled look-back over tiles (all counts final, so it never waits on
// compute) and scatters tracks, vertices and the kept frames' hits into frame
// order (Sec. V-A: kept frames are stored).
// The filter kernel with a compile-time MODE runs one stage on fixed per-frame
// slots (stage-isolated parity tests).
#include <cstdint>
#include <cuda_runtime.h>

#include "m3e_device.cuh"
#include "m3e_kernels.h"

#ifndef M3E_MIN_BLOCKS
#define M3E_MIN_BLOCKS 4   // CTAs per SM the register allocation targets (64 regs: 32 warps/SM)
#endif
#ifndef M3E_NO_FLAT_SELECT
#define M3E_NO_FLAT_SELECT 0   // 1: the selection kernel walks frame by frame (select_frame_warp) only
#endif
#ifndef M3E_MIN_BLOCKS_SEL
#define M3E_MIN_BLOCKS_SEL 4   // same for the selection kernel of the split path
#endif
#ifndef M3E_MIN_BLOCKS_SEL_BIG
#define M3E_MIN_BLOCKS_SEL_BIG 3   // its big-frame variant: 80 registers (the mask walks: 16.5 against 18.2 ms per 1e6
                                   // phase-II frames at 4 CTAs / 64 registers; the row-mask walk before them: 30.3 / 28.4)
#endif

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
__device__ __forceinline__ void prefetch_l2(const void* p) {
    asm volatile("prefetch.global.L2 [%0];" ::"l"(p));
}
__device__ __forceinline__ uint32_t warp_sum(uint32_t v) {
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
    return v;
}

// output track slots: a warp-batch owns bslot[b] consecutive slots of out.tracks
// from tbase[b]; its tracks fill the front, the rest are marked unused
// (frame = 0xFFFFFFFF, every other byte 0)
__device__ __forceinline__ void write_unused_slot(m3e_track* p) {
    uint4* d = reinterpret_cast<uint4*>(p);
    d[0] = make_uint4(0xFFFFFFFFu, 0u, 0u, 0u);
    d[1] = make_uint4(0u, 0u, 0u, 0u);
}
// a frame's first track for the vertex stage: an out.tracks index, or kInFitG |
// a fit_g index (no track output requested, or the caller's capacity exceeded)
constexpr uint32_t kInFitG = 0x80000000u;

__device__ __forceinline__ bool below(uint32_t i, uint32_t lim) { return i < lim; }

// Internal index checks of the check build (-DM3E_CHECK, lib/libm3e_check.so): a
// failed check records its source line (the first one wins) instead of trapping;
// m3e_debug_check() reads and clears it.  Compiled out of the production library.
__device__ unsigned int g_m3e_check_line;
#ifdef M3E_CHECK
#define M3E_CHECK_IDX(cond) \
    do { if (!(cond)) atomicCAS(&g_m3e_check_line, 0u, (unsigned int)__LINE__); } while (0)
#else
#define M3E_CHECK_IDX(cond) do { } while (0)
#endif

// ----------------------------------------------------------- shared state ----
// per-frame results of the warp-batch being processed
struct BatchState {
    int nstored[kFB], ncand[kFB], ntrk[kFB], nneg[kFB], ncomb[kFB], reason[kFB];
    uint32_t o_trk[kFB + 1], o_kept[kFB + 1], o_hits[kFB + 1];   // exclusive prefixes (+ total)
};

// A warp-batch computes for ~10^5 cycles against a ~10^3-cycle bulk-copy latency,
// so one staging buffer per warp suffices; the freed shared memory keeps L1 large
// and holds the warp-batch's candidates instead.
constexpr int kNBuf = 1;
constexpr int kCandSmem = 256;   // candidates of a warp-batch kept in shared memory

// Shared state of select_batch_flat (one warp-batch, frames j < kFB)
struct FlatSel {
    uint4 pl[64];      // Phi_01 pair list {g0 | g1 << 8 | s2 << 16 | j << 24, u bits, n2, 0} (g = staging-window
                       // index); after the walk: per-frame table {list start, store prefix, s0 | s1 << 8 |
                       // s2 << 16, stored}
    uint4 rec[kFB];    // frames with pairs, by rank: {pair prefix, s0 | s1 << 8 | s2 << 16 | j << 24,
                       // n1 | n2 << 8, 1/n1 bits}
    int cnt[kFB];      // Selection-Cut survivors per frame
};

// Cold vertex-stage scratch of one warp, in global memory (L1/L2 resident;
// touched for ~1.5% of frames), so that it does not cost shared memory.
struct VScratch {
    m3e_vertex vtx[32];   // by frame lane: kFB frames of a warp-batch
    uint32_t vcomb[kMaxCombsCap];
    uint8_t vlist[2][kMaxTracksCap];
};

// Shared state of select_frame_mask (selection kernel, big-frame calls); it overlays
// the shared-memory candidate array and the other walks' state, so that kernel keeps
// every candidate in global memory.  NW = 64-bit words per mask: frames of up to 64
// (NW = 1) or kMask2Hits (NW = 2) hits in layers 1 and 2
constexpr int kMask2Hits = 96;
template <int NW> struct MaskSel;
template <> struct MaskSel<1> {
    unsigned long long m12[64];   // Phi_12 mask of layer-1 hit i1 over layer 2 (bit i2)
    unsigned long long pm[65];    // layer 2 in z order: pm[r] = the hits of z-rank < r
    float zs[64];                 // layer-2 z, ascending
    uint8_t ord[64];              // layer-2 hit of z-rank r
    uint2 pl[64];                 // Phi_01 pair list {i0 | i1 << 10, u(i0, i1)}
};
template <> struct MaskSel<2> {   // (m12: the warp's global scratch, L1 / L2)
    unsigned long long pm[kMask2Hits + 1][2];
    float zs[kMask2Hits];
    uint8_t ord[kMask2Hits];
    uint2 pl[64];
};

struct __align__(16) WarpSmem {
    float hx[kNBuf][kHCap];
    float hy[kNBuf][kHCap];
    float hz[kNBuf][kHCap];
    uint32_t offs[kNBuf][4 * kFB + 4];
    uint64_t bar[kNBuf];
    uint32_t b_batch[kNBuf], b_winlo[kNBuf], b_winhi[kNBuf];
    union {
        struct {
            uint32_t cidx[kCandSmem];        // candidates (flat warp-batch index < kCandSmem)
            union {
                struct {                     // per-frame selection (select_frame_warp) and the fused stages
                    float crt[kCandSmem];
                    uint2 pl[64];            // Phi_01 pair list: {i0 | i1 << 10, u(i0, i1)}
                };
                FlatSel fl;                  // warp-batch-flat selection (select_batch_flat)
            };
        };
        MaskSel<1> ms1;                      // mask-factorised big-frame selection (select_frame_mask)
        MaskSel<2> ms2;
    };
    BatchState st;
    uint32_t pref[kFB + 1];          // candidates: exclusive prefix
    int npos[kFB];                   // stored positive tracks per frame (vertex gate)
    uint32_t q[64];                  // Delta-lambda + Phi_12 survivors (selection FIFO)
    uint32_t acc[12];                // run summary: kept_by_reason[6], cand, frames, tracks, hits, overflow
};

// the mask walks' state fits the space of the candidate array and the other walks'
static_assert(sizeof(MaskSel<1>) <= kCandSmem * 4 + kCandSmem * 4 + 64 * 8 &&
                  sizeof(MaskSel<2>) <= kCandSmem * 4 + kCandSmem * 4 + 64 * 8,
              "mask-walk state larger than the space it overlays");

struct Smem {
    WarpSmem w[kWarps];
    DevParams P;   // copy for the out-of-line vertex routine (no address of a kernel parameter is taken)
};

size_t smem_bytes() { return sizeof(Smem); }

// view of frame j of the warp-batch in buffer `buf`
__device__ __forceinline__ Frame frame_view(const KArgs& A, const WarpSmem& W, int buf, int j) {
    Frame F;
    const uint32_t* o = W.offs[buf] + 4 * j;
    const uint32_t g = o[0];
#pragma unroll
    for (int l = 0; l < 4; ++l) {
        F.s[l] = (int)(o[l] - g);
        F.n[l] = (int)(o[l + 1] - o[l]);
    }
    const bool inwin = g >= W.b_winlo[buf] && o[4] <= W.b_winhi[buf];
    if (inwin) {
        const uint32_t d = g - W.b_winlo[buf];
        F.x = W.hx[buf] + d;
        F.y = W.hy[buf] + d;
        F.z = W.hz[buf] + d;
    } else {  // warp-batch larger than the staging window: read this frame from HBM
        F.x = A.x + g;
        F.y = A.y + g;
        F.z = A.z + g;
    }
    return F;
}

__device__ __forceinline__ void prefetch_bulk_l2(const void* p, uint32_t bytes) {
    asm volatile("cp.async.bulk.prefetch.L2.global [%0], %1;" ::"l"(p), "r"(bytes) : "memory");
}
// lane 0: claim warp-batch b into buffer buf and start its bulk copies
// next warp-batch of this launch (>= nbatch: none left); the split path's fused
// launch only takes the warp-batches the selection kernel could not store
__device__ __forceinline__ uint32_t claim_batch(const KArgs& A) {
    const uint32_t t = atomicAdd(A.bticket, 1u);
    if (!A.spill_list) return t;
    return t < *reinterpret_cast<volatile const uint32_t*>(A.ticket + 5) ? A.spill_list[t] : A.nbatch;
}

// (lo, hi) = the warp-batch's first and end hit, offsets[4 f0] and offsets[4 (f0 + nf)]
__device__ __forceinline__ void issue_load_w(const KArgs& A, WarpSmem& W, int buf, uint32_t b, uint32_t lo,
                                             uint32_t hi) {
    W.b_batch[buf] = b;
    if (b >= A.nbatch) return;
    const uint32_t f0 = b * (uint32_t)A.fb;
    const uint32_t nf = min(A.F - f0, (uint32_t)A.fb);
    const uint32_t wlo = lo & ~3u;
    const uint32_t whi = min((hi + 3u) & ~3u, wlo + (uint32_t)kHCap);
    W.b_winlo[buf] = wlo;
    W.b_winhi[buf] = whi;
    W.offs[buf][4 * nf] = hi;
    const uint32_t hb = (whi - wlo) * 4u, ob = nf * 16u;
    fence_proxy_async();
    mbar_arrive_expect_tx(&W.bar[buf], 3u * hb + ob);
    bulk_g2s(W.offs[buf], A.offsets + 4 * (size_t)f0, ob, &W.bar[buf]);
    if (hb) {
        bulk_g2s(W.hx[buf], A.x + wlo, hb, &W.bar[buf]);
        bulk_g2s(W.hy[buf], A.y + wlo, hb, &W.bar[buf]);
        bulk_g2s(W.hz[buf], A.z + wlo, hb, &W.bar[buf]);
    }
}
__device__ __forceinline__ void issue_load(const KArgs& A, WarpSmem& W, int buf, uint32_t b) {
    uint32_t lo = 0u, hi = 0u;
    if (b < A.nbatch) {
        const uint32_t f0 = b * (uint32_t)A.fb;
        const uint32_t nf = min(A.F - f0, (uint32_t)A.fb);
        lo = A.offsets[4 * f0];
        hi = A.offsets[4 * (f0 + nf)];
    }
    issue_load_w(A, W, buf, b, lo, hi);
}
// window bounds of warp-batch b (lane 0; loads left in flight until used)
__device__ __forceinline__ void batch_bounds(const KArgs& A, uint32_t b, uint32_t& lo, uint32_t& hi) {
    if (b < A.nbatch) {
        const uint32_t f0 = b * (uint32_t)A.fb;
        const uint32_t nf = min(A.F - f0, (uint32_t)A.fb);
        lo = A.offsets[4 * f0];
        hi = A.offsets[4 * (f0 + nf)];
    }
}

// exclusive scan of v[0..n) (n <= 32) in place by the warp, v[n] = total
__device__ __forceinline__ void warp_scan(uint32_t* v, int n) {
    const int lane = threadIdx.x & 31;
    const uint32_t a = lane < n ? v[lane] : 0u;
    uint32_t inc = a;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
        const uint32_t t = __shfl_up_sync(0xffffffffu, inc, o);
        if (lane >= o) inc += t;
    }
    const uint32_t tot = __shfl_sync(0xffffffffu, inc, 31);
    __syncwarp();
    if (lane < n) v[lane] = inc - a;
    if (lane == 0) v[n] = tot;
    __syncwarp();
}

// inclusive warp prefix sum
__device__ __forceinline__ uint32_t warp_incl(uint32_t v) {
    const int lane = threadIdx.x & 31;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
        const uint32_t t = __shfl_up_sync(0xffffffffu, v, o);
        if (lane >= o) v += t;
    }
    return v;
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

// Decoupled look-back of the pack kernel.  Status word of tile t = {epoch<<2 |
// state, tracks, kept frames, kept hits}; state 1 = aggregate, 2 = inclusive.
__device__ __forceinline__ void publish_aggregate(const KArgs& A, uint32_t t, uint3 agg) {
    const uint32_t tag = (A.epoch << 2) | (t == 0 ? 2u : 1u);
    if ((threadIdx.x & 31) == 0) st_volatile_v4(A.status + t, make_uint4(tag, agg.x, agg.y, agg.z));
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
            st = make_uint4(tagI, 0u, 0u, 0u);  // virtual inclusive zero before warp-batch 0
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

__device__ __forceinline__ uint32_t popc_t(uint32_t v) { return (uint32_t)__popc(v); }
__device__ __forceinline__ uint32_t popc_t(unsigned long long v) { return (uint32_t)__popcll(v); }
__device__ __forceinline__ int ffs_t(uint32_t v) { return __ffs(v); }
__device__ __forceinline__ int ffs_t(unsigned long long v) { return __ffsll(v); }
// combinations per frame up to which the flat walk takes a frame (bounds the walk
// of an overflowing frame); 64-bit masks: phase-II frames (~56 hits per layer)
template <typename MT>
__device__ __forceinline__ constexpr int kMaxFlatCombos() { return sizeof(MT) == 4 ? (int)kBigCombos : 1 << 19; }

// Selection Cuts (Alg. 2, Eq. 2-5) of a whole staged warp-batch (production
// path, SELECT_C), factorised by the hits each cut depends on and walked with
// one lane per ROW of a bit matrix across all frames of the warp-batch:
//   A. one lane per (frame, i0) row: the row's Phi_01 mask over the frame's
//      layer-1 hits (bit i1), a loop over n1 <= 32;
//   B. the set bits, in (frame, i0, i1) order, go to the pair list with the
//      pair's Delta-lambda offset u(i0, i1); one lane per listed pair computes the
//      Delta-lambda + Phi_12 mask over the frame's layer-2 hits (bit i2);
//   C. those set bits, in (frame, i0, i1, i2) order, go to the FIFO; each full 32
//      of it is tested for the r_t window on all lanes, and the survivors are
//      counted per frame (match_any) and capped at cuts_max (R3).
// Bits leave a mask in order through bounded ordered emission (warp prefix of
// popcounts, lower lanes first), so a dense frame never overruns the lists.
// Rows / pairs map to lanes by a ballot search over segment starts (redux.or).
// Compared with one lane per (i0, i1) or (pair, i2) element this drops the
// per-element index arithmetic: ~130 instead of ~300 warp instructions per
// phase-I frame.  Survivor set and order are those of Alg. 2; n_cand =
// min(#survivors, cuts_max + 1), overflow frames store nothing; candidates are
// written to the store at one atomicAdd per warp-batch.
// Eligible warp-batches: all frames inside the staging window, every frame with
// n1, n2 <= 32 and n0 n1 n2 <= kBigCombos (so the walk of an overflowing frame is
// bounded); returns false, having written nothing, for the others (per-frame
// walk).
#ifndef M3E_SEL_FSETP
#define M3E_SEL_FSETP 1   // mask bits from predicates (0: from the sign bits of the differences)
#endif
template <typename MT>   // bit-mask type: uint32_t (layers 1, 2 up to 32 hits) or unsigned long long (64)
__device__ __forceinline__ bool select_batch_flat(const KArgs& A, WarpSmem& W, uint32_t b, uint32_t f0, int nf,
                                                  uint32_t* gl) {
    const DevParams& P = A.P;
    const int lane = threadIdx.x & 31;
    const unsigned lt = (1u << lane) - 1u, le = lt | (1u << lane);
    if (W.offs[0][4 * nf] > W.b_winhi[0]) return false;   // warp-batch larger than the window
    FlatSel& S = W.fl;
    const float* hx = W.hx[0];
    const float* hy = W.hy[0];
    const float* hz = W.hz[0];
    // lane j = frame j: window-relative layer starts and counts
    const bool isf = lane < nf;
    const uint32_t* o = W.offs[0] + 4 * (isf ? lane : 0);
    const uint32_t wlo = W.b_winlo[0];
    const int s0 = (int)(o[0] - wlo), s1 = (int)(o[1] - wlo), s2 = (int)(o[2] - wlo);
    const int n0 = isf ? (int)(o[1] - o[0]) : 0, n1 = (int)(o[2] - o[1]), n2 = (int)(o[3] - o[2]);
    constexpr int kMB = 8 * (int)sizeof(MT);
    if (__any_sync(0xffffffffu, isf && (n1 > kMB || n2 > kMB || n0 * n1 * n2 > kMaxFlatCombos<MT>()))) return false;
    // rows of frames with pairs to test
    const int nr = (n1 > 0 && n2 > 0) ? n0 : 0;
    const uint32_t ra_i = warp_incl((uint32_t)nr);
    const uint32_t NR = __shfl_sync(0xffffffffu, ra_i, 31);
    const unsigned nem = __ballot_sync(0xffffffffu, nr > 0);
    const uint32_t sp = (uint32_t)s0 | ((uint32_t)s1 << 8) | ((uint32_t)s2 << 16);
    if (nr > 0)
        S.rec[__popc(nem & lt)] = make_uint4(ra_i - (uint32_t)nr, sp | ((uint32_t)lane << 24),
                                             (uint32_t)n1 | ((uint32_t)n2 << 8), 0u);
    if (lane < kFB) S.cnt[lane] = 0;
    __syncwarp();
    // segment starts held by lane = rank (no bit for lanes past the last segment)
    const uint32_t RAr = lane < __popc(nem) ? S.rec[lane].x : 0xFFFFFFFFu;

    int pn = 0, qn = 0, L = 0, cb = 0;
    // C. r_t window (on squares, as pass_rtc_sq) for q[0..n); survivors counted per
    // frame and appended to the warp-batch list
    auto drain = [&](int n) {
        const uint32_t pk = W.q[min(lane, n - 1)];
        const int g0 = (int)(pk & 255u), g1 = (int)((pk >> 8) & 255u), g2 = (int)((pk >> 16) & 255u);
        const int j = (int)(pk >> 24);
        const float x1 = hx[g1], y1 = hy[g1];
        const float ax = hx[g0] - x1, ay = hy[g0] - y1, bx = hx[g2] - x1, by = hy[g2] - y1;
        const float cx = bx - ax, cy = by - ay;
        const float cz = ax * by - ay * bx;
        const float num = (ax * ax + ay * ay) * (bx * bx + by * by) * (cx * cx + cy * cy);
        const float den = 4.0f * cz * cz;
        const bool pass = (lane < n) & (cz != 0.0f) & (num >= den * P.rt_min2) & (num <= den * P.rt_max2);
        const unsigned m = __ballot_sync(0xffffffffu, pass);
        const unsigned grp = __match_any_sync(0xffffffffu, j);
        const int cj = S.cnt[j];
        const bool keep = pass && cj + __popc(m & grp & lt) < P.cuts_max;
        const unsigned mk = __ballot_sync(0xffffffffu, keep);
        if (keep) {
            const int idx = L + __popc(mk & lt);
            if (idx < kCandSmem) W.cidx[idx] = pk; else gl[idx] = pk;
        }
        __syncwarp();
        if (lane == __ffs(grp) - 1) S.cnt[j] = cj + __popc(m & grp);
        __syncwarp();
        L += __popc(mk);
    };
    // B + C for the K = pn <= 32 listed pairs: one lane per pair, its mask over
    // layer 2, ordered emission into the FIFO, full 32s drained
    auto expand = [&]() {   // the first K = min(pn, 32) listed pairs
        const int K = min(pn, 32);
        uint4 pe = make_uint4(0u, 0u, 0u, 0u);
        MT rem = 0;
        if (lane < K) {
            pe = S.pl[lane];
            const int g1 = (int)((pe.x >> 8) & 255u), t2 = (int)((pe.x >> 16) & 255u), m2 = (int)pe.z;
            const float x1 = hx[g1], y1 = hy[g1];
            const float u = __uint_as_float(pe.y);
            // four layer-2 hits per iteration, two per packed fp32 operation (same
            // per-hit arithmetic as select_frame_warp: fmaf for Delta-lambda, cos_sep for
            // Phi_12)
            for (int k0 = 0; k0 < m2; k0 += 4) {
#if M3E_SEL_FSETP
                uint32_t nib = 0u;   // pass bits of the four hits k0 .. k0 + 3
#endif
#pragma unroll
                for (int h = 0; h < 4; h += 2) {
                    const int k = k0 + h;
                    const float2 zz = make_float2(hz[t2 + k], hz[t2 + k + 1]);
                    const float2 dl = __ffma2_rn(zz, make_float2(P.inv_dr12, P.inv_dr12), make_float2(-u, -u));
                    const float2 c12 = cos_sep2(x1, y1, make_float2(hx[t2 + k], hx[t2 + k + 1]),
                                                make_float2(hy[t2 + k], hy[t2 + k + 1]), P.inv_r1r2);
                    // |dl| <= dl_max and c12 >= c12_min as signs of exact differences
                    // (a - b is 0 only for a == b and has the sign of a - b: same decisions)
                    const float2 a = __fadd2_rn(c12, make_float2(-P.c12_min, -P.c12_min));
#if M3E_SEL_FSETP
                    // compared on predicates (FSETP), the four bits assembled with constant shifts
                    if (a.x >= 0.0f && fabsf(dl.x) <= P.dl_max) nib |= 1u << h;
                    if (a.y >= 0.0f && fabsf(dl.y) <= P.dl_max) nib |= 2u << h;
#else
                    const float2 b = __fadd2_rn(make_float2(P.dl_max, P.dl_max), make_float2(-fabsf(dl.x), -fabsf(dl.y)));
                    const uint32_t fail = ((__float_as_uint(a.x) | __float_as_uint(b.x)) >> 31) |
                                          (((__float_as_uint(a.y) | __float_as_uint(b.y)) >> 30) & 2u);
                    rem |= (MT)(fail ^ 3u) << k;
#endif
                }
#if M3E_SEL_FSETP
                rem |= (MT)nib << k0;
#endif
            }
            rem &= m2 >= kMB ? ~(MT)0 : ((MT)1 << m2) - 1;   // hits past the frame's layer 2
        }
        __syncwarp();
        {   // drop the K expanded pairs
            const uint4 v = lane < pn - K ? S.pl[K + lane] : make_uint4(0u, 0u, 0u, 0u);
            __syncwarp();
            if (lane < pn - K) S.pl[lane] = v;
            pn -= K;
            __syncwarp();
        }
        // FIFO entry g0 | g1 << 8 | g2 << 16 | j << 24 (the pair's s2 field replaced by g2)
        const uint32_t ebase = pe.x & 0xFF00FFFFu, t2 = (pe.x >> 16) & 255u;
        for (;;) {
            const uint32_t c = popc_t(rem);
            const uint32_t inc = warp_incl(c), exc = inc - c;
            const uint32_t tot = __shfl_sync(0xffffffffu, inc, 31);
            const uint32_t fr = 64u - (uint32_t)qn;
            const uint32_t take = exc >= fr ? 0u : min(c, fr - exc);
            uint32_t pos = (uint32_t)qn + exc;
            for (uint32_t t = 0; t < take; ++t) {
                const uint32_t k = ffs_t(rem) - 1;
                M3E_CHECK_IDX(pos < 64u && t2 + k < (uint32_t)kHCap);
                W.q[pos++] = ebase | ((t2 + k) << 16);
                rem &= rem - (MT)1;
            }
            qn += (int)min(tot, fr);
            __syncwarp();
            while (qn >= 32) {
                drain(32);
                const uint32_t v = lane < qn - 32 ? W.q[32 + lane] : 0u;
                __syncwarp();
                if (lane < qn - 32) W.q[lane] = v;
                qn -= 32;
                __syncwarp();
            }
            if (tot <= fr) break;
        }
    };
    // A. rows, 32 per step
    for (uint32_t r0 = 0; r0 < NR; r0 += 32) {
        const uint32_t bit = RAr - r0 < 32u ? 1u << (RAr - r0) : 0u;
        const unsigned M = __reduce_or_sync(0xffffffffu, bit);
        const uint4 rc = S.rec[cb + __popc(M & le) - 1];
        cb += __popc(M);
        const uint32_t r = r0 + lane;
        const int i0 = (int)(r - rc.x);
        const int g0 = (int)(rc.y & 255u) + i0, t1 = (int)((rc.y >> 8) & 255u), m1 = (int)(rc.z & 255u);
        MT rem = 0;
        float z0 = 0.0f;
        if (r < NR) {
            const float x0 = hx[g0], y0 = hy[g0];
            z0 = hz[g0];
            // four layer-1 hits per iteration, two per packed fp32 operation (cos_sep)
            for (int k0 = 0; k0 < m1; k0 += 4) {
#if M3E_SEL_FSETP
                uint32_t nib = 0u;
#endif
#pragma unroll
                for (int h = 0; h < 4; h += 2) {
                    const int k = k0 + h;
                    const float2 c = cos_sep2(x0, y0, make_float2(hx[t1 + k], hx[t1 + k + 1]),
                                              make_float2(hy[t1 + k], hy[t1 + k + 1]), P.inv_r0r1);
                    // c >= c01_min as the sign of the exact difference
                    const float2 d = __fadd2_rn(c, make_float2(-P.c01_min, -P.c01_min));
#if M3E_SEL_FSETP
                    if (d.x >= 0.0f) nib |= 1u << h;
                    if (d.y >= 0.0f) nib |= 2u << h;
#else
                    const uint32_t fail = (__float_as_uint(d.x) >> 31) | ((__float_as_uint(d.y) >> 30) & 2u);
                    rem |= (MT)(fail ^ 3u) << k;
#endif
                }
#if M3E_SEL_FSETP
                rem |= (MT)nib << k0;
#endif
            }
            rem &= m1 >= kMB ? ~(MT)0 : ((MT)1 << m1) - 1;   // hits past the frame's layer 1
        }
        // pair entry {g0 | g1 << 8 | s2 << 16 | j << 24, u, n2, 0}
        const uint32_t ehi = rc.y & 0xFFFF0000u, m2 = rc.z >> 8;
        for (;;) {
            const uint32_t c = popc_t(rem);
            const uint32_t inc = warp_incl(c), exc = inc - c;
            const uint32_t tot = __shfl_sync(0xffffffffu, inc, 31);
            const uint32_t fr = 64u - (uint32_t)pn;   // pair list capacity 64, expanded 32 at a time
            const uint32_t take = exc >= fr ? 0u : min(c, fr - exc);
            uint32_t pos = (uint32_t)pn + exc;
            for (uint32_t t = 0; t < take; ++t) {
                const int k = ffs_t(rem) - 1;
                // Delta-lambda = z2 / dr12 - u(i0, i1), u = z1 (1/dr12 + 1/dr01) - z0 / dr01
                const float u = pair_u(P, z0, hz[t1 + k]);
                M3E_CHECK_IDX(pos < 64u && t1 + k < kHCap);
                S.pl[pos++] = make_uint4((uint32_t)g0 | ((uint32_t)(t1 + k) << 8) | ehi, __float_as_uint(u), m2, 0u);
                rem &= rem - (MT)1;
            }
            pn += (int)min(tot, fr);
            __syncwarp();
            while (pn >= 32) expand();
            if (tot <= fr) break;
        }
    }
    while (pn > 0) expand();
    if (qn > 0) drain(qn);
    __syncwarp();

    // per-frame results (lane j): n_cand, reason, list start, store prefix
    const int c = isf ? S.cnt[lane] : 0;
    const int count = min(c, P.cuts_max + 1);
    const int reason = count > P.cuts_max ? M3E_REASON_TRIPLET_OVERFLOW : M3E_REASON_NONE;
    const uint32_t ns = reason == M3E_REASON_NONE ? (uint32_t)c : 0u;
    const uint32_t lc = (uint32_t)min(c, P.cuts_max);
    const uint32_t ls = warp_incl(lc) - lc;
    const uint32_t sp_i = warp_incl(ns);
    const uint32_t tot = __shfl_sync(0xffffffffu, sp_i, 31);
    const uint32_t nslot = warp_sum(min(ns, (uint32_t)P.max_tracks));   // its output track slots
    if (isf) {
        A.sel[f0 + lane] = (uint32_t)count | ((uint32_t)reason << 16);
        S.pl[lane] = make_uint4(ls, sp_i - ns, sp, ns);
    }
    unsigned long long base = 0;
    if (lane == 0 && tot) base = atomicAdd(reinterpret_cast<unsigned long long*>(A.ticket + 6), tot);
    base = __shfl_sync(0xffffffffu, base, 0);
    const bool fits = base + tot <= A.cand_cap;
    __syncwarp();
    if (fits) {
        // list entry e of frame j -> store entry base + store prefix + (e - list start);
        // entries of overflow frames are dropped
        for (int e = lane; e < L; e += 32) {
            const uint32_t pk = e < kCandSmem ? W.cidx[e] : gl[e];
            const uint32_t j = pk >> 24;
            const uint4 ft = S.pl[j];
            if (ft.w) {
                // hit offsets inside the frame (window index - the frame's window start)
                const uint32_t s0w = ft.z & 255u;
                const uint32_t o0 = (pk & 255u) - s0w, o1 = ((pk >> 8) & 255u) - s0w, o2 = ((pk >> 16) & 255u) - s0w;
                A.cand_g[base + ft.y + ((uint32_t)e - ft.x)] = make_uint4(wlo + s0w, f0 + j, o1 | (o2 << 16), o0);
            }
        }
    } else {
        // a warp-batch that does not fit leaves its (partial) range marked unused
        const uint32_t nw = base < A.cand_cap ? (uint32_t)(A.cand_cap - base) : 0u;
        for (uint32_t e = lane; e < nw; e += 32) A.cand_g[base + e] = make_uint4(0u, kSpilled, 0u, 0u);
    }
    if (lane == 0) {
        A.bsel[b] = fits ? (uint32_t)base : kSpilled;
        A.bcnt[b] = fits ? tot : 0u;
        A.bslot[b] = nslot;
        if (!fits) A.spill_out[atomicAdd(A.ticket + 5, 1u)] = b;   // for the fused kernel
    }
    return true;
}

// Selection Cuts (Alg. 2, Eq. 2-5) of one big frame (phase-II occupancy, up to 64
// (NW = 1) or kMask2Hits (NW = 2) hits in layers 1 and 2; whole warp), factorised by
// the hits each cut depends on so that no (i0, i1, i2) combination is evaluated
// arithmetically:
//   1. Phi_12 depends on (i1, i2) only: one lane per layer-1 hit computes its mask
//      over layer 2, m12[i1] (n1 n2 tests instead of one per (i0, i1, i2));
//   2. Delta-lambda = fma(z2, 1/dr12, -u(i0, i1)) is non-decreasing in z2 (for a
//      given pair), so the layer-2 hits passing it form a contiguous run in z
//      order: layer 2 is ranked by z once, with prefix masks pm[r] of the r lowest;
//   3. one lane per (i0) row: the Phi_01 mask over layer 1, its set bits emitted in
//      order to the pair list with u(i0, i1);
//   4. one lane per listed pair: two binary searches over the sorted z give the
//      run [lo, hi) with the very predicate |fma(z2, 1/dr12, -u)| <= dl_max, and the
//      pair's layer-2 survivors are m12[i1] & pm[hi] & ~pm[lo]; their set bits go in
//      order to the FIFO, whose full 32s are tested for the r_t window (Eq. 5).
// Every decision is the per-hit fp32 test of the other walks (cos_sep2, pair_u,
// pass_rtc_sq), so survivor set and (i0, i1, i2) order are those of Alg. 2 and the
// other walks' (R3 overflow: stops past cuts_max).  Candidates i0 | i1 << 10 |
// i2 << 20 go to out[pos], pos < cuts_max; returns min(#survivors, cuts_max + 1).
// gm12: NW = 2 only, the warp's global scratch for m12 (n1 x 2 words).
template <int NW>
__device__ __forceinline__ int select_frame_mask(const DevParams& P, const Frame& F, MaskSel<NW>& M,
                                                 unsigned long long* gm12, uint32_t* q, uint32_t* out) {
    typedef unsigned long long u64;
    const int lane = threadIdx.x & 31;
    const unsigned lt = (1u << lane) - 1u;
    const int n0 = F.n[0], n1 = F.n[1], n2 = F.n[2];
    if (n0 == 0 || n1 == 0 || n2 == 0) return 0;
    const float *X = F.x, *Y = F.y, *Z = F.z;
    const int s0 = F.s[0], s1 = F.s[1], s2 = F.s[2];
    auto m12 = [&](int i1, int w) -> u64& {
        if constexpr (NW == 1) return M.m12[i1];
        else return gm12[2 * i1 + w];
    };
    auto pm = [&](int r, int w) -> u64& {
        if constexpr (NW == 1) return M.pm[r];
        else return M.pm[r][w];
    };
    // mask of the first n hits, word w
    auto fullw = [](int n, int w) -> u64 {
        const int b = n - 64 * w;
        return b >= 64 ? ~0ull : (b <= 0 ? 0ull : (1ull << b) - 1ull);
    };
    // cut bits of hit a against layer-l hits k0.. (four per step, two per packed op);
    // reads past the layer's end stay inside the window / input slack and are masked
    auto row = [&](float xa, float ya, int sl, int nl, float inv, float cmin, u64 (&m)[NW]) {
#pragma unroll
        for (int w = 0; w < NW; ++w) m[w] = 0ull;
#pragma unroll
        for (int w = 0; w < NW; ++w) {
            const int kend = min(nl - 64 * w, 64);
            for (int k0 = 0; k0 < kend; k0 += 4) {
#pragma unroll
                for (int h = 0; h < 4; h += 2) {
                    const int k = k0 + h, g = sl + 64 * w + k;
                    const float2 c = cos_sep2(xa, ya, make_float2(X[g], X[g + 1]), make_float2(Y[g], Y[g + 1]), inv);
                    const float2 d = __fadd2_rn(c, make_float2(-cmin, -cmin));   // c >= cmin: sign bit
                    const uint32_t fail = (__float_as_uint(d.x) >> 31) | ((__float_as_uint(d.y) >> 30) & 2u);
                    m[w] |= (u64)(fail ^ 3u) << k;
                }
            }
            m[w] &= fullw(nl, w);
        }
    };
    // 1. Phi_12 rows
    for (int i1 = lane; i1 < n1; i1 += 32) {
        M3E_CHECK_IDX(n1 <= (NW == 1 ? 64 : kMask2Hits) && n2 <= (NW == 1 ? 64 : kMask2Hits));
        u64 m[NW];
        row(X[s1 + i1], Y[s1 + i1], s2, n2, P.inv_r1r2, P.c12_min, m);
#pragma unroll
        for (int w = 0; w < NW; ++w) m12(i1, w) = m[w];
    }
    // 2. layer 2 ranked by z (ties by index), prefix masks in rank order
    for (int i2 = lane; i2 < n2; i2 += 32) {
        const float z = Z[s2 + i2];
        int r = 0;
        for (int k = 0; k < n2; ++k) {
            const float zk = Z[s2 + k];
            r += (int)((zk < z) | ((zk == z) & (k < i2)));
        }
        M3E_CHECK_IDX(r < n2 && n2 <= (NW == 1 ? 64 : kMask2Hits));
        M.zs[r] = z;
        M.ord[r] = (uint8_t)i2;
    }
    __syncwarp();
    {   // lane l: ranks RPL l .. RPL l + RPL - 1 (RPL = 2 NW), an inclusive OR-scan per word
        constexpr int RPL = 2 * NW;
        u64 part[NW], inc[NW], ex[NW];
#pragma unroll
        for (int w = 0; w < NW; ++w) part[w] = 0ull;
        const int r0 = RPL * lane;
#pragma unroll
        for (int t = 0; t < RPL; ++t)
            if (r0 + t < n2) {
                const int i = M.ord[r0 + t];
#pragma unroll
                for (int w = 0; w < NW; ++w)   // (constant indices: the words stay in registers)
                    if ((i >> 6) == w) part[w] |= 1ull << (i & 63);
            }
#pragma unroll
        for (int w = 0; w < NW; ++w) {
            inc[w] = part[w];
#pragma unroll
            for (int o = 1; o < 32; o <<= 1) {
                const u64 t = __shfl_up_sync(0xffffffffu, inc[w], o);
                if (lane >= o) inc[w] |= t;
            }
            ex[w] = __shfl_up_sync(0xffffffffu, inc[w], 1);
            if (lane == 0) {
                ex[w] = 0ull;
                pm(0, w) = 0ull;
            }
        }
        // pm[r0 + t + 1] = ex | bits of ranks r0 .. r0 + t
#pragma unroll
        for (int t = 0; t < RPL; ++t)
            if (r0 + t < n2) {
                const int i = M.ord[r0 + t];
#pragma unroll
                for (int w = 0; w < NW; ++w)
                    if ((i >> 6) == w) ex[w] |= 1ull << (i & 63);
#pragma unroll
                for (int w = 0; w < NW; ++w) pm(r0 + t + 1, w) = ex[w];
            }
    }
    __syncwarp();
    int count = 0, qn = 0, pn = 0;
    // r_t window for q[0..n) (n <= 32); true once the frame overflows
    auto drain = [&](int n) -> bool {
        const uint32_t pk = q[min(lane, n - 1)];
        const bool pass = lane < n && pass_rtc_sq(P, F, pk & 1023u, (pk >> 10) & 1023u, (pk >> 20) & 1023u);
        const unsigned m = __ballot_sync(0xffffffffu, pass);
        const int pos = count + __popc(m & lt);
        if (pass && pos < P.cuts_max) out[pos] = pk;
        count += __popc(m);
        return count > P.cuts_max;
    };
    // ordered emission of the set bits of every lane's mask (lower lanes first, word 0
    // first) into list L (capacity 64, fill n); `sink(k, pos)` writes bit k at pos;
    // `flush()` runs whenever >= 32 are listed and returns true on overflow
    auto emit = [&](u64 (&rem)[NW], int& n, auto sink, auto flush) -> bool {
        for (;;) {
            uint32_t c = 0;
#pragma unroll
            for (int w = 0; w < NW; ++w) c += (uint32_t)__popcll(rem[w]);
            const uint32_t inc = warp_incl(c), exc = inc - c;
            const uint32_t tot = __shfl_sync(0xffffffffu, inc, 31);
            const uint32_t fr = 64u - (uint32_t)n;
            const uint32_t take = exc >= fr ? 0u : min(c, fr - exc);
            uint32_t pos = (uint32_t)n + exc;
            for (uint32_t t = 0; t < take; ++t) {
                int k;
                if (NW == 1 || rem[0]) {
                    k = __ffsll(rem[0]) - 1;
                    rem[0] &= rem[0] - 1ull;
                } else {
                    k = 64 + __ffsll(rem[NW - 1]) - 1;
                    rem[NW - 1] &= rem[NW - 1] - 1ull;
                }
                sink(k, pos++);
            }
            n += (int)min(tot, fr);
            __syncwarp();
            if (flush()) return true;
            if (tot <= fr) return false;
        }
    };
    // the first K = min(pn, 32) listed pairs: their layer-2 survivors, in order, to
    // the FIFO; true once the frame overflows
    auto expand = [&]() -> bool {
        const int K = min(pn, 32);
        u64 rem[NW];
#pragma unroll
        for (int w = 0; w < NW; ++w) rem[w] = 0ull;
        uint32_t pe = 0;
        if (lane < K) {
            const uint2 e = M.pl[lane];
            pe = e.x;
            const float u = __uint_as_float(e.y);
            int lo = 0, hi = n2;   // first z-rank with fma(z, 1/dr12, -u) >= -dl_max
            while (lo < hi) {
                const int mid = (lo + hi) >> 1;
                if (fmaf(M.zs[mid], P.inv_dr12, -u) < -P.dl_max) lo = mid + 1; else hi = mid;
            }
            int lo2 = lo, hi2 = n2;   // first z-rank with fma(z, 1/dr12, -u) > dl_max
            while (lo2 < hi2) {
                const int mid = (lo2 + hi2) >> 1;
                if (fmaf(M.zs[mid], P.inv_dr12, -u) > P.dl_max) hi2 = mid; else lo2 = mid + 1;
            }
            const int i1 = (int)((e.x >> 10) & 1023u);
#pragma unroll
            for (int w = 0; w < NW; ++w) rem[w] = m12(i1, w) & pm(lo2, w) & ~pm(lo, w);
        }
        __syncwarp();
        {   // drop the K expanded pairs
            const uint2 v = lane < pn - K ? M.pl[K + lane] : make_uint2(0u, 0u);
            __syncwarp();
            if (lane < pn - K) M.pl[lane] = v;
            pn -= K;
            __syncwarp();
        }
        return emit(rem, qn, [&](int k, uint32_t pos) {
                        M3E_CHECK_IDX(pos < 64u && k < n2);
                        q[pos] = pe | ((uint32_t)k << 20);
                    },
                    [&]() -> bool {
                        while (qn >= 32) {
                            if (drain(32)) return true;
                            const uint32_t v = lane < qn - 32 ? q[32 + lane] : 0u;
                            __syncwarp();
                            if (lane < qn - 32) q[lane] = v;
                            qn -= 32;
                            __syncwarp();
                        }
                        return false;
                    });
    };
    // 3. rows, 32 per step: Phi_01 masks, pairs emitted in order
    for (int r0 = 0; r0 < n0; r0 += 32) {
        const int i0 = r0 + lane;
        u64 rem[NW];
        float z0 = 0.0f;
        if (i0 < n0) {
            z0 = Z[s0 + i0];
            row(X[s0 + i0], Y[s0 + i0], s1, n1, P.inv_r0r1, P.c01_min, rem);
        } else {
#pragma unroll
            for (int w = 0; w < NW; ++w) rem[w] = 0ull;
        }
        if (emit(rem, pn,
                 [&](int k, uint32_t pos) {
                     M3E_CHECK_IDX(pos < 64u && k < n1);
                     M.pl[pos] = make_uint2((uint32_t)i0 | ((uint32_t)k << 10), __float_as_uint(pair_u(P, z0, Z[s1 + k])));
                 },
                 [&]() -> bool {
                     while (pn >= 32)
                         if (expand()) return true;
                     return false;
                 }))
            return P.cuts_max + 1;
    }
    while (pn > 0)
        if (expand()) return P.cuts_max + 1;
    if (qn > 0 && drain(qn)) return P.cuts_max + 1;
    return count;
}

// Vertex selection of frame j (Sec. IV-C, Alg. 4; whole warp), out of line: it
// runs for ~1.5% of frames and keeps its fp64 registers and code out of the
// main loop.
// nt accepted tracks tj[0..nt) of frame `frame` (reason none); returns the
// combination count (max_combs + 1 on overflow) and the negative-track count;
// the vertex, if any, goes to *vout.
struct VOut {
    int ncomb, nneg, vtx;
};
static __device__ __noinline__ VOut vertex_frame(const DevParams* __restrict__ Pp, VScratch& V, int nt,
                                                 const m3e_track* tj, const Frame& Fv, uint32_t frame,
                                                 m3e_vertex* vout) {
    const DevParams& P = *Pp;
    const int lane = threadIdx.x & 31;
    const unsigned lt_mask = (1u << lane) - 1u;
    int ncomb = 0, nneg_out = 0;
    bool has_vtx = false;
    {
        // charge-sorted index lists, in track order
        int npos = 0, nneg = 0;
        for (int i0 = 0; i0 < nt; i0 += 32) {
            const int i = i0 + lane;
            const float kap = i < nt ? tj[i].kappa : 0.0f;
            const bool ispos = i < nt && kap > 0.0f, isneg = i < nt && kap < 0.0f;
            const unsigned mp = __ballot_sync(0xffffffffu, ispos);
            const unsigned mn = __ballot_sync(0xffffffffu, isneg);
            if (ispos) V.vlist[0][npos + __popc(mp & lt_mask)] = (uint8_t)i;
            if (isneg) V.vlist[1][nneg + __popc(mn & lt_mask)] = (uint8_t)i;
            npos += __popc(mp);
            nneg += __popc(mn);
        }
        __syncwarp();
        nneg_out = nneg;
        if (npos >= 2 && nneg >= 1) {
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
                        const int a = V.vlist[0][ia], bb = V.vlist[0][ib], e = V.vlist[1][ie];
                        const double dE = track_energy(P, tj[a].kappa) + track_energy(P, tj[bb].kappa) +
                                          track_energy(P, tj[e].kappa) - kMuMass;
                        pass = fabs(dE) <= P.e_window;
                        code = (uint32_t)a | ((uint32_t)bb << 8) | ((uint32_t)e << 16);
                    }
                }
                const unsigned m = __ballot_sync(0xffffffffu, pass);
                const int pos = ncomb + __popc(m & lt_mask);
                if (pass && pos < P.max_combs) V.vcomb[pos] = code;
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
                    const uint32_t code = V.vcomb[c];
                    // the same inline routine as triple_kernel's (identical rounding)
                    const VTrk T0 = make_vtrk(P, tj[code & 255u], Fv);
                    const VTrk T1 = make_vtrk(P, tj[(code >> 8) & 255u], Fv);
                    const VTrk T2 = make_vtrk(P, tj[(code >> 16) & 255u], Fv);
                    const VResult r = vertex_triple_inl(P, T0, T1, T2);
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
                        const uint32_t code = V.vcomb[widx];
                        m3e_vertex v;
                        v.frame = frame;
                        v.track[0] = (uint16_t)(code & 255u);
                        v.track[1] = (uint16_t)((code >> 8) & 255u);
                        v.track[2] = (uint16_t)((code >> 16) & 255u);
                        v.pad = 0;
                        v.pad2 = 0;
                        v.x = bres.x; v.y = bres.y; v.z = bres.z;
                        v.chi2 = bres.chi2;
                        v.target_dist = (float)bres.tdist;
                        v.p_total = (float)bres.ptot;
                        *vout = v;
                    }
                }
            }
        }
    }
    VOut r;
    r.ncomb = ncomb;
    r.nneg = nneg_out;
    r.vtx = has_vtx ? 1 : 0;
    return r;
}

// per-warp run summary -> the call's m3e_summary (one lane)
__device__ __forceinline__ void flush_summary(m3e_summary* sm, const uint32_t* acc) {
    typedef unsigned long long u64;
    if (acc[7]) atomicAdd((u64*)&sm->frames, (u64)acc[7]);
    for (int i = 0; i < 6; ++i)
        if (acc[i]) atomicAdd((u64*)&sm->kept_by_reason[i], (u64)acc[i]);
    if (acc[6]) atomicAdd((u64*)&sm->candidates, (u64)acc[6]);
    if (acc[8]) atomicAdd((u64*)&sm->tracks, (u64)acc[8]);
    if (acc[9]) atomicAdd((u64*)&sm->kept_hits, (u64)acc[9]);
    if (acc[M3E_REASON_VERTEX]) atomicAdd((u64*)&sm->vertices, (u64)acc[M3E_REASON_VERTEX]);
    if (acc[10]) atomicExch((u64*)&sm->overflow, 1ull);
    if (acc[11]) atomicAdd((u64*)&sm->track_slots, (u64)acc[11]);
}

// ------------------------------------------------------------------ kernel ----
template <int MODE, bool BIG>
__global__ void __launch_bounds__(kThreads, MODE == kModeSelectC ? (BIG ? M3E_MIN_BLOCKS_SEL_BIG : M3E_MIN_BLOCKS_SEL)
                                                                  : M3E_MIN_BLOCKS)
    filter_kernel(const KArgs A) {
    extern __shared__ __align__(16) uint8_t smem_raw[];
    Smem& S = *reinterpret_cast<Smem*>(smem_raw);
    const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
    const unsigned lt_mask = (1u << lane) - 1u;
    const DevParams& P = A.P;
    constexpr bool kOut = MODE == kModeFull || MODE == kModePack;   // ordered outputs
    WarpSmem& W = S.w[warp];
    const size_t gwarp = (size_t)blockIdx.x * kWarps + warp;
    VScratch& V = reinterpret_cast<VScratch*>(A.vscratch)[gwarp];

    if (tid == 0) S.P = A.P;
    if (lane == 0) {
        for (int i = 0; i < kNBuf; ++i) mbar_init(&W.bar[i], 1);
        fence_mbar_init();
    }
    __syncthreads();   // the only CTA barrier before the final summary flush
    // lane 0 (one staging buffer): claims pipelined two warp-batches ahead, so that
    // neither the ticket's atomic nor the next batch's window bounds is waited
    // for when its bulk copies are issued: c1 = the next warp-batch (bounds
    // loaded), c2 = the one after (claim in flight)
    // (selection kernel only: the other launches have few or no warp-batches)
    constexpr bool kAhead = kNBuf == 1 && MODE == kModeSelectC;
    uint32_t c1 = 0u, c1lo = 0u, c1hi = 0u, c2 = 0u;
    if (lane == 0) {
        issue_load(A, W, 0, claim_batch(A));
        if constexpr (kAhead) {
            c1 = claim_batch(A);
            batch_bounds(A, c1, c1lo, c1hi);
            c2 = claim_batch(A);
        }
    }
    __syncwarp();
    int buf = 0;
    uint32_t phase[kNBuf] = {};
    if (lane < 12) W.acc[lane] = 0u;   // run summary of this warp (shared memory, lane 0 updates)
    __syncwarp();

    // candidate / track slots: per-warp scratch (FULL) or the caller's fixed slots
    // (stage modes)
    uint32_t* cidx;
    float* crt;
    m3e_fit_record* crec;
    m3e_track* ctrk_base;
    constexpr bool kFlat = MODE == kModeFull || MODE == kModeSelectC;   // flat warp-batch candidate index
    // candidates below this flat index stay in shared memory (W.cidx); the big-frame
    // selection kernel keeps them all in global memory (its mask walk overlays W.cidx)
    constexpr uint32_t kCandS = (BIG && MODE == kModeSelectC) ? 0u : (uint32_t)kCandSmem;
    if constexpr (kFlat) {
        cidx = A.pool_idx + gwarp * A.pool_stride;
        crt = A.pool_rt + gwarp * A.pool_stride;
        crec = A.pool_rec + gwarp * A.pool_stride;
        ctrk_base = A.pool_trk + gwarp * A.trk_stride;
    } else {
        cidx = A.s_cand;
        crt = A.s_rt;
        crec = A.s_rec;
        ctrk_base = A.s_trk;
    }

    for (;;) {
        const uint32_t b = W.b_batch[buf];
        if (b >= A.nbatch) break;
        if (kNBuf == 2 && lane == 0) issue_load(A, W, buf ^ 1, claim_batch(A));
        mbar_wait(&W.bar[buf], phase[buf]);
        phase[buf] ^= 1u;

        BatchState& B = W.st;
        const uint32_t f0 = b * (uint32_t)A.fb;
        const int nf = (int)min(A.F - f0, (uint32_t)A.fb);
        const size_t cfirst = kFlat ? 0 : (size_t)f0 * P.cuts_max;   // slot of frame 0
        const size_t tfirst = MODE == kModeFull ? 0 : (size_t)f0 * P.max_tracks;
        m3e_track* ctrk = ctrk_base;

        // ---------------------------------------------------- S: Selection Cuts
        // production path: the whole warp-batch as one flat walk (eligible
        // warp-batches; the per-frame walk below handles the others)
        bool flat_done = false;
        if constexpr (MODE == kModeSelectC && !M3E_NO_FLAT_SELECT) {
            flat_done = select_batch_flat<uint32_t>(A, W, b, f0, nf, cidx);
        }
        if constexpr (MODE == kModeFull || MODE == kModeSelect || MODE == kModeSelectC) {
          if (!flat_done) {
            uint32_t cbase = 0;   // flat: candidate index of frame j's first candidate
            for (int j = 0; j < nf; ++j) {
                const Frame Fv = frame_view(A, W, buf, j);
                const bool inval = Fv.n[0] > kMaxLayerHits || Fv.n[1] > kMaxLayerHits ||
                                   Fv.n[2] > kMaxLayerHits || Fv.n[3] > kMaxLayerHits;
                int count = 0;
                if (!inval) {
                    uint32_t* ci = cidx + cfirst + (size_t)j * P.cuts_max;
                    float* cr = crt + cfirst + (size_t)j * P.cuts_max;
                    auto emit = [&](int pos, uint32_t packed, float rt) {
                        if constexpr (kFlat) {
                            const uint32_t fi = cbase + (uint32_t)pos;
                            if (below(fi, kCandS)) {
                                W.cidx[fi] = packed;
                                W.crt[fi] = rt;
                            } else {
                                cidx[fi] = packed;
                                crt[fi] = rt;
                            }
                        } else {
                            ci[pos] = packed;
                            cr[pos] = rt;
                        }
                    };
                    count = -1;
                    if constexpr (BIG && MODE == kModeSelectC) {
                        // big frames of up to 96 hits in layers 1 and 2: the mask-factorised walk
                        if (Fv.n[1] <= 64 && Fv.n[2] <= 64) {
                            count = select_frame_mask<1>(P, Fv, W.ms1, nullptr, W.q, cidx + cbase);
                            __syncwarp();
                        } else if (Fv.n[1] <= kMask2Hits && Fv.n[2] <= kMask2Hits && A.pair_scratch) {
                            count = select_frame_mask<2>(
                                P, Fv, W.ms2,
                                reinterpret_cast<unsigned long long*>(
                                    (reinterpret_cast<uintptr_t>(A.pair_scratch + gwarp * kPairWords) + 7) & ~(uintptr_t)7),
                                W.q,
                                cidx + cbase);
                            __syncwarp();
                        }
                    }
                    if (count < 0 && BIG && (long long)Fv.n[0] * Fv.n[1] * Fv.n[2] > kBigCombos && A.pair_scratch) {
                        CandSink sk;
                        if constexpr (kFlat) {
                            sk = CandSink{W.cidx, W.crt, cidx, crt, cbase, kCandS};
                        } else {
                            sk = CandSink{ci, cr, ci, cr, 0u, 0u};
                        }
                        // (its address is passed: a copy here, so that Fv stays in registers
                        // instead of being stored to local memory for every frame)
                        const Frame Fb = Fv;
                        count = select_frame_big(&S.P, Fb, W.q, A.pair_scratch + gwarp * kPairWords, sk, kPairCapG);
                        __syncwarp();
                    }
                    if (count < 0) {
                        const uint32_t g = W.offs[buf][4 * j];
                        if (MODE == kModeSelectC && g >= W.b_winlo[buf] && W.offs[buf][4 * j + 4] <= W.b_winhi[buf]) {
                            // staged frame: the same walk with shared-memory addressing
                            Frame Fs = Fv;
                            const uint32_t d = g - W.b_winlo[buf];
                            Fs.x = W.hx[buf] + d;
                            Fs.y = W.hy[buf] + d;
                            Fs.z = W.hz[buf] + d;
                            count = select_frame_warp<MODE != kModeSelectC>(P, Fs, W.q, W.pl, emit);
                        } else {
                            count = select_frame_warp<MODE != kModeSelectC>(P, Fv, W.q, W.pl, emit);
                        }
                    }
                    __syncwarp();
                }
                const int r = inval ? M3E_REASON_INVALID
                                    : (count > P.cuts_max ? M3E_REASON_TRIPLET_OVERFLOW : M3E_REASON_NONE);
                if (lane == 0) {
                    B.ncand[j] = count;
                    B.reason[j] = r;
                    B.nstored[j] = r == M3E_REASON_NONE ? count : 0;
                }
                cbase += r == M3E_REASON_NONE ? (uint32_t)count : 0u;
            }
          }
        } else if constexpr (MODE == kModeFit) {
            for (int j = lane; j < nf; j += 32) {
                const int n = A.s_ncand[f0 + j];
                B.ncand[j] = n;
                B.reason[j] = n > P.cuts_max ? M3E_REASON_TRIPLET_OVERFLOW : M3E_REASON_NONE;
                B.nstored[j] = n > P.cuts_max ? 0 : n;
            }
        } else if constexpr (MODE == kModeVertex) {
            for (int j = lane; j < nf; j += 32) {
                B.ncand[j] = 0;
                B.nstored[j] = 0;
                B.reason[j] = M3E_REASON_NONE;
                B.ntrk[j] = min((int)A.s_ntrk[f0 + j], P.max_tracks);
            }
        } else {  // kModePack
            for (int j = lane; j < nf; j += 32) {
                B.ncand[j] = 0;
                B.nstored[j] = 0;
                B.ntrk[j] = 0;
                B.ncomb[j] = 0;
                B.nneg[j] = 0;
                B.reason[j] = A.s_reason[f0 + j];
            }
        }
        __syncwarp();

        if (MODE == kModeSelectC && !flat_done) {   // candidates -> store, warp-batch contiguous
            for (int j = lane; j < nf; j += 32) {
                A.sel[f0 + j] = (uint32_t)B.ncand[j] | ((uint32_t)B.reason[j] << 16);
                W.pref[j] = (uint32_t)B.nstored[j];
            }
            __syncwarp();
            warp_scan(W.pref, nf);
            const uint32_t tot = W.pref[nf];
            unsigned long long base = 0;
            if (lane == 0 && tot) base = atomicAdd(reinterpret_cast<unsigned long long*>(A.ticket + 6), tot);
            base = __shfl_sync(0xffffffffu, base, 0);
            const bool fits = base + tot <= A.cand_cap;
            // a warp-batch that does not fit leaves its (partial) range marked unused
            const uint32_t nw = fits ? tot : (base < A.cand_cap ? (uint32_t)(A.cand_cap - base) : 0u);
            for (uint32_t e = lane; e < nw; e += 32) {
                uint4 c = make_uint4(0u, kSpilled, 0u, 0u);
                if (fits) {
                    const uint32_t pk = below(e, kCandS) ? W.cidx[e] : cidx[e];
                    const int j = find_frame(W.pref, nf, e);
                    const uint32_t* of = W.offs[buf] + 4 * j;
                    c.x = of[0];                                  // frame's first hit
                    c.y = f0 + (uint32_t)j;                       // frame
                    c.z = ((of[1] - of[0]) + ((pk >> 10) & 1023u)) | (((of[2] - of[0]) + ((pk >> 20) & 1023u)) << 16);
                    c.w = pk & 1023u;                             // hit offsets inside the frame
                }
                A.cand_g[base + e] = c;
            }
            const uint32_t nslot =
                warp_sum(lane < nf ? min((uint32_t)B.nstored[lane], (uint32_t)P.max_tracks) : 0u);
            if (lane == 0) {
                A.bsel[b] = fits ? (uint32_t)base : kSpilled;
                A.bcnt[b] = fits ? tot : 0u;
                A.bslot[b] = nslot;
                if (!fits) A.spill_out[atomicAdd(A.ticket + 5, 1u)] = b;   // for the fused kernel
            }
        }

        if constexpr (MODE == kModeSelect) {
            for (int j = lane; j < nf; j += 32) {
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

        // --------- F + T: triplet fit, one lane per candidate, fused with the
        // per-frame ballot compaction of the accepted tracks (candidate order)
        if constexpr (MODE == kModeFull || MODE == kModeFit) {
            for (int j = lane; j < nf; j += 32) {
                W.pref[j] = (uint32_t)B.nstored[j];
                B.ntrk[j] = 0;
                B.nneg[j] = 0;
                W.npos[j] = 0;
            }
            __syncwarp();
            warp_scan(W.pref, nf);
            const int total = (int)W.pref[nf];
            for (int e0 = 0; e0 < total; e0 += 32) {
                const int e = e0 + lane;
                const bool valid = e < total;
                const int j = valid ? find_frame(W.pref, nf, (uint32_t)e) : kFB;
                FitOut o;
                uint32_t pk = 0;
                size_t slot = 0;
                o.status = 7;
                if (valid) {
                    float rt;
                    if constexpr (MODE == kModeFull) {   // flat warp-batch candidate index
                        slot = (size_t)e;
                        if (e < kCandSmem) {
                            pk = W.cidx[e];
                            rt = W.crt[e];
                        } else {
                            pk = cidx[e];
                            rt = crt[e];
                        }
                    } else {
                        slot = cfirst + (size_t)j * P.cuts_max + (e - (int)W.pref[j]);
                        pk = cidx[slot];
                        rt = crt[slot];
                    }
                    const Frame Fv = frame_view(A, W, buf, j);
                    o = fit_candidate<!BIG>(P, Fv, pk & 1023u, (pk >> 10) & 1023u, (pk >> 20) & 1023u, rt);
                }
                if constexpr (MODE == kModeFit) {   // per-candidate record (stage tap)
                    if (valid) {
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
                }
                const bool acc = valid && o.status == 0 && B.reason[j] == M3E_REASON_NONE;
                const unsigned m_acc = __ballot_sync(0xffffffffu, acc);
                const unsigned grp = __match_any_sync(0xffffffffu, j);   // lanes of the same frame
                const int pos = (valid ? B.ntrk[j] : 0) + __popc(m_acc & grp & lt_mask);
                const bool store = acc && pos < P.max_tracks;
                if (store) {
                    m3e_track t;
                    t.frame = f0 + j;
                    t.hit[0] = (uint16_t)(pk & 1023u);
                    t.hit[1] = (uint16_t)((pk >> 10) & 1023u);
                    t.hit[2] = (uint16_t)((pk >> 20) & 1023u);
                    t.hit[3] = (uint16_t)o.hit3;
                    t.kappa = o.kappa;
                    t.chi2 = o.chi2;
                    t.cos_theta01 = o.cth01;
                    t.cx = o.cx;
                    t.cy = o.cy;
                    ctrk[tfirst + (size_t)j * P.max_tracks + pos] = t;
                }
                const unsigned m_neg = __ballot_sync(0xffffffffu, store && o.kappa < 0.0f);
                const unsigned m_pos = __ballot_sync(0xffffffffu, store && o.kappa > 0.0f);
                __syncwarp();
                if (valid && lane == __ffs(grp) - 1) {   // group leader updates the frame's counters
                    B.ntrk[j] += __popc(m_acc & grp);
                    B.nneg[j] += __popc(m_neg & grp);
                    W.npos[j] += __popc(m_pos & grp);
                }
                __syncwarp();
            }
            for (int j = lane; j < nf; j += 32) {
                if (B.reason[j] != M3E_REASON_NONE) continue;
                const int cnt = B.ntrk[j];
                B.ntrk[j] = min(cnt, P.max_tracks + 1);
                if (cnt > P.max_tracks) {
                    B.reason[j] = M3E_REASON_TRACK_OVERFLOW;
                    B.nneg[j] = 0;
                }
            }
            __syncwarp();
        }

        if constexpr (MODE == kModeFit) {
            for (int j = lane; j < nf; j += 32) {
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
            // FULL: charge counts known from F, only frames with e+e+e- candidates
            // (nf <= kFB <= 32: one lane per frame)
            bool need = lane < nf;
            if constexpr (MODE == kModeFull) {
                need = need && B.reason[lane] == M3E_REASON_NONE && W.npos[lane] >= 2 && B.nneg[lane] >= 1;
                if (lane < nf && !need) B.ncomb[lane] = 0;
            }
            __syncwarp();
            for (unsigned todo = __ballot_sync(0xffffffffu, need); todo; todo &= todo - 1) {
                const int j = __ffs(todo) - 1;
                const Frame Fv = frame_view(A, W, buf, j);
                if (B.reason[j] == M3E_REASON_NONE) {
                    const VOut r = vertex_frame(&S.P, V, min(B.ntrk[j], P.max_tracks),
                                                ctrk + tfirst + (size_t)j * P.max_tracks, Fv, f0 + j, &V.vtx[j]);
                    if (lane == 0) {
                        B.ncomb[j] = r.ncomb;
                        B.nneg[j] = r.nneg;
                        if (r.ncomb > P.max_combs) B.reason[j] = M3E_REASON_COMB_OVERFLOW;
                        else if (r.vtx) B.reason[j] = M3E_REASON_VERTEX;
                    }
                } else if (lane == 0) {
                    B.ncomb[j] = 0;
                }
                __syncwarp();
            }
        }
        if constexpr (MODE == kModeVertex) {
            for (int j = lane; j < nf; j += 32) {
                m3e_frame_out fo;
                fo.n_cand = 0;
                fo.n_tracks = (uint16_t)B.ntrk[j];
                fo.n_combs = (uint16_t)B.ncomb[j];
                fo.reason = (uint8_t)B.reason[j];
                fo.n_neg = (uint8_t)min(B.nneg[j], 255);
                fo.track_first = (uint32_t)(tfirst + (size_t)j * P.max_tracks);
                fo.kept_index = 0xFFFFFFFFu;
                A.out.frames[f0 + j] = fo;
                if (B.reason[j] == M3E_REASON_VERTEX && A.s_vtx) A.s_vtx[f0 + j] = V.vtx[j];
            }
        }

        // --------------------- O: records in place, tracks / kept frames staged
        if constexpr (kOut) {
            for (int j = lane; j < nf; j += 32) {
                const int r = B.reason[j];
                const bool kept = r != M3E_REASON_NONE;
                const bool has_tracks = r == M3E_REASON_NONE || r == M3E_REASON_TRACK_OVERFLOW ||
                                        r == M3E_REASON_COMB_OVERFLOW || r == M3E_REASON_VERTEX;
                B.o_trk[j] = (MODE == kModeFull && has_tracks) ? (uint32_t)min(B.ntrk[j], P.max_tracks) : 0u;
                B.o_kept[j] = kept ? 1u : 0u;
                B.o_hits[j] = kept ? (W.offs[buf][4 * j + 4] - W.offs[buf][4 * j]) : 0u;
            }
            __syncwarp();
            warp_scan(B.o_trk, nf);
            warp_scan(B.o_kept, nf);
            warp_scan(B.o_hits, nf);
            const uint32_t nt = B.o_trk[nf], nk = B.o_kept[nf];
            uint32_t s_trk = 0, s_kept = 0;
            if (lane == 0) {
                if (nt && A.stage_trk) s_trk = atomicAdd(A.ticket + 1, nt);
                if (nk) s_kept = atomicAdd(A.ticket + 2, nk);
            }
            s_trk = __shfl_sync(0xffffffffu, s_trk, 0);
            s_kept = __shfl_sync(0xffffffffu, s_kept, 0);
            bool overflow = false;
            const m3e_outputs& O = A.out;
            for (int j = lane; j < nf; j += 32) {
                const int r = B.reason[j];
                if (O.reason) O.reason[f0 + j] = (uint8_t)r;
                if (O.frames) {   // track_first / kept_index: warp-batch relative until the pack kernel
                    m3e_frame_out fo;
                    fo.n_cand = (uint16_t)B.ncand[j];
                    fo.n_tracks = (uint16_t)B.ntrk[j];
                    fo.n_combs = (uint16_t)B.ncomb[j];
                    fo.reason = (uint8_t)r;
                    fo.n_neg = (uint8_t)min(B.nneg[j], 255);
                    fo.track_first = B.o_trk[j];
                    fo.kept_index = r != M3E_REASON_NONE ? B.o_kept[j] : 0xFFFFFFFFu;
                    O.frames[f0 + j] = fo;
                }
                if (r != M3E_REASON_NONE) {
                    const uint32_t k = s_kept + B.o_kept[j];
                    if (k < A.stage_kept_cap) {
                        KeptRec kr;
                        kr.frame = f0 + j;
                        kr.pad = 0;
                        if (r == M3E_REASON_VERTEX) {
                            kr.v = V.vtx[j];
                        } else {
                            kr.v = m3e_vertex{};
                            kr.v.frame = 0xFFFFFFFFu;
                        }
                        A.stage_kept[k] = kr;
                    } else {
                        overflow = true;
                    }
                }
            }
            if constexpr (MODE == kModeFull) {
                if (A.stage_trk) {
                    for (uint32_t e = lane; e < nt; e += 32) {
                        const int j = find_frame(B.o_trk, nf, e);
                        const uint32_t dst = s_trk + e;
                        if (dst < A.stage_trk_cap) {
                            const uint4* s4 = reinterpret_cast<const uint4*>(ctrk + (size_t)j * P.max_tracks +
                                                                             (e - B.o_trk[j]));
                            uint4* d4 = reinterpret_cast<uint4*>(A.stage_trk + dst);
                            d4[0] = s4[0];
                            d4[1] = s4[1];
                        } else {
                            overflow = true;
                        }
                    }
                }
            }
            // its track slots: sum over frames of min(stored candidates, max_tracks), as
            // the selection kernel counts them
            const uint32_t nslot =
                warp_sum(lane < nf ? min((uint32_t)B.nstored[lane], (uint32_t)P.max_tracks) : 0u);
            if (lane == 0) {
                BatchStat bs;
                bs.n_trk = nt;
                bs.n_kept = nk;
                bs.n_hits = B.o_hits[nf];
                bs.s_trk = s_trk;
                bs.s_kept = s_kept;
                bs.nf = nf;
                bs.n_slot = nslot;
                bs.pad = 0;
                A.bstat[b] = bs;
            }
            // run summary: per-warp counters in shared memory, flushed once at the end
            const int rj = lane < nf ? B.reason[lane] : -1;   // nf <= kFB <= 32
            uint32_t kr[6];
#pragma unroll
            for (int r = 0; r < 6; ++r) kr[r] = __popc(__ballot_sync(0xffffffffu, rj == r));
            const uint32_t cand = warp_sum(lane < nf ? (uint32_t)B.nstored[lane] : 0u);
            if (lane == 0) {
                for (int r = 0; r < 6; ++r) W.acc[r] += kr[r];
                W.acc[6] += cand;
                W.acc[7] += nf;
                W.acc[8] += nt;
                W.acc[9] += B.o_hits[nf];
            }
            if (__any_sync(0xffffffffu, overflow) && lane == 0) W.acc[10] = 1u;
        }
        __syncwarp();
        if constexpr (kNBuf == 2) {
            buf ^= 1;
        } else if (lane == 0) {
            if constexpr (kAhead) {
                issue_load_w(A, W, 0, c1, c1lo, c1hi);
                c1 = c2;
                batch_bounds(A, c1, c1lo, c1hi);
                c2 = claim_batch(A);
            } else {
                issue_load(A, W, 0, claim_batch(A));
            }
        }
        __syncwarp();
    }

    if constexpr (kOut) {
        __syncwarp();
        if (lane == 0 && A.out.summary) flush_summary(A.out.summary, W.acc);
    }
}

// -------------------------------------------------------- slot scan kernel ----
// Between the selection and the fit kernel: every warp-batch's first slot in the
// output track array, tbase[b] = sum of bslot over the warp-batches before b
// (warp-batch order = frame order), so that the fit kernel writes each accepted
// track straight into its final place (the track array is frame-ordered; a
// warp-batch's rejected candidates leave unused slots at the end of its range).
// Single pass: tiles of kScanTile warp-batches claimed in order by a ticket, a
// block scan, and a decoupled look-back over the tiles' {tag, sum} words.
__device__ __forceinline__ void st_volatile_v2(uint2* p, uint2 v) {
    asm volatile("st.volatile.global.v2.u32 [%0], {%1, %2};" ::"l"(p), "r"(v.x), "r"(v.y) : "memory");
}
__device__ __forceinline__ uint2 ld_volatile_v2(const uint2* p) {
    uint2 v;
    asm volatile("ld.volatile.global.v2.u32 {%0, %1}, [%2];" : "=r"(v.x), "=r"(v.y) : "l"(p) : "memory");
    return v;
}

__global__ void __launch_bounds__(kThreads) slot_scan_kernel(const __grid_constant__ KArgs A) {
    __shared__ uint32_t wsum[kWarps];
    __shared__ uint32_t s_tile, s_base;
    const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
    const uint32_t ntiles = (A.nbatch + kScanTile - 1) / kScanTile;
    const uint32_t tagA = (A.epoch << 2) | 1u, tagI = (A.epoch << 2) | 2u;
    for (;;) {
        if (tid == 0) s_tile = atomicAdd(A.ticket + 12, 1u);
        __syncthreads();
        const uint32_t t = s_tile;
        if (t >= ntiles) break;
        const uint32_t b0 = t * kScanTile + tid * kScanItems;
        uint32_t v[kScanItems];
        uint32_t sum = 0;
#pragma unroll
        for (int i = 0; i < kScanItems; ++i) {
            v[i] = b0 + i < A.nbatch ? A.bslot[b0 + i] : 0u;
            sum += v[i];
        }
        const uint32_t inc = warp_incl(sum);
        if (lane == 31) wsum[warp] = inc;
        __syncthreads();
        uint32_t woff = 0, agg = 0;
#pragma unroll
        for (int w = 0; w < kWarps; ++w) {
            woff += w < warp ? wsum[w] : 0u;
            agg += wsum[w];
        }
        if (warp == 0) {
            uint32_t ex = 0;
            if (t == 0) {
                if (lane == 0) st_volatile_v2(A.sstatus, make_uint2(tagI, agg));
            } else {
                if (lane == 0) st_volatile_v2(A.sstatus + t, make_uint2(tagA, agg));
                int j = (int)t - 1;
                for (;;) {
                    const int idx = j - lane;
                    uint2 st = make_uint2(tagI, 0u);   // virtual inclusive zero before tile 0
                    if (idx >= 0) {
                        do {
                            st = ld_volatile_v2(A.sstatus + idx);
                        } while (st.x != tagA && st.x != tagI);
                    }
                    const unsigned m = __ballot_sync(0xffffffffu, st.x == tagI);
                    const int k = m ? __ffs(m) - 1 : 32;   // nearest predecessor with an inclusive prefix
                    ex += warp_sum(lane <= k ? st.y : 0u);
                    if (m) break;
                    j -= 32;
                }
                if (lane == 0) st_volatile_v2(A.sstatus + t, make_uint2(tagI, ex + agg));
            }
            if (lane == 0) s_base = ex;
        }
        __syncthreads();
        uint32_t run = s_base + woff + inc - sum;
#pragma unroll
        for (int i = 0; i < kScanItems; ++i) {
            if (b0 + i < A.nbatch) A.tbase[b0 + i] = run;
            run += v[i];
        }
        __syncthreads();   // s_tile / wsum reused by the next tile
    }
}

cudaError_t launch_slot_scan(const KArgs& a, int grid, cudaStream_t s) {
    slot_scan_kernel<<<grid, kThreads, 0, s>>>(a);
    return cudaGetLastError();
}

// ------------------------------------------------------------- pack kernel ----
// Output stage O + packer (north-star row (f)), one pass over tiles of 256
// warp-batches:
//   counts  one thread per warp-batch: from the per-frame selection / track /
//           vertex words (fit and vertex kernels) its output tracks (each frame's
//           first max_tracks accepted; none for triplet-overflow or invalid
//           frames), its track slots (bslot), kept frames and their hits; the
//           in-batch prefixes per frame go to shared memory.  Warp-batches the
//           fused kernel ran (candidate store full; every warp-batch on the fused
//           variant) bring their counts and staged outputs in their BatchStat;
//   bases   the tile's {slots, kept frames, hits} are scanned at once and a
//           decoupled look-back over tiles gives its global bases (every count is
//           final: it never waits on compute);
//   frames  every frame record written once with its final track_first (the
//           warp-batch's first slot + the in-batch prefix: where the fit kernel
//           put its tracks) and kept_index, and the reason byte;
//   tracks  only the fused kernel's warp-batches (none at phase I): staged tracks
//           copied into their slots, the rest of the slots marked unused;
//   kept    each kept frame listed {frame, first packed hit, vertex source} at its
//           kept index for kept_kernel, which copies them (no dependent loads here:
//           a slow warp would hold the tile at its barriers).
// The run summary is accumulated per thread and flushed once per warp.
#ifndef M3E_PACK_MIN_BLOCKS
#define M3E_PACK_MIN_BLOCKS 3   // 80 registers, no spills (4 CTAs: 64 registers and spills, slower)
#endif
struct PackSmem {
    uint32_t wagg[kWarps][3];
    uint32_t base[3];
    uint32_t tile;
    uint32_t ptrk[kPackTile + 1];   // exclusive prefix of the tile's tracks per warp-batch (+ total)
    uint32_t pkept[kPackTile];      // ... of its kept frames
    uint32_t src[kPackTile];        // first track's source: store index, or staging index | 1 << 31 (fused)
    uint32_t sw[kPackTile * kFB];   // per frame of the tile: selection word,
    uint32_t fw[kPackTile * kFB];   // track / vertex word,
    uint16_t ftrk[kPackTile * kFB]; // output tracks -> exclusive prefix inside its warp-batch,
    uint16_t fhit[kPackTile * kFB]; // hits if kept,
    uint8_t fkept[kPackTile * kFB]; // kept flag -> exclusive prefix inside its warp-batch
};

size_t pack_smem_bytes() { return sizeof(PackSmem); }

__global__ void __launch_bounds__(kThreads, M3E_PACK_MIN_BLOCKS) pack_kernel(const __grid_constant__ KArgs A) {
    extern __shared__ __align__(16) uint8_t pack_smem_raw[];
    PackSmem& S = *reinterpret_cast<PackSmem*>(pack_smem_raw);
    const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
    const m3e_outputs& O = A.out;
    const DevParams& P = A.P;
    const uint32_t ntiles = (A.nbatch + kPackTile - 1) / kPackTile;
    const uint32_t fb = (uint32_t)A.fb;
    uint32_t acc[12] = {};   // run summary of this thread: kept_by_reason[6], cand, frames, tracks, hits,
                             // -, track slots
    bool overflow = false;
    for (;;) {
        if (tid == 0) S.tile = atomicAdd(A.ticket + 3, 1u);
        __syncthreads();
        const uint32_t t = S.tile;
        if (t >= ntiles) break;
        const uint32_t b = t * kPackTile + tid;
        const bool inb = b < A.nbatch;
        const bool fused = inb && (!A.bsel || A.bsel[b] == kSpilled);   // outputs staged by the fused kernel
        // n_slot: the warp-batch's slots in out.tracks (the selection kernel's count, which
        // the slot scan and the fit kernel used; the fused kernel's on the fused variant)
        uint32_t n_trk = 0, n_kept = 0, n_hits = 0, s_kept = 0, src = 0, n_slot = 0, f_trk = 0;
        if (fused) {
            const BatchStat bs = A.bstat[b];
            f_trk = bs.n_trk;
            n_kept = bs.n_kept;
            n_hits = bs.n_hits;
            s_kept = bs.s_kept;
            n_slot = A.bslot ? A.bslot[b] : bs.n_slot;
            src = bs.s_trk | 0x80000000u;
        } else if (inb) {
            src = A.bsel[b];
            n_slot = A.bslot[b];
        }
        acc[11] += n_slot;
        S.src[tid] = src;
        __syncthreads();
        const uint32_t f0 = t * kPackTile * fb;
        const uint32_t f1 = min(A.F, (t + 1) * kPackTile * fb);
        // per frame (coalesced): the words, its output tracks, kept flag and hits;
        // the loads of four strided frames issued before any is used
        for (uint32_t fa = f0 + tid; fa < f1; fa += 4 * kThreads) {
            uint32_t swv[4], wv[4];
#pragma unroll
            for (int u = 0; u < 4; ++u) {
                const uint32_t f = fa + u * kThreads;
                const bool on = f < f1 && !(S.src[(f - f0) / fb] >> 31);   // not the fused kernel's frame
                swv[u] = on ? A.sel[f] : 0xFFFFFFFFu;
                wv[u] = on ? A.fw[f] : 0u;
            }
#pragma unroll
            for (int u = 0; u < 4; ++u) {
                const uint32_t f = fa + u * kThreads;
                if (swv[u] == 0xFFFFFFFFu) continue;
                const uint32_t i = f - f0, sw = swv[u], w = wv[u];
                const int reason = (int)(w >> 24);
                const bool kept = reason != M3E_REASON_NONE;
                const bool has_tracks = reason != M3E_REASON_TRIPLET_OVERFLOW && reason != M3E_REASON_INVALID;
                const uint32_t o_trk = has_tracks ? min(w & 0xFFu, (uint32_t)P.max_tracks) : 0u;
                const uint32_t nh = kept ? A.offsets[4 * (size_t)f + 4] - A.offsets[4 * (size_t)f] : 0u;
                S.sw[i] = sw;
                S.fw[i] = w;
                S.ftrk[i] = (uint16_t)o_trk;
                S.fhit[i] = (uint16_t)nh;
                S.fkept[i] = kept ? 1 : 0;
                acc[reason < 6 ? reason : 5] += 1u;
                acc[6] += (sw >> 16) == M3E_REASON_NONE ? (sw & 0xFFFFu) : 0u;   // candidates stored
                acc[7] += 1u;
                acc[8] += o_trk;
                acc[9] += nh;
            }
        }
        __syncthreads();
        // per warp-batch: sums, and the per-frame counts turned into in-batch prefixes
        if (inb && !fused) {
            const uint32_t nf = min(A.F - b * fb, fb);
            for (uint32_t j = 0; j < nf; ++j) {
                const uint32_t i = tid * fb + j;
                const uint32_t ot = S.ftrk[i], ok = S.fkept[i];
                S.ftrk[i] = (uint16_t)n_trk;
                S.fkept[i] = (uint8_t)n_kept;
                n_trk += ot;
                n_kept += ok;
                n_hits += S.fhit[i];
            }
        }
        // block-wide scan of the three counts (track slots, kept frames, their hits),
        // then the look-back
        uint32_t it = n_slot, ik = n_kept, ih = n_hits;
#pragma unroll
        for (int o = 1; o < 32; o <<= 1) {
            const uint32_t a = __shfl_up_sync(0xffffffffu, it, o);
            const uint32_t c = __shfl_up_sync(0xffffffffu, ik, o);
            const uint32_t d = __shfl_up_sync(0xffffffffu, ih, o);
            if (lane >= o) { it += a; ik += c; ih += d; }
        }
        if (lane == 31) { S.wagg[warp][0] = it; S.wagg[warp][1] = ik; S.wagg[warp][2] = ih; }
        __syncthreads();
        if (warp == 0) {
            uint32_t a0 = lane < kWarps ? S.wagg[lane][0] : 0u, a1 = lane < kWarps ? S.wagg[lane][1] : 0u,
                     a2 = lane < kWarps ? S.wagg[lane][2] : 0u;
            const uint3 agg = make_uint3(warp_sum(a0), warp_sum(a1), warp_sum(a2));
            publish_aggregate(A, t, agg);
            const uint3 ex = resolve(A, t, agg);
            if (lane == 0) { S.base[0] = ex.x; S.base[1] = ex.y; S.base[2] = ex.z; }
        }
        uint32_t w0 = 0, w1 = 0, w2 = 0;   // this warp's offset inside the tile
        for (int w = 0; w < warp; ++w) { w0 += S.wagg[w][0]; w1 += S.wagg[w][1]; w2 += S.wagg[w][2]; }
        S.ptrk[tid] = w0 + it - n_slot;
        S.pkept[tid] = w1 + ik - n_kept;
        if (tid == kThreads - 1) S.ptrk[kPackTile] = w0 + it;
        __syncthreads();
        const uint32_t base_trk = S.base[0], base_kept = S.base[1];
        const uint32_t g_slot_b = base_trk + S.ptrk[tid];   // this warp-batch's first slot
        // the fit kernel wrote the tracks of warp-batches whose slots fit the capacity
        // into out.tracks; the others are missing from it
        if (O.tracks && inb && !fused && n_trk > 0 &&
            (uint64_t)g_slot_b + n_slot > min(O.track_capacity, (uint64_t)kInFitG))
            overflow = true;
        const uint32_t g_kept_b = base_kept + w1 + ik - n_kept, g_hits_b = S.base[2] + w2 + ih - n_hits;
        // ---- frame records, once, with call-global indices
        {
            for (uint32_t f = f0 + tid; f < f1; f += kThreads) {
                const uint32_t i = f - f0, bl = i / fb;
                if (S.src[bl] >> 31) {   // fused kernel's record: batch-relative indices
                    if (O.frames) {
                        uint2* p = reinterpret_cast<uint2*>(reinterpret_cast<uint8_t*>(O.frames + f) + 8);
                        uint2 w = *p;
                        w.x += base_trk + S.ptrk[bl];
                        if (w.y != 0xFFFFFFFFu) w.y += base_kept + S.pkept[bl];
                        *p = w;
                    }
                    continue;
                }
                const uint32_t sw = S.sw[i], w = S.fw[i];
                const int reason = (int)(w >> 24);
                if (O.reason) O.reason[f] = (uint8_t)reason;
                if (O.frames) {
                    m3e_frame_out fo;
                    fo.n_cand = (uint16_t)(sw & 0xFFFFu);
                    fo.n_tracks = (uint16_t)(w & 0xFFu);
                    fo.n_combs = (uint16_t)((w >> 16) & 0xFFu);
                    fo.reason = (uint8_t)reason;
                    fo.n_neg = (uint8_t)((w >> 8) & 0xFFu);
                    fo.track_first = base_trk + S.ptrk[bl] + S.ftrk[i];
                    fo.kept_index = reason != M3E_REASON_NONE ? base_kept + S.pkept[bl] + S.fkept[i] : 0xFFFFFFFFu;
                    O.frames[f] = fo;
                }
            }
        }
        // ---- tracks of the fused kernel's warp-batches (staged; none at phase I): one
        // warp per warp-batch, its slots = staged tracks, then unused-slot marks
        if (O.tracks && A.stage_trk) {
            unsigned todo = __ballot_sync(0xffffffffu, fused && n_slot > 0);
            while (todo) {
                const int sl = __ffs(todo) - 1;
                todo &= todo - 1;
                const uint32_t nt = __shfl_sync(0xffffffffu, f_trk, sl);
                const uint32_t ns = __shfl_sync(0xffffffffu, n_slot, sl);
                const uint32_t st = __shfl_sync(0xffffffffu, src, sl) & 0x7FFFFFFFu;
                const uint32_t g = __shfl_sync(0xffffffffu, g_slot_b, sl);
                for (uint32_t k = lane; k < max(ns, nt); k += 32) {
                    const uint32_t dst = g + k;
                    if (dst >= O.track_capacity || k >= ns || st + k >= A.stage_trk_cap) {
                        overflow = true;
                    } else if (k < nt) {
                        const uint4* s4 = reinterpret_cast<const uint4*>(A.stage_trk + st + k);
                        uint4* d4 = reinterpret_cast<uint4*>(O.tracks + dst);
                        d4[0] = s4[0];
                        d4[1] = s4[1];
                    } else {
                        write_unused_slot(O.tracks + dst);
                    }
                }
            }
        }
        // ---- kept frames (rare): each one's {frame, first packed hit, vertex source}
        // listed at its kept index; kept_kernel copies them (no dependent loads here:
        // a slow warp would hold the whole tile at its barriers)
        if (inb && n_kept > 0) {
            uint32_t kidx = g_kept_b, hb = g_hits_b;
            if (fused) {   // the fused kernel's staged kept records
                for (uint32_t j = 0; j < n_kept; ++j, ++kidx) {
                    if (s_kept + j >= A.stage_kept_cap || kidx >= O.kept_capacity) {
                        overflow = true;
                        continue;
                    }
                    const uint32_t f = A.stage_kept[s_kept + j].frame;
                    A.kept_rec[kidx] = make_uint4(f, hb, 0x80000000u | (s_kept + j), 0u);
                    hb += A.offsets[4 * (size_t)f + 4] - A.offsets[4 * (size_t)f];
                }
            } else {
                const uint32_t nf = min(A.F - b * fb, fb);
                for (uint32_t j = 0; j < nf; ++j) {
                    const uint32_t i = tid * fb + j, r = S.fw[i] >> 24;
                    if (r == M3E_REASON_NONE) continue;
                    if (kidx < O.kept_capacity) A.kept_rec[kidx] = make_uint4(b * fb + j, hb, r, 0u);
                    else overflow = true;
                    ++kidx;
                    hb += S.fhit[i];
                }
            }
        }
        // the call's last warp-batch closes the packed offsets and publishes the
        // kept-frame count for kept_kernel
        if (inb && b == A.nbatch - 1) {
            const uint32_t K = g_kept_b + n_kept;
            if (O.kept_offsets && K <= O.kept_capacity) O.kept_offsets[4 * (size_t)K] = g_hits_b + n_hits;
            A.ticket[13] = K;
        }
        __syncthreads();
    }
    // run summary: one flush per warp (the fused kernel flushed its own frames)
    uint32_t sacc[12];
#pragma unroll
    for (int r = 0; r < 12; ++r) sacc[r] = warp_sum(acc[r]);
    sacc[10] = __any_sync(0xffffffffu, overflow) ? 1u : 0u;
    if (lane == 0 && O.summary) flush_summary(O.summary, sacc);
}

// ------------------------------------------------------------- kept kernel ----
// The kept frames listed by the pack kernel (kept_rec[k] = {frame, first packed hit,
// vertex source}), one warp each: frame index, packed layer offsets, vertex record
// (the vertex stage's, the fused kernel's staged one, or none) and the hits, SoA.
__global__ void __launch_bounds__(kThreads) kept_kernel(const __grid_constant__ KArgs A) {
    const int lane = threadIdx.x & 31;
    const m3e_outputs& O = A.out;
    const uint32_t K = min(*reinterpret_cast<const volatile uint32_t*>(A.ticket + 13), (uint32_t)O.kept_capacity);
    bool overflow = false;
    for (uint32_t k = (blockIdx.x * kThreads + threadIdx.x) >> 5; k < K; k += (gridDim.x * kThreads) >> 5) {
        const uint4 r = A.kept_rec[k];
        const uint32_t f = r.x, hb = r.y;
        const uint32_t lo = A.offsets[4 * (size_t)f];
        const uint32_t nh = A.offsets[4 * (size_t)f + 4] - lo;
        if (lane == 0) {
            if (O.kept_frame) O.kept_frame[k] = f;
            if (O.vertices) {
                m3e_vertex vx;
                if (r.z & 0x80000000u) {
                    vx = A.stage_kept[r.z & 0x7FFFFFFFu].v;
                } else if (r.z == M3E_REASON_VERTEX) {
                    vx = A.vrec[A.vk[f]];
                } else {
                    vx = m3e_vertex{};
                    vx.frame = 0xFFFFFFFFu;
                }
                O.vertices[k] = vx;
            }
        }
        if (O.kept_offsets && lane < 4) O.kept_offsets[4 * (size_t)k + lane] = hb + (A.offsets[4 * (size_t)f + lane] - lo);
        if (O.kept_x)
            for (uint32_t e = lane; e < nh; e += 32) {
                const uint32_t dst = hb + e;
                if (dst < O.kept_hit_capacity) {
                    O.kept_x[dst] = A.x[lo + e];
                    O.kept_y[dst] = A.y[lo + e];
                    O.kept_z[dst] = A.z[lo + e];
                } else {
                    overflow = true;
                }
            }
    }
    if (__any_sync(0xffffffffu, overflow) && lane == 0 && O.summary)
        atomicExch(reinterpret_cast<unsigned long long*>(&O.summary->overflow), 1ull);
}

cudaError_t read_check_line(unsigned int* line) {
#ifdef M3E_CHECK
    cudaError_t e = cudaMemcpyFromSymbol(line, g_m3e_check_line, sizeof(unsigned int));
    if (e != cudaSuccess) return e;
    const unsigned int zero = 0;
    return cudaMemcpyToSymbol(g_m3e_check_line, &zero, sizeof(unsigned int));
#else
    *line = 0xFFFFFFFFu;   // checks not compiled in
    return cudaSuccess;
#endif
}

cudaError_t launch_kept(const KArgs& a, int grid, cudaStream_t s) {
    kept_kernel<<<grid, kThreads, 0, s>>>(a);
    return cudaGetLastError();
}

// ------------------------------------------------------------ fit kernel ----
// Split path, F + T: the triplet fit (Sec. IV-B, Alg. 3, Eqs. 5-8) of
// every stored candidate and the per-frame track stage.  Each warp keeps a ring
// of two warp-batch slots in shared memory: a slot holds the warp-batch's hits
// and layer offsets, staged by TMA bulk copies (double-buffered: the next
// warp-batch loads while the current one is fitted), and its store segment (the
// candidates in frame order, L2-prefetched by a bulk prefetch).  Candidates are
// fitted one lane per candidate, 32 at a time; a chunk runs on from the end of
// the current warp-batch into the next one, so lanes stay dense although a
// warp-batch holds ~50 candidates.  Accepted tracks are ranked per frame
// (match_any on slot | frame; candidate order = Alg. 3's order); the first
// max_tracks of each frame (the tracks a frame outputs, R3) are written straight
// into their final place: compacted to the front of the warp-batch's slot range
// in out.tracks (from tbase[b], slot_scan_kernel), so the track array needs no
// reordering copy; without a track output (or past its capacity) to the front of
// the warp-batch's store segment in fit_g, for the vertex stage.  Rejected
// candidates write nothing.  Once a warp-batch is consumed, one lane per frame:
// track-overflow decision, the frame's track word, and frames with e+ e+ e-
// appended to the vertex list; the warp-batch's unused slots are marked; its slot
// then takes the next warp-batch.
#ifndef M3E_FIT_HCAP
#define M3E_FIT_HCAP 288   // measured (fit ms): 240 4.35, 288 4.20, 320 4.23, 384 5.21 (2 CTAs per SM)
#endif
constexpr int kFitHCap = M3E_FIT_HCAP;   // hits of a warp-batch staged (larger ones are read from HBM)

struct __align__(16) FitSlot {
    float hx[kFitHCap], hy[kFitHCap], hz[kFitHCap];
    uint32_t offs[4 * kFB + 4];   // layer offsets of the warp-batch's frames (+ end)
    uint32_t selw[kFB];           // its frames' selection words (cp.async)
    uint64_t bar;
    const float* px;              // hit arrays as seen by a global hit index: the staged window
    const float* py;              // shifted by its first hit (generic addresses), or the inputs
    const float* pz;              // in HBM for a warp-batch larger than the window
    m3e_track* td;                // where its output tracks go: out.tracks + its first slot, or the
                                  // front of its store segment in fit_g (no track output requested)
    uint32_t b, f0, nf, winlo;    // warp-batch, its frames, first staged hit (0xFFFFFFFF: from HBM)
    uint32_t sbase, n, t, nacc;   // store segment, its entries, entries consumed, output tracks written
    uint32_t tcode, nslot;        // its first track for the vertex stage (kInFitG | fit_g index, or the
                                  // out.tracks index), its slots in out.tracks (0: tracks in fit_g)
    int cnt[kFB], neg[kFB], pos[kFB];   // per frame: accepted, stored e-, stored e+
};

// descriptor words of the warp's next warp-batch, fetched ahead by cp.async:
// {first hit, end hit, store segment, its entries, first track slot, track slots}
struct FitPre {
    uint32_t w[6];
};

__device__ __forceinline__ void cp_async4(void* dst, const void* src) {
    asm volatile("cp.async.ca.shared.global [%0], [%1], 4;" ::"r"(smem_u32(dst)), "l"(src) : "memory");
}
__device__ __forceinline__ void cp_async_commit() { asm volatile("cp.async.commit_group;" ::: "memory"); }
__device__ __forceinline__ void cp_async_wait_all() { asm volatile("cp.async.wait_all;" ::: "memory"); }

// lanes 0-3: start fetching the descriptor words of warp-batch b (none if b >= nbatch)
__device__ __forceinline__ void fit_prefetch(const KArgs& A, FitPre& D, uint32_t b) {
    const int lane = threadIdx.x & 31;
    if (b < A.nbatch && lane < 6) {
        const uint32_t f0 = b * (uint32_t)A.fb;
        const uint32_t nf = min(A.F - f0, (uint32_t)A.fb);
        const uint32_t* src = lane == 0 ? A.offsets + 4 * (size_t)f0
                            : lane == 1 ? A.offsets + 4 * (size_t)(f0 + nf)
                            : lane == 2 ? A.bsel + b
                            : lane == 3 ? A.bcnt + b
                            : lane == 4 ? A.tbase + b : A.bslot + b;
        cp_async4(&D.w[lane], src);
    }
    cp_async_commit();
}

// whole warp: warp-batch b into slot S (every read of the slot's previous
// warp-batch done); its descriptor is in D; then D starts fetching b_next
__device__ __forceinline__ void fit_assign(const KArgs& A, FitSlot& S, FitPre& D, uint32_t b, uint32_t b_next) {
    const int lane = threadIdx.x & 31;
    cp_async_wait_all();
    __syncwarp();
    if (lane < kFB) {
        S.cnt[lane] = 0;
        S.neg[lane] = 0;
        S.pos[lane] = 0;
    }
    const bool live = b < A.nbatch;
    const uint32_t f0 = b * (uint32_t)A.fb;
    const uint32_t nf = live ? min(A.F - f0, (uint32_t)A.fb) : 0u;
    if ((uint32_t)lane < nf) cp_async4(&S.selw[lane], A.sel + f0 + lane);   // waited for by fit_frames
    if (lane == 0) {
        S.b = b;
        S.t = 0;
        S.nacc = 0;
        S.f0 = f0;
        S.nf = nf;
        S.n = 0;
        if (live) {
            const uint32_t lo = D.w[0], hi = D.w[1], sb = D.w[2];
            const uint32_t n = sb == kSpilled ? 0u : D.w[3];
            const uint32_t wlo = lo & ~3u, whi = (hi + 3u) & ~3u;
            const bool inw = whi - wlo <= (uint32_t)kFitHCap;
            S.winlo = inw ? wlo : 0xFFFFFFFFu;
            const uintptr_t sh = (uintptr_t)wlo * sizeof(float);
            S.px = inw ? reinterpret_cast<const float*>(reinterpret_cast<uintptr_t>(S.hx) - sh) : A.x;
            S.py = inw ? reinterpret_cast<const float*>(reinterpret_cast<uintptr_t>(S.hy) - sh) : A.y;
            S.pz = inw ? reinterpret_cast<const float*>(reinterpret_cast<uintptr_t>(S.hz) - sh) : A.z;
            S.sbase = sb;
            S.n = n;
            // tracks straight into their final slots when the caller asked for them and
            // the warp-batch's slot range fits its capacity (else into fit_g; the pack
            // kernel reports the overflow)
            const uint32_t tb = D.w[4], ns = D.w[5];
            const bool to_out = A.out.tracks != nullptr && sb != kSpilled &&
                                (uint64_t)tb + ns <= min(A.out.track_capacity, (uint64_t)kInFitG);
            S.td = to_out ? A.out.tracks + tb : A.fit_g + (sb == kSpilled ? 0u : sb);
            S.tcode = to_out ? tb : (kInFitG | (sb == kSpilled ? 0u : sb));
            S.nslot = to_out ? ns : 0u;
            S.offs[4 * nf] = hi;
            if (n) prefetch_bulk_l2(A.cand_g + sb, n * (uint32_t)sizeof(uint4));
            const uint32_t hb = inw ? (whi - wlo) * 4u : 0u, ob = nf * 16u;
            fence_proxy_async();
            mbar_arrive_expect_tx(&S.bar, 3u * hb + ob);
            bulk_g2s(S.offs, A.offsets + 4 * (size_t)f0, ob, &S.bar);
            if (hb) {
                bulk_g2s(S.hx, A.x + wlo, hb, &S.bar);
                bulk_g2s(S.hy, A.y + wlo, hb, &S.bar);
                bulk_g2s(S.hz, A.z + wlo, hb, &S.bar);
            }
        }
    }
    __syncwarp();   // D read, slot published
    fit_prefetch(A, D, b_next);
}

// T: one lane per frame of the consumed warp-batch in slot S
__device__ __forceinline__ void fit_frames(const KArgs& A, FitSlot& S) {
    const int lane = threadIdx.x & 31;
    const DevParams& P = A.P;
    cp_async_wait_all();   // S.selw
    __syncwarp();
    const bool active = (uint32_t)lane < S.nf && S.sbase != kSpilled;
    int c = 0, nneg = 0, npos = 0, reason = M3E_REASON_NONE;
    if (active) {
        c = S.cnt[lane];
        nneg = S.neg[lane];
        npos = S.pos[lane];
        reason = (int)(S.selw[lane] >> 16);
        if (reason == M3E_REASON_NONE && c > P.max_tracks) {
            reason = M3E_REASON_TRACK_OVERFLOW;
            nneg = 0;
        }
        A.fw[S.f0 + lane] = (uint32_t)min(c, P.max_tracks + 1) | ((uint32_t)min(nneg, 255) << 8) |
                            ((uint32_t)reason << 24);
    }
    // the frame's first output track: the warp-batch's first track + prefix of the
    // stored counts
    const uint32_t stored = active ? (uint32_t)min(c, P.max_tracks) : 0u;
    const uint32_t cs = S.tcode + warp_incl(stored) - stored;
    // the warp-batch's unused slots in out.tracks (its rejected candidates'): marked
#ifndef M3E_NO_MARK
    for (uint32_t k = S.nacc + (uint32_t)lane; k < S.nslot; k += 32) write_unused_slot(S.td + k);
#endif
    // frames for the vertex stage (Alg. 4 needs two e+ and one e-)
    const bool need = active && reason == M3E_REASON_NONE && npos >= 2 && nneg >= 1;
    const unsigned m = __ballot_sync(0xffffffffu, need);
    if (m) {
        uint32_t base = 0;
        if (lane == 0) base = atomicAdd(A.ticket + 9, (uint32_t)__popc(m));
        base = __shfl_sync(0xffffffffu, base, 0);
        if (need) A.vlist[base + __popc(m & ((1u << lane) - 1u))] = make_uint2(S.f0 + (uint32_t)lane, cs);
    }
}

// one stored candidate: the frame's hit arrays x/y/z (pointers to its first hit),
// its layer offsets `of` (of[4] = end), the hit offsets o0, o1, o2 inside the frame
template <bool kPairs>
__device__ __forceinline__ FitOut fit_entry(const DevParams& P, const float* x, const float* y, const float* z,
                                            const uint32_t* of, uint32_t o0, uint32_t o1, uint32_t o2) {
    Frame F;
    F.x = x;
    F.y = y;
    F.z = z;
    F.s[0] = 0;
    F.s[1] = (int)(of[1] - of[0]);
    F.s[2] = (int)(of[2] - of[0]);
    F.s[3] = (int)(of[3] - of[0]);
    F.n[0] = F.s[1];
    F.n[1] = F.s[2] - F.s[1];
    F.n[2] = F.s[3] - F.s[2];
    F.n[3] = (int)(of[4] - of[3]);
    const float3 h0 = make_float3(x[o0], y[o0], z[o0]);
    const float3 h1 = make_float3(x[o1], y[o1], z[o1]);
    const float3 h2 = make_float3(x[o2], y[o2], z[o2]);
    // r_tc of the selection (Eq. 5, same fp32 code as the selection's)
    const float2 dc = chords(h0, h1, h2);
    return fit_candidate_hd<kPairs>(P, F, h0, h1, h2, circle_radius_d(h0, h1, h2, dc), dc);
}
#ifndef M3E_FIT_WARPS
#define M3E_FIT_WARPS 8        // warps per CTA of the fit kernel
#endif
#ifndef M3E_FIT_MIN_BLOCKS
#define M3E_FIT_MIN_BLOCKS 3   // 80 registers (no spills), 24 warps per SM
#endif
constexpr int kFitWarps = M3E_FIT_WARPS;
template <bool BIG>   // BIG: calls of big frames (phase II), the layer-3 search one hit at a time
__global__ void __launch_bounds__(32 * kFitWarps, M3E_FIT_MIN_BLOCKS) fit_kernel(const __grid_constant__ KArgs A) {
    extern __shared__ __align__(16) uint8_t fit_smem_raw[];
    FitSlot* R = reinterpret_cast<FitSlot*>(fit_smem_raw) + 2 * (threadIdx.x >> 5);   // the warp's two slots
    FitPre& D = reinterpret_cast<FitPre*>(fit_smem_raw + 2 * kFitWarps * sizeof(FitSlot))[threadIdx.x >> 5];
    const int lane = threadIdx.x & 31;
    const unsigned lt = (1u << lane) - 1u;
    const DevParams& P = A.P;
    // warp-batches claimed with an atomic ticket, pipelined so that no claim or
    // descriptor load is waited for: `claim` (lane 0) is the warp-batch after next,
    // bq the next one, whose descriptor D is being fetched
    if (lane == 0) {
        mbar_init(&R[0].bar, 1);
        mbar_init(&R[1].bar, 1);
        fence_mbar_init();
    }
    uint32_t claim = 0;
    if (lane == 0) claim = atomicAdd(A.ticket + 8, 1u);
    uint32_t bq = __shfl_sync(0xffffffffu, claim, 0);
    fit_prefetch(A, D, bq);
    if (lane == 0) claim = atomicAdd(A.ticket + 8, 1u);
    auto refill = [&](FitSlot& S) {
        const uint32_t bn = __shfl_sync(0xffffffffu, claim, 0);
        fit_assign(A, S, D, bq, bn);
        bq = bn;
        if (lane == 0) claim = atomicAdd(A.ticket + 8, 1u);
    };
    refill(R[0]);
    refill(R[1]);
    uint32_t ph = 0u;      // mbarrier parity of slot s: bit s
    uint32_t ready = 0u;   // slot s loaded (waited): bit s
    int cur = 0;
    for (;;) {
        FitSlot& C = R[cur];
        FitSlot& X = R[cur ^ 1];
        if (C.b >= A.nbatch) break;   // claims are in order: X is past the end too
        if (!((ready >> cur) & 1u)) {
            mbar_wait(&C.bar, (ph >> cur) & 1u);
            ph ^= 1u << cur;
            ready |= 1u << cur;
        }
        const uint32_t left = C.n - C.t;
        const uint32_t xleft = X.n - X.t;
        // the chunk runs on into the next warp-batch when this one has < 32 left
        const bool useX = left < 32u && xleft > 0u;
        if (useX && !((ready >> (cur ^ 1)) & 1u)) {
            mbar_wait(&X.bar, (ph >> (cur ^ 1)) & 1u);
            ph ^= 1u << (cur ^ 1);
            ready |= 1u << (cur ^ 1);
        }
        __syncwarp();
        const bool inX = (uint32_t)lane >= left;
        const uint32_t idx = inX ? X.t + ((uint32_t)lane - left) : C.t + (uint32_t)lane;
        const bool valid = inX ? (useX && (uint32_t)lane - left < xleft) : true;
        FitSlot& L = inX ? X : C;
        int key = 64 + lane;   // slot | frame (invalid lanes: a key of their own)
        int j = 0;
        FitOut o;
        o.status = 7;
        o.hit3 = 0;
        uint4 e = make_uint4(0u, 0u, 0u, 0u);
        if (valid) {
            M3E_CHECK_IDX(L.sbase + idx < A.cand_cap && idx < L.n);
            e = A.cand_g[L.sbase + idx];
            j = (int)(e.y - L.f0);
            M3E_CHECK_IDX(j >= 0 && (uint32_t)j < L.nf);
            // a staged frame lies inside the slot's window
            M3E_CHECK_IDX(L.winlo == 0xFFFFFFFFu ||
                          (e.x >= L.winlo && e.x - L.winlo + (L.offs[4 * j + 4] - L.offs[4 * j]) <= (uint32_t)kFitHCap));
            key = (inX ? 16 : 0) + j;
            // the entry locates the triplet's hits: {first hit of the frame, frame,
            // offsets of h1 | h2 << 16, offset of h0} (inside the frame)
            const uint32_t* of = L.offs + 4 * j;
            const uint32_t o0 = e.w, o1 = e.z & 0xFFFFu, o2 = e.z >> 16;
            if constexpr (BIG) {
                // big frames (often past the window): per-slot generic base pointers
                o = fit_entry<false>(P, L.px + e.x, L.py + e.x, L.pz + e.x, of, o0, o1, o2);
            } else if (L.winlo != 0xFFFFFFFFu) {
                // staged frame: the slot's arrays indexed directly, so every hit load
                // is a shared-memory load with 32-bit addressing (LDS)
                const uint32_t d = e.x - L.winlo;
                o = fit_entry<true>(P, L.hx + d, L.hy + d, L.hz + d, of, o0, o1, o2);
            } else {   // (rare at phase I) a second inlined copy with global loads
                o = fit_entry<true>(P, A.x + e.x, A.y + e.x, A.z + e.x, of, o0, o1, o2);
            }
            e.z = (o1 - (of[1] - of[0])) | ((o2 - (of[2] - of[0])) << 16);   // layer-local h1 | h2
        }
        const bool acc = o.status == 0;
        // per-frame rank among accepted candidates (candidate order); the first
        // max_tracks are the frame's output tracks (R3)
        const unsigned grp = __match_any_sync(0xffffffffu, key);
        const unsigned ma = __ballot_sync(0xffffffffu, acc);
        const int before = valid ? L.cnt[j] : 0;
        const int rank = before + __popc(ma & grp & lt);
        const bool st = acc && rank < P.max_tracks;
        const unsigned ms = __ballot_sync(0xffffffffu, st);
        const unsigned mx = __ballot_sync(0xffffffffu, valid && inX);
        const unsigned mn = __ballot_sync(0xffffffffu, st && o.kappa < 0.0f);
        const unsigned mp = __ballot_sync(0xffffffffu, st && o.kappa > 0.0f);
        if (st) {   // the m3e_track record as two 16 B stores (the array is 16 B aligned)
            const uint4 w0 = make_uint4(e.y, (e.w & 0xFFFFu) | (e.z << 16), (e.z >> 16) | ((uint32_t)o.hit3 << 16),
                                        __float_as_uint(o.kappa));
            const uint4 w1 = make_uint4(__float_as_uint(o.chi2), __float_as_uint(o.cth01), __float_as_uint(o.cx),
                                        __float_as_uint(o.cy));
            M3E_CHECK_IDX(L.nslot == 0u || L.nacc + __popc(ms & (inX ? mx : ~mx) & lt) < L.nslot);
            uint4* d4 = reinterpret_cast<uint4*>(L.td + L.nacc + __popc(ms & (inX ? mx : ~mx) & lt));
            d4[0] = w0;
            d4[1] = w1;
        }
        __syncwarp();
        if (valid && lane == __ffs(grp) - 1) {
            L.cnt[j] = before + __popc(ma & grp);
            L.neg[j] += __popc(mn & grp);
            L.pos[j] += __popc(mp & grp);
        }
        if (lane == 0) {
            C.nacc += __popc(ms & ~mx);
            C.t += min(left, 32u);
            X.nacc += __popc(ms & mx);
            X.t += __popc(mx);
        }
        __syncwarp();
        if (C.t == C.n) {   // warp-batch consumed: its frames, then the slot takes the next one
            fit_frames(A, C);
            refill(C);
            ready &= ~(1u << cur);
            cur ^= 1;
        }
    }
}

// ------------------------------------------------------------- vertex kernels ----
// Split path, V for the frames the fit kernel's track stage listed (the output
// stage O is the pack kernel); results identical to the fused kernel's stage V.

// V, three kernels over the frames the track stage listed (Alg. 4,
// Sec. IV-C; same arithmetic and order as vertex_frame):
//   vertex_kernel  one warp per listed frame: its first max_tracks accepted tracks
//                  (candidate order), charge lists, phase 1 (energy window over
//                  (e+_a < e+_b, e-) in row-major order, ballot-compacted, capped
//                  at max_combs); the passing triples are appended to a global
//                  triple list (one atomicAdd per frame);
//   triple_kernel  phase 2, one THREAD per listed triple (dense lanes across
//                  frames: a frame has ~2 triples, so a lane per triple inside one
//                  frame's warp leaves most lanes idle);
//   vpost_kernel   one thread per listed frame: the passing triple with the
//                  smallest chi2 (earliest on ties) is the frame's vertex.
// A frame whose triples do not fit the list runs vertex_frame in place.
__device__ __forceinline__ const m3e_track* vtracks(const KArgs& A, uint32_t code) {
    return (code & kInFitG) ? A.fit_g + (code & ~kInFitG) : A.out.tracks + code;
}

struct VRes {
    double x, y, z, chi2, tdist, ptot;
    int pass, pad;
};

struct VertexSmem {
    DevParams P;                          // for the out-of-line routines
    uint32_t ent[kWarps][2][kMaxTracksCap];   // charge lists: store offset | track index << 16
    double en[kWarps][2][kMaxTracksCap];      // their energies
    uint2 cmb[kWarps][kMaxCombsCap];          // passing triples: {offsets a | b << 10 | e << 20, a | b << 8 | e << 16}
};

#ifndef M3E_VERTEX_MIN_BLOCKS
#define M3E_VERTEX_MIN_BLOCKS 4
#endif
__global__ void __launch_bounds__(kThreads, M3E_VERTEX_MIN_BLOCKS) vertex_kernel(const __grid_constant__ KArgs A) {
    extern __shared__ __align__(16) uint8_t vsm_raw[];
    VertexSmem& S = *reinterpret_cast<VertexSmem*>(vsm_raw);
    const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
    const unsigned lt_mask = (1u << lane) - 1u;
    if (tid == 0) S.P = A.P;
    __syncthreads();
    const DevParams& P = A.P;
    const size_t gwarp = (size_t)blockIdx.x * kWarps + warp;
    const uint32_t n = *reinterpret_cast<const volatile uint32_t*>(A.ticket + 9);
    uint32_t* ep = S.ent[warp][0];
    uint32_t* en_ = S.ent[warp][1];
    double* Ep = S.en[warp][0];
    double* En = S.en[warp][1];
    uint2* cmb = S.cmb[warp];
    for (uint32_t k = (uint32_t)gwarp; k < n; k += gridDim.x * kWarps) {
        const uint2 e = A.vlist[k];
        const uint32_t f = e.x;
        // the frame's output tracks, contiguous from e.y (fit kernel)
        const m3e_track* ft = vtracks(A, e.y);
        const uint32_t nj = min(A.fw[f] & 0xFFu, (uint32_t)P.max_tracks);
        // accepted tracks (track index = rank among the frame's accepted entries,
        // the first max_tracks only) split by charge, in track order
        int nt = 0, npos = 0, nneg = 0;
        for (uint32_t k0 = 0; k0 < nj && nt < P.max_tracks; k0 += 32) {
            const uint32_t c = k0 + lane;
            float kap = 0.0f;
            bool acc = false;
            if (c < nj) {
                M3E_CHECK_IDX((e.y & kInFitG) ? (e.y & ~kInFitG) + c < A.cand_cap
                                              : (uint64_t)e.y + c < A.out.track_capacity);
                acc = true;
                kap = ft[c].kappa;
            }
            const unsigned m = __ballot_sync(0xffffffffu, acc);
            const int ti = nt + __popc(m & lt_mask);
            acc = acc && ti < P.max_tracks;
            const bool ispos = acc && kap > 0.0f, isneg = acc && kap < 0.0f;
            const unsigned mp = __ballot_sync(0xffffffffu, ispos);
            const unsigned mn = __ballot_sync(0xffffffffu, isneg);
            const uint32_t code = c | ((uint32_t)ti << 16);
            if (ispos) {
                const int p = npos + __popc(mp & lt_mask);
                ep[p] = code;
                Ep[p] = track_energy(P, kap);
            }
            if (isneg) {
                const int p = nneg + __popc(mn & lt_mask);
                en_[p] = code;
                En[p] = track_energy(P, kap);
            }
            nt += __popc(m);
            npos += __popc(mp);
            nneg += __popc(mn);
        }
        __syncwarp();
        // Alg. 4 phase 1 (the track stage listed the frame: npos >= 2, nneg >= 1)
        const int tot = npos * npos * nneg;
        int ncomb = 0;
        for (int base = 0; base < tot; base += 32) {
            const int t = base + lane;
            bool pass = false;
            uint2 cc = make_uint2(0u, 0u);
            if (t < tot) {
                const int ia = t / (npos * nneg), rem = t - ia * npos * nneg;
                const int ib = rem / nneg, ie = rem - ib * nneg;
                if (ia < ib) {
                    const double dE = Ep[ia] + Ep[ib] + En[ie] - kMuMass;
                    pass = fabs(dE) <= P.e_window;
                    const uint32_t a = ep[ia], bb = ep[ib], ee = en_[ie];
                    cc = make_uint2((a & 0xFFFFu) | ((bb & 0xFFFFu) << 10) | ((ee & 0xFFFFu) << 20),
                                    (a >> 16) | ((bb >> 16) << 8) | ((ee >> 16) << 16));
                }
            }
            const unsigned m = __ballot_sync(0xffffffffu, pass);
            const int pos = ncomb + __popc(m & lt_mask);
            if (pass && pos < P.max_combs) cmb[pos] = cc;
            ncomb += __popc(m);
            if (ncomb > P.max_combs) break;
        }
        __syncwarp();
        uint32_t tb = 0;
        bool inplace = false;
        if (ncomb > P.max_combs) {
            ncomb = P.max_combs + 1;
        } else if (ncomb > 0) {
            if (lane == 0) tb = atomicAdd(A.ticket + 11, (uint32_t)ncomb);
            tb = __shfl_sync(0xffffffffu, tb, 0);
            inplace = tb + (uint32_t)ncomb > A.tri_cap;
            if (!inplace)
                for (int c = lane; c < ncomb; c += 32) A.tri[tb + c] = make_uint4(k, cmb[c].x, cmb[c].y, 0u);
        }
        int reason = ncomb > P.max_combs ? M3E_REASON_COMB_OVERFLOW : M3E_REASON_NONE;
        if (inplace) {   // triple list full: the whole vertex selection of this frame here
            VScratch& V = reinterpret_cast<VScratch*>(A.vscratch)[gwarp];
            m3e_track* pool = A.pool_trk + gwarp * A.trk_stride;
            int m_ = 0;
            for (uint32_t k0 = 0; k0 < nj; k0 += 32) {
                const uint32_t c = k0 + lane;
                const bool acc = c < nj;
                const unsigned m = __ballot_sync(0xffffffffu, acc);
                const int p = m_ + __popc(m & lt_mask);
                if (acc && p < P.max_tracks) pool[p] = ft[c];
                m_ += __popc(m);
            }
            __syncwarp();
            Frame Fv;
            const uint4 o4 = *reinterpret_cast<const uint4*>(A.offsets + 4 * (size_t)f);
            const uint32_t o5 = A.offsets[4 * (size_t)f + 4];
            Fv.x = A.x + o4.x;
            Fv.y = A.y + o4.x;
            Fv.z = A.z + o4.x;
            Fv.s[0] = 0;
            Fv.s[1] = (int)(o4.y - o4.x);
            Fv.s[2] = (int)(o4.z - o4.x);
            Fv.s[3] = (int)(o4.w - o4.x);
            Fv.n[0] = Fv.s[1];
            Fv.n[1] = (int)(o4.z - o4.y);
            Fv.n[2] = (int)(o4.w - o4.z);
            Fv.n[3] = (int)(o5 - o4.w);
            const VOut r = vertex_frame(&S.P, V, min(m_, P.max_tracks), pool, Fv, f, A.vrec + k);
            reason = r.ncomb > P.max_combs ? M3E_REASON_COMB_OVERFLOW : (r.vtx ? M3E_REASON_VERTEX : M3E_REASON_NONE);
        }
        if (lane == 0) {
            A.fw[f] = (A.fw[f] & 0xFFu) | ((uint32_t)min(nneg, 255) << 8) | ((uint32_t)ncomb << 16) |
                      ((uint32_t)reason << 24);
            if (reason == M3E_REASON_VERTEX) A.vk[f] = k;
            // triples for phase 2 (count 0: none; in place: already decided)
            A.vtr[k] = make_uint2(tb, (reason == M3E_REASON_NONE && !inplace) ? (uint32_t)ncomb : 0u);
        }
        __syncwarp();
    }
}

// phase 2: one thread per listed triple
#ifndef M3E_TRIPLE_MIN_BLOCKS
#define M3E_TRIPLE_MIN_BLOCKS 3   // 80 registers: occupancy beats the spills (measured 1 / 2 / 3: 0.74 / 0.58 / 0.52 ms vertex stage)
#endif
__global__ void __launch_bounds__(kThreads, M3E_TRIPLE_MIN_BLOCKS) triple_kernel(const __grid_constant__ KArgs A) {
    __shared__ DevParams SP;
    if (threadIdx.x == 0) SP = A.P;
    __syncthreads();
    const uint32_t n0 = *reinterpret_cast<const volatile uint32_t*>(A.ticket + 11);
    const uint32_t n = n0 < A.tri_cap ? n0 : (uint32_t)A.tri_cap;
    for (uint32_t t = blockIdx.x * kThreads + threadIdx.x; t < n; t += gridDim.x * kThreads) {
        const uint4 e = A.tri[t];
        if (e.x >= *reinterpret_cast<const volatile uint32_t*>(A.ticket + 9)) continue;   // never (guard)
        const uint2 v = A.vlist[e.x];
        const uint32_t g0 = A.offsets[4 * (size_t)v.x];
        Frame Fv;
        Fv.x = A.x + g0;
        Fv.y = A.y + g0;
        Fv.z = A.z + g0;
        Fv.s[0] = 0;
        const m3e_track* ft = vtracks(A, v.y);
        const VTrk T0 = make_vtrk(SP, ft[e.y & 1023u], Fv);
        const VTrk T1 = make_vtrk(SP, ft[(e.y >> 10) & 1023u], Fv);
        const VTrk T2 = make_vtrk(SP, ft[(e.y >> 20) & 1023u], Fv);
        const VResult r = vertex_triple_inl(SP, T0, T1, T2);
        VRes o;
        o.x = r.x; o.y = r.y; o.z = r.z;
        o.chi2 = r.chi2;
        o.tdist = r.tdist;
        o.ptot = r.ptot;
        o.pass = r.pass;
        o.pad = 0;
        A.tres[t] = o;
    }
}

// phase 3: one thread per listed frame
__global__ void __launch_bounds__(kThreads) vpost_kernel(const __grid_constant__ KArgs A) {
    const uint32_t n = *reinterpret_cast<const volatile uint32_t*>(A.ticket + 9);
    for (uint32_t k = blockIdx.x * kThreads + threadIdx.x; k < n; k += gridDim.x * kThreads) {
        const uint2 r = A.vtr[k];
        if (r.y == 0u) continue;
        double bchi = 1e300;
        uint32_t bi = 0xFFFFFFFFu;
        for (uint32_t t = r.x; t < r.x + r.y; ++t) {
            const VRes& o = A.tres[t];
            if (o.pass && o.chi2 < bchi) { bchi = o.chi2; bi = t; }
        }
        if (bi == 0xFFFFFFFFu) continue;
        const uint32_t f = A.vlist[k].x;
        const VRes o = A.tres[bi];
        const uint32_t code = A.tri[bi].z;
        m3e_vertex v;
        v.frame = f;
        v.track[0] = (uint16_t)(code & 255u);
        v.track[1] = (uint16_t)((code >> 8) & 255u);
        v.track[2] = (uint16_t)((code >> 16) & 255u);
        v.pad = 0;
        v.pad2 = 0;
        v.x = o.x; v.y = o.y; v.z = o.z;
        v.chi2 = o.chi2;
        v.target_dist = (float)o.tdist;
        v.p_total = (float)o.ptot;
        A.vrec[k] = v;
        A.fw[f] = (A.fw[f] & 0x00FFFFFFu) | ((uint32_t)M3E_REASON_VERTEX << 24);
        A.vk[f] = k;
    }
}

// host path: add the chunk's bases to its device outputs before they are copied
__global__ void rebase_kernel(const Rebase r) {
    const uint64_t stride = (uint64_t)gridDim.x * blockDim.x;
    const uint64_t i0 = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (r.frames)
        for (uint64_t i = i0; i < r.n_frames; i += stride) {
            m3e_frame_out& fo = r.frames[i];
            fo.track_first += r.base_trk;
            if (fo.kept_index != 0xFFFFFFFFu) fo.kept_index += r.base_kept;
        }
    if (r.tracks)
        for (uint64_t i = i0; i < r.n_tracks; i += stride)
            if (r.tracks[i].frame != 0xFFFFFFFFu) r.tracks[i].frame += r.frame0;   // (unused slots stay marked)
    for (uint64_t i = i0; i < r.n_kept; i += stride) {
        if (r.kept_frame) r.kept_frame[i] += r.frame0;
        if (r.kept_offsets)
            for (int l = 0; l < 4; ++l) r.kept_offsets[4 * i + l] += r.base_hits;
        if (r.vertices && r.vertices[i].frame != 0xFFFFFFFFu) r.vertices[i].frame += r.frame0;
    }
}

cudaError_t launch_rebase(const Rebase& r, int sms, cudaStream_t s) {
    rebase_kernel<<<sms * 4, kThreads, 0, s>>>(r);
    return cudaGetLastError();
}

cudaError_t launch_vertex(const KArgs& a, int grid, int sms, cudaStream_t s) {
    const size_t smem = sizeof(VertexSmem);
    cudaError_t e = cudaFuncSetAttribute(vertex_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    if (e != cudaSuccess) return e;
    vertex_kernel<<<grid, kThreads, smem, s>>>(a);
    if ((e = cudaGetLastError()) != cudaSuccess) return e;
    triple_kernel<<<sms * triple_blocks_per_sm(), kThreads, 0, s>>>(a);
    if ((e = cudaGetLastError()) != cudaSuccess) return e;
    vpost_kernel<<<sms * 2, kThreads, 0, s>>>(a);
    return cudaGetLastError();
}

int triple_blocks_per_sm() {
    int n = 0;
    if (cudaOccupancyMaxActiveBlocksPerMultiprocessor(&n, triple_kernel, kThreads, 0) != cudaSuccess) return 1;
    return n > 0 ? n : 1;
}

int vertex_blocks_per_sm() {
    int n = 0;
    const size_t smem = sizeof(VertexSmem);
    if (cudaFuncSetAttribute(vertex_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem) != cudaSuccess)
        return 1;
    if (cudaOccupancyMaxActiveBlocksPerMultiprocessor(&n, vertex_kernel, kThreads, smem) != cudaSuccess) return 1;
    return n > 0 ? n : 1;
}


template <bool BIG>
static cudaError_t launch_fit_t(const KArgs& a, int grid, cudaStream_t s) {
    const size_t smem = 2 * kFitWarps * sizeof(FitSlot) + kFitWarps * sizeof(FitPre);
    cudaError_t e = cudaFuncSetAttribute(fit_kernel<BIG>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    if (e != cudaSuccess) return e;
    fit_kernel<BIG><<<grid, 32 * kFitWarps, smem, s>>>(a);
    return cudaGetLastError();
}

cudaError_t launch_fit(const KArgs& a, bool big, int grid, cudaStream_t s) {
    return big ? launch_fit_t<true>(a, grid, s) : launch_fit_t<false>(a, grid, s);
}

int fit_blocks_per_sm() {
    int n = 0;
    const size_t smem = 2 * kFitWarps * sizeof(FitSlot) + kFitWarps * sizeof(FitPre);
    if (cudaFuncSetAttribute(fit_kernel<false>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem) != cudaSuccess)
        return 1;
    if (cudaOccupancyMaxActiveBlocksPerMultiprocessor(&n, fit_kernel<false>, 32 * kFitWarps, smem) != cudaSuccess)
        return 1;
    return n > 0 ? n : 1;
}

cudaError_t launch_pack(const KArgs& a, int grid, cudaStream_t s) {
    const size_t smem = sizeof(PackSmem);
    cudaError_t e = cudaFuncSetAttribute(pack_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    if (e != cudaSuccess) return e;
    pack_kernel<<<grid, kThreads, smem, s>>>(a);
    return cudaGetLastError();
}

template <int MODE, bool BIG>
static cudaError_t launch_mode(const KArgs& a, int grid, cudaStream_t s) {
    const size_t smem = smem_bytes();
    cudaError_t e =
        cudaFuncSetAttribute(filter_kernel<MODE, BIG>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    if (e != cudaSuccess) return e;
    filter_kernel<MODE, BIG><<<grid, kThreads, smem, s>>>(a);
    return cudaGetLastError();
}

cudaError_t launch_filter(int mode, bool big, const KArgs& a, int grid, cudaStream_t s) {
    switch (mode) {
        case kModeFull: return big ? launch_mode<kModeFull, true>(a, grid, s) : launch_mode<kModeFull, false>(a, grid, s);
        case kModeSelect:
            return big ? launch_mode<kModeSelect, true>(a, grid, s) : launch_mode<kModeSelect, false>(a, grid, s);
        case kModeSelectC:
            return big ? launch_mode<kModeSelectC, true>(a, grid, s) : launch_mode<kModeSelectC, false>(a, grid, s);
        case kModeFit: return launch_mode<kModeFit, false>(a, grid, s);
        case kModeVertex: return launch_mode<kModeVertex, false>(a, grid, s);
        case kModePack: return launch_mode<kModePack, false>(a, grid, s);
    }
    return cudaErrorInvalidValue;
}


template <int MODE, bool BIG>
static int occupancy() {
    int n = 0;
    const size_t smem = smem_bytes();
    if (cudaFuncSetAttribute(filter_kernel<MODE, BIG>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem) !=
        cudaSuccess)
        return 1;
    if (cudaOccupancyMaxActiveBlocksPerMultiprocessor(&n, filter_kernel<MODE, BIG>, kThreads, smem) != cudaSuccess)
        return 1;
    return n > 0 ? n : 1;
}

int blocks_per_sm(int mode, bool big) {
    switch (mode) {
        case kModeFull: return big ? occupancy<kModeFull, true>() : occupancy<kModeFull, false>();
        case kModeSelect: return big ? occupancy<kModeSelect, true>() : occupancy<kModeSelect, false>();
        case kModeSelectC: return big ? occupancy<kModeSelectC, true>() : occupancy<kModeSelectC, false>();
        case kModeFit: return occupancy<kModeFit, false>();
        case kModeVertex: return occupancy<kModeVertex, false>();
        case kModePack: return occupancy<kModePack, false>();
    }
    return 1;
}

}  // namespace m3e

static_assert(sizeof(m3e::VScratch) <= m3e::kVScratchBytes, "kVScratchBytes too small");
static_assert(sizeof(m3e::VRes) == m3e::kVResBytes, "kVResBytes");
