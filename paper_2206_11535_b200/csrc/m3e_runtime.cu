// m3e_runtime.cu -- C ABI of libm3e.so (include/m3e.h): context and workspace
// management, parameter validation, the device-buffer entry points, and the
// host-buffer path that streams chunks host->device on two CUDA streams so the
// copy of chunk c+1 overlaps the filter of chunk c (Sec. V-A/V-B:
// "one chunk to be transferred to and processed by the GPU, while the next one
// is filled"; "CUDA streams are used").
#include <algorithm>
#include <cmath>
#include <cstdlib>
#include <cstdio>
#include <cstring>
#include <string>
#include <vector>

#include <cuda_runtime.h>

#include "m3e.h"
#include "m3e_device.cuh"
#include "m3e_kernels.h"

using namespace m3e;

namespace {

thread_local std::string g_err = "no error";

int fail(int code, const std::string& msg) {
    g_err = msg;
    return code;
}
int cuda_fail(cudaError_t e, const char* what) {
    g_err = std::string(what) + ": " + cudaGetErrorString(e);
    return M3E_ERR_CUDA;
}
#define CK(call)                                          \
    do {                                                  \
        cudaError_t e_ = (call);                          \
        if (e_ != cudaSuccess) return cuda_fail(e_, #call); \
    } while (0)

// one independent set of device workspace (a CUDA stream's worth)
struct Workspace {
    uint32_t* ticket = nullptr;
    uint4* status = nullptr;
    size_t status_n = 0;
    uint32_t* pool_idx = nullptr;
    float* pool_rt = nullptr;
    m3e_fit_record* pool_rec = nullptr;
    m3e_track* pool_trk = nullptr;
    size_t pool_stride = 0, trk_stride = 0;
    int pool_ctas = 0;
    uint32_t epoch = 0;
    BatchStat* bstat = nullptr;
    size_t bstat_n = 0;
    m3e_track* stage_trk = nullptr;
    size_t stage_trk_n = 0;
    KeptRec* stage_kept = nullptr;
    size_t stage_kept_n = 0;
    uint4* kept_rec = nullptr;          // kept-frame list (pack -> kept kernel)
    uint32_t* pair_scratch = nullptr;   // big-frame selection lists, kPairWords per warp
    int pair_warps = 0;
    void* vscratch = nullptr;           // vertex-stage scratch, kVScratchBytes per warp
    uint4* cand_g = nullptr;            // candidate store of the split path
    m3e_track* fit_g = nullptr;         // output tracks, compacted per store segment (fit kernel)
    size_t cand_n = 0;
    uint32_t* sel = nullptr;            // per-frame selection words of the split path
    uint32_t* fw = nullptr;             // per-frame track/vertex words of the split path
    uint32_t* vk = nullptr;             // per-frame vertex list position
    uint2* vlist = nullptr;             // frames for the vertex stage
    m3e_vertex* vrec = nullptr;         // their vertices
    uint2* vtr = nullptr;               // their triple ranges
    uint4* tri = nullptr;               // listed e+e+e- triples
    void* tres = nullptr;               // their phase-2 results
    size_t tri_n = 0;
    size_t sel_n = 0;
    uint32_t* bsel = nullptr;           // per-warp-batch store offsets of the split path
    uint32_t* bcnt = nullptr;           // per-warp-batch store entries
    uint32_t* spill = nullptr;          // warp-batches the store could not take
    uint32_t* bslot = nullptr;          // per-warp-batch output track slots
    uint32_t* tbase = nullptr;          // ... and its first slot (slot scan)
    size_t bsel_n = 0;
    uint2* sstatus = nullptr;           // slot-scan look-back words, one per scan tile
    size_t sstatus_n = 0;
    bool sstatus_fresh = false;
    bool status_fresh = false;          // status words allocated, not yet zeroed
    size_t bytes = 0;
};

// device staging of one chunk for m3e_filter_host
struct Chunk {
    float *x = nullptr, *y = nullptr, *z = nullptr;
    uint32_t* offsets = nullptr;
    uint8_t* reason = nullptr;
    m3e_frame_out* frames = nullptr;
    m3e_track* tracks = nullptr;
    m3e_vertex* vertices = nullptr;
    uint32_t* kept_frame = nullptr;
    uint32_t* kept_offsets = nullptr;
    float *kx = nullptr, *ky = nullptr, *kz = nullptr;
    m3e_summary* summary = nullptr;      // device
    m3e_summary* h_summary = nullptr;    // pinned host
    uint64_t cap_frames = 0, cap_hits = 0, cap_tracks = 0;
    cudaEvent_t ev_summary = nullptr, ev_free = nullptr;
    bool used = false;
};

}  // namespace

constexpr int kNEv = 7;   // timing events per m3e_filter call (6 kernel intervals)

struct m3e_context {
    int device = 0;
    int sms = 148;
    uint64_t max_frames = 0, max_hits = 0;
    Workspace ws[2];
    cudaStream_t st[2] = {nullptr, nullptr};
    Chunk ch[2];
    uint64_t chunk_frames = 0;
    bool timing = false;
    bool split = true;              // two-kernel production path (M3E_FUSED=1 in the environment: one kernel)
    uint64_t cand_per_frame = 16;   // candidate-store entries per frame (M3E_CAND_STORE; tests force spills)
    uint64_t tri_cap = 0;           // vertex-stage triple list entries (M3E_TRI_CAP; 0: one per frame)
    std::vector<cudaEvent_t> tev;   // kNEv events per timed m3e_filter call
    size_t tev_used = 0;
    size_t tev_split = 0;           // timed calls that ran the split path
};

namespace {

void free_ws(Workspace& w) {
    cudaFree(w.cand_g);
    cudaFree(w.fit_g);
    cudaFree(w.sel);
    cudaFree(w.fw);
    cudaFree(w.vk);
    cudaFree(w.vlist);
    cudaFree(w.vrec);
    cudaFree(w.vtr);
    cudaFree(w.tri);
    cudaFree(w.tres);
    cudaFree(w.bsel);
    cudaFree(w.bcnt);
    cudaFree(w.spill);
    cudaFree(w.bslot);
    cudaFree(w.tbase);
    cudaFree(w.sstatus);
    cudaFree(w.pair_scratch);
    cudaFree(w.vscratch);
    cudaFree(w.bstat);
    cudaFree(w.stage_trk);
    cudaFree(w.stage_kept);
    cudaFree(w.kept_rec);
    cudaFree(w.ticket);
    cudaFree(w.status);
    cudaFree(w.pool_idx);
    cudaFree(w.pool_rt);
    cudaFree(w.pool_rec);
    cudaFree(w.pool_trk);
    w = Workspace{};
}

void free_chunk(Chunk& c) {
    cudaFree(c.x); cudaFree(c.y); cudaFree(c.z); cudaFree(c.offsets);
    cudaFree(c.reason); cudaFree(c.frames); cudaFree(c.tracks); cudaFree(c.vertices);
    cudaFree(c.kept_frame); cudaFree(c.kept_offsets); cudaFree(c.kx); cudaFree(c.ky); cudaFree(c.kz);
    cudaFree(c.summary);
    if (c.h_summary) cudaFreeHost(c.h_summary);
    if (c.ev_summary) cudaEventDestroy(c.ev_summary);
    if (c.ev_free) cudaEventDestroy(c.ev_free);
    c = Chunk{};
}

int validate(const m3e_params* p) {
    if (!p) return fail(M3E_ERR_INVALID_ARGUMENT, "params is NULL");
    for (int l = 0; l < 4; ++l)
        if (!(p->layer_r[l] > 0) || (l && !(p->layer_r[l] > p->layer_r[l - 1])))
            return fail(M3E_ERR_INVALID_ARGUMENT, "layer_r must be positive and increasing");
    if (!(p->b_field > 0)) return fail(M3E_ERR_INVALID_ARGUMENT, "b_field must be > 0");
    if (p->cuts_max < 1 || p->cuts_max > kMaxCutsCap)
        return fail(M3E_ERR_INVALID_ARGUMENT, "cuts_max must be in [1, 1023]");
    if (p->max_tracks < 1 || p->max_tracks > kMaxTracksCap)
        return fail(M3E_ERR_INVALID_ARGUMENT, "max_tracks must be in [1, 128]");
    if (p->max_combs < 0 || p->max_combs + 1 > kMaxCombsCap)
        return fail(M3E_ERR_INVALID_ARGUMENT, "max_combs must be in [0, 127]");
    if (!(p->x_over_x0 > 0)) return fail(M3E_ERR_INVALID_ARGUMENT, "x_over_x0 must be > 0");
    if (!(p->target_r > 0) || !(p->target_half > 0))
        return fail(M3E_ERR_INVALID_ARGUMENT, "target dimensions must be > 0");
    return M3E_OK;
}

DevParams make_dev_params(const m3e_params* p) {
    DevParams d;
    for (int l = 0; l < 4; ++l) d.R[l] = (float)p->layer_r[l];
    d.inv_dr01 = (float)(1.0 / (p->layer_r[1] - p->layer_r[0]));
    d.inv_dr12 = (float)(1.0 / (p->layer_r[2] - p->layer_r[1]));
    d.inv_r0r1 = (float)(1.0 / (p->layer_r[0] * p->layer_r[1]));
    d.inv_r1r2 = (float)(1.0 / (p->layer_r[1] * p->layer_r[2]));
    d.dl_max = (float)p->dlambda_max;
    d.c01_min = (float)p->cos_phi01_min;
    d.c12_min = (float)p->cos_phi12_min;
    d.rt_min = (float)p->rt_min;
    d.rt_max = (float)p->rt_max;
    d.rt_min2 = d.rt_min * d.rt_min;
    d.rt_max2 = d.rt_max * d.rt_max;
    const double X = p->x_over_x0;
    // Highland (R7): sigma = 13.6 MeV / p * sqrt(X) (1 + 0.038 ln X), p = PT_CONV B / k
    const double chl = 13.6 * std::sqrt(X) * (1.0 + 0.038 * std::log(X)) / (kPtConv * p->b_field);
    d.chl = (float)chl;
    d.chi2_max = (float)p->chi2_max;
    d.R3sq = (float)(p->layer_r[3] * p->layer_r[3]);
    d.cuts_max = p->cuts_max;
    d.max_tracks = p->max_tracks;
    d.max_combs = p->max_combs;
    d.ptb = kPtConv * p->b_field;
    d.chl_d = chl;
    d.e_window = p->e_window;
    d.rlim = p->target_r + p->xy_margin;
    d.sig_pix2 = p->sigma_pixel * p->sigma_pixel;
    d.chi2v_max = p->chi2_vertex_max;
    d.tdist_max = p->target_dist_max;
    d.ptot_max = p->p_total_max;
    d.target_r = p->target_r;
    d.target_half = p->target_half;
    return d;
}

// frames per warp-batch: keep a batch's hits within the shared-memory window
#ifndef M3E_FB_SLACK
#define M3E_FB_SLACK 1.3   // frames per warp-batch = window / (slack x mean hits): measured 1.0 / 1.15 / 1.3 -> 12.81 / 12.58 / 12.48 ms
#endif
int choose_fb(uint64_t F, uint64_t H) {
    if (F == 0) return kFB;
    const double mean = (double)H / (double)F;
    int fb = (int)((double)kHCap / (M3E_FB_SLACK * std::max(mean, 1.0)));
    return std::max(1, std::min(kFB, fb));
}

int ensure_ws(m3e_context* c, Workspace& w, uint64_t nbatch, const m3e_params* p, int fb, int ctas) {
    if (!w.ticket) {
        CK(cudaMalloc(&w.ticket, 16 * sizeof(uint32_t)));
        w.bytes += 16 * sizeof(uint32_t);
    }
    const uint64_t ntiles = (nbatch + kPackTile - 1) / kPackTile;
    if (w.bstat_n < nbatch) {
        cudaFree(w.bstat);
        w.bytes -= w.bstat_n * sizeof(BatchStat);
        const size_t n = std::max<size_t>(nbatch, 4096);
        CK(cudaMalloc(&w.bstat, n * sizeof(BatchStat)));
        w.bstat_n = n;
        w.bytes += n * sizeof(BatchStat);
    }
    if (w.status_n < ntiles) {
        cudaFree(w.status);
        w.bytes -= w.status_n * sizeof(uint4);
        const size_t n = std::max<size_t>(ntiles, 1024);
        CK(cudaMalloc(&w.status, n * sizeof(uint4)));
        w.status_n = n;
        w.status_fresh = true;   // zeroed on the launch stream before its first use (run_mode)
        w.bytes += n * sizeof(uint4);
        w.epoch = 0;
        w.sstatus_fresh = true;   // epochs restart: no stale slot-scan tag may match either
    }
    const size_t ps = (size_t)fb * p->cuts_max, ts = (size_t)fb * p->max_tracks;
    if (w.pool_ctas < ctas || w.pool_stride < ps || w.trk_stride < ts) {
        w.bytes -= w.pool_ctas ? (size_t)w.pool_ctas * kWarps *
                                     (w.pool_stride * (sizeof(uint32_t) + sizeof(float) + sizeof(m3e_fit_record)) +
                                      w.trk_stride * sizeof(m3e_track))
                               : 0;
        cudaFree(w.pool_idx); cudaFree(w.pool_rt); cudaFree(w.pool_rec); cudaFree(w.pool_trk);
        const size_t PS = std::max(ps, (size_t)kFB * 768), TS = std::max(ts, (size_t)kFB * 64);
        const int n = std::max(ctas, w.pool_ctas) * kWarps;   // per warp
        CK(cudaMalloc(&w.pool_idx, PS * n * sizeof(uint32_t)));
        CK(cudaMalloc(&w.pool_rt, PS * n * sizeof(float)));
        CK(cudaMalloc(&w.pool_rec, PS * n * sizeof(m3e_fit_record)));
        CK(cudaMalloc(&w.pool_trk, TS * n * sizeof(m3e_track)));
        w.pool_stride = PS;
        w.trk_stride = TS;
        w.pool_ctas = n / kWarps;
        w.bytes += PS * n * (sizeof(uint32_t) + sizeof(float) + sizeof(m3e_fit_record)) + TS * n * sizeof(m3e_track);
    }
    if (w.pair_warps < ctas * kWarps) {
        cudaFree(w.pair_scratch);
        cudaFree(w.vscratch);
        w.bytes -= (size_t)w.pair_warps * (kPairWords * sizeof(uint32_t) + kVScratchBytes);
        w.pair_warps = ctas * kWarps;
        CK(cudaMalloc(&w.pair_scratch, (size_t)w.pair_warps * kPairWords * sizeof(uint32_t)));
        CK(cudaMalloc(&w.vscratch, (size_t)w.pair_warps * kVScratchBytes));
        w.bytes += (size_t)w.pair_warps * (kPairWords * sizeof(uint32_t) + kVScratchBytes);
    }
    (void)c;
    return M3E_OK;
}

// split path: candidate store (kCandPerFrame entries per frame; warp-batches
// that do not fit are flagged and re-selected by the filter kernel), per-frame
// selection words and per-warp-batch store offsets
constexpr uint64_t kCandPerFrame = 16;
int ensure_split(Workspace& w, uint64_t F, uint64_t nbatch, uint64_t per_frame, uint64_t tri_per_frame) {
    // (capped at 2^30 entries, 53 GB: warp-batches past it are re-selected by the fused kernel)
    const uint64_t nc = std::min<uint64_t>(std::max<uint64_t>(per_frame * F, 1u << 10), 1ull << 30);
    if (w.cand_n < nc) {
        cudaFree(w.cand_g);
        cudaFree(w.fit_g);
        w.bytes -= w.cand_n * (sizeof(uint4) + sizeof(m3e_track));
        w.cand_n = 0;
        CK(cudaMalloc(&w.cand_g, nc * sizeof(uint4)));
        CK(cudaMalloc(&w.fit_g, nc * sizeof(m3e_track)));
        w.cand_n = nc;
        w.bytes += nc * (sizeof(uint4) + sizeof(m3e_track));
    }
    if (w.sel_n < F) {
        constexpr size_t per = 3 * sizeof(uint32_t) + 2 * sizeof(uint2) + sizeof(m3e_vertex);
        cudaFree(w.sel); cudaFree(w.fw); cudaFree(w.vk); cudaFree(w.vlist); cudaFree(w.vrec); cudaFree(w.vtr);
        w.bytes -= w.sel_n * per;
        w.sel_n = 0;
        CK(cudaMalloc(&w.sel, F * sizeof(uint32_t)));
        CK(cudaMalloc(&w.fw, F * sizeof(uint32_t)));
        CK(cudaMalloc(&w.vk, F * sizeof(uint32_t)));
        CK(cudaMalloc(&w.vlist, F * sizeof(uint2)));
        CK(cudaMalloc(&w.vrec, F * sizeof(m3e_vertex)));
        CK(cudaMalloc(&w.vtr, F * sizeof(uint2)));
        w.sel_n = F;
        w.bytes += F * per;
    }
    // e+e+e- triples of the vertex stage: one per frame on average (phase I: ~0.04);
    // frames whose triples do not fit run the vertex selection in place
    const uint64_t nt = std::min<uint64_t>(std::max<uint64_t>(tri_per_frame * F, 4096), 1ull << 28);
    if (w.tri_n < nt) {
        cudaFree(w.tri); cudaFree(w.tres);
        w.bytes -= w.tri_n * (sizeof(uint4) + kVResBytes);
        w.tri_n = 0;
        CK(cudaMalloc(&w.tri, nt * sizeof(uint4)));
        CK(cudaMalloc(&w.tres, nt * kVResBytes));
        w.tri_n = nt;
        w.bytes += nt * (sizeof(uint4) + kVResBytes);
    }
    if (w.bsel_n < nbatch) {
        cudaFree(w.bsel);
        cudaFree(w.bcnt);
        cudaFree(w.spill);
        cudaFree(w.bslot);
        cudaFree(w.tbase);
        w.bytes -= 5 * w.bsel_n * sizeof(uint32_t);
        w.bsel_n = 0;
        CK(cudaMalloc(&w.bsel, nbatch * sizeof(uint32_t)));
        CK(cudaMalloc(&w.bcnt, nbatch * sizeof(uint32_t)));
        CK(cudaMalloc(&w.spill, nbatch * sizeof(uint32_t)));
        CK(cudaMalloc(&w.bslot, nbatch * sizeof(uint32_t)));
        CK(cudaMalloc(&w.tbase, nbatch * sizeof(uint32_t)));
        w.bsel_n = nbatch;
        w.bytes += 5 * nbatch * sizeof(uint32_t);
    }
    const uint64_t nst = (nbatch + kScanTile - 1) / kScanTile;
    if (w.sstatus_n < nst) {
        cudaFree(w.sstatus);
        w.bytes -= w.sstatus_n * sizeof(uint2);
        const size_t n = std::max<size_t>(nst, 1024);
        CK(cudaMalloc(&w.sstatus, n * sizeof(uint2)));
        w.sstatus_n = n;
        w.sstatus_fresh = true;   // zeroed on the launch stream before its first use
        w.bytes += n * sizeof(uint2);
    }
    return M3E_OK;
}

// staging of the filter kernel's tracks and kept-frame records, sized by the
// caller's output capacities (the pack kernel copies them into place)
int ensure_stage(Workspace& w, uint64_t trk, uint64_t kept) {
    if (w.stage_trk_n < trk) {
        cudaFree(w.stage_trk);
        w.bytes -= w.stage_trk_n * sizeof(m3e_track);
        CK(cudaMalloc(&w.stage_trk, trk * sizeof(m3e_track)));
        w.stage_trk_n = trk;
        w.bytes += trk * sizeof(m3e_track);
    }
    if (w.stage_kept_n < kept || !w.kept_rec) {
        cudaFree(w.stage_kept);
        cudaFree(w.kept_rec);
        w.bytes -= w.stage_kept_n * (sizeof(KeptRec) + sizeof(uint4));
        kept = std::max<uint64_t>(kept, 1);
        CK(cudaMalloc(&w.stage_kept, kept * sizeof(KeptRec)));
        CK(cudaMalloc(&w.kept_rec, kept * sizeof(uint4)));
        w.stage_kept_n = kept;
        w.bytes += kept * (sizeof(KeptRec) + sizeof(uint4));
    }
    return M3E_OK;
}

uint32_t next_epoch(Workspace& w) {
    w.epoch = (w.epoch + 1) & 0x3FFFFFFFu;
    if (w.epoch == 0) w.epoch = 1;
    return w.epoch;
}

// common launch of one mode over frames [0, F)
int run_mode(m3e_context* ctx, Workspace& w, int mode, const m3e_params* p, const float* x, const float* y,
             const float* z, const uint32_t* offsets, uint64_t F, uint64_t H, KArgs a, cudaStream_t s) {
    int rc = validate(p);
    if (rc) return rc;
    if (F >= (1ull << 31)) return fail(M3E_ERR_INVALID_ARGUMENT, "too many frames in one call");
    if (F == 0) return M3E_OK;
    if (!x || !y || !z || !offsets) return fail(M3E_ERR_INVALID_ARGUMENT, "input pointer is NULL");
    if (a.out.tracks && (reinterpret_cast<uintptr_t>(a.out.tracks) & 15u))
        return fail(M3E_ERR_INVALID_ARGUMENT, "tracks must be 16-byte aligned");
    const int fb = choose_fb(F, H);
    const uint64_t nbatch = (F + fb - 1) / fb;
    // big-frame variant (pair-factorised selection compiled in) for high occupancy
    const bool big = (mode == kModeFull || mode == kModeSelect) && (double)H > kBigMeanHits * (double)F;
    // production path split by stage (Selection Cuts | fit | tracks, vertex,
    // output staging), each kernel with its hot code in the instruction cache and
    // its own occupancy; the fused kernel then runs only the warp-batches whose
    // candidates did not fit the store
    const bool split = mode == kModeFull && ctx->split;
    // candidate store and triple list per frame: phase-I defaults, scaled up for
    // big frames (phase II: ~270 candidates and up to max_combs triples per frame)
    const uint64_t mean_hits = F ? H / F : 0;
    const uint64_t cand_pf = (big && ctx->cand_per_frame == kCandPerFrame)
                                 ? std::max<uint64_t>(kCandPerFrame, 3 * mean_hits / 2)
                                 : ctx->cand_per_frame;
    const uint64_t tri_pf = big ? 32 : 1;
    const int bps = blocks_per_sm(mode, big);
    const int grid = (int)std::min<uint64_t>(nbatch, (uint64_t)ctx->sms * bps);
    const int sgrid = split ? (int)std::min<uint64_t>(nbatch, (uint64_t)ctx->sms * blocks_per_sm(kModeSelectC, big))
                            : 0;
    const int vgrid = split ? ctx->sms * vertex_blocks_per_sm() : 0;   // its warps own vscratch / pool slots
    rc = ensure_ws(ctx, w, nbatch, p, fb, std::max(std::max(grid, sgrid), vgrid));
    if (rc) return rc;
    if (split) {
        rc = ensure_split(w, F, nbatch, cand_pf, tri_pf);
        if (rc) return rc;
    }
    a.P = make_dev_params(p);
    a.x = x; a.y = y; a.z = z; a.offsets = offsets;
    a.F = (uint32_t)F;
    a.fb = fb;
    a.nbatch = (uint32_t)nbatch;
    a.ticket = w.ticket;
    a.bticket = w.ticket;
    a.status = w.status;
    a.epoch = next_epoch(w);
    a.pool_idx = w.pool_idx; a.pool_rt = w.pool_rt; a.pool_rec = w.pool_rec; a.pool_trk = w.pool_trk;
    a.pool_stride = w.pool_stride;
    a.pair_scratch = w.pair_scratch;
    a.vscratch = w.vscratch;
    a.trk_stride = w.trk_stride;
    const bool packs = mode == kModeFull || mode == kModePack;
    if (packs) {
        const bool want_trk = mode == kModeFull && a.out.tracks != nullptr;
        rc = ensure_stage(w, want_trk ? a.out.track_capacity : 0, a.out.kept_capacity);
        if (rc) return rc;
        a.bstat = w.bstat;
        a.stage_trk = want_trk ? w.stage_trk : nullptr;
        a.stage_trk_cap = want_trk ? a.out.track_capacity : 0;
        a.stage_kept = w.stage_kept;
        a.kept_rec = w.kept_rec;
        a.stage_kept_cap = a.out.kept_capacity;
    }
    CK(cudaMemsetAsync(w.ticket, 0, 16 * sizeof(uint32_t), s));
    if (w.status_fresh) {   // look-back words: no stale epoch tag may survive from recycled memory
        CK(cudaMemsetAsync(w.status, 0, w.status_n * sizeof(uint4), s));
        w.status_fresh = false;
    }
    if (split && w.sstatus_fresh) {
        CK(cudaMemsetAsync(w.sstatus, 0, w.sstatus_n * sizeof(uint2), s));
        w.sstatus_fresh = false;
    }
    if (a.out.summary) CK(cudaMemsetAsync(a.out.summary, 0, sizeof(m3e_summary), s));
    const bool tm = ctx->timing && &w == &ctx->ws[0] && ctx->tev_used + kNEv <= ctx->tev.size();
    cudaEvent_t* ev = tm ? &ctx->tev[ctx->tev_used] : nullptr;
    if (tm) CK(cudaEventRecord(ev[0], s));
    if (split) {
        KArgs sa = a;
        sa.cand_g = w.cand_g;
        sa.cand_cap = std::min<uint64_t>(w.cand_n, std::max<uint64_t>(cand_pf * F, 1u << 10));
        sa.sel = w.sel;
        sa.bsel = w.bsel;
        sa.bcnt = w.bcnt;
        sa.bslot = w.bslot;
        sa.spill_out = w.spill;
        CK(launch_filter(kModeSelectC, big, sa, sgrid, s));
        // every warp-batch's first slot in out.tracks (frame order), for the fit kernel
        sa.tbase = w.tbase;
        sa.sstatus = w.sstatus;
        CK(launch_slot_scan(sa, (int)std::min<uint64_t>((nbatch + kScanTile - 1) / kScanTile,
                                                        (uint64_t)ctx->sms * 4), s));
        if (tm) CK(cudaEventRecord(ev[1], s));
        a.cand_g = w.cand_g;
        a.fit_g = w.fit_g;
        a.cand_cap = sa.cand_cap;
        a.sel = w.sel;
        a.bsel = w.bsel;
        a.bcnt = w.bcnt;
        a.bslot = w.bslot;
        a.tbase = w.tbase;
        a.fw = w.fw;
        a.vk = w.vk;
        a.vlist = w.vlist;
        a.vrec = w.vrec;
        a.vtr = w.vtr;
        a.tri = w.tri;
        a.tres = reinterpret_cast<VRes*>(w.tres);
        a.tri_cap = ctx->tri_cap ? std::min<uint64_t>(ctx->tri_cap, w.tri_n) : w.tri_n;
        CK(launch_fit(a, big, ctx->sms * fit_blocks_per_sm(), s));   // F + T (track stage)
        if (tm) CK(cudaEventRecord(ev[2], s));
        if (tm) CK(cudaEventRecord(ev[3], s));
        CK(launch_vertex(a, vgrid, ctx->sms, s));
        if (tm) CK(cudaEventRecord(ev[4], s));
        a.spill_list = w.spill;   // the fused kernel takes only the spilled warp-batches
        a.bticket = w.ticket + 4;
    } else if (tm) {
        for (int k = 1; k <= 4; ++k) CK(cudaEventRecord(ev[k], s));
    }
    // (split path: only the warp-batches the store could not take, none at phase I:
    // one CTA per SM is plenty and keeps the empty launch short)
    CK(launch_filter(mode, big, a, split ? std::min(grid, ctx->sms) : grid, s));
    if (tm) CK(cudaEventRecord(ev[5], s));
    if (packs) {
        const uint64_t ntiles = (nbatch + kPackTile - 1) / kPackTile;
        const int pgrid = (int)std::min<uint64_t>(ntiles, (uint64_t)ctx->sms * 8);
        CK(launch_pack(a, pgrid, s));
        CK(launch_kept(a, ctx->sms * 4, s));   // the kept frames the pack kernel listed
    }
    if (tm) {
        CK(cudaEventRecord(ev[6], s));
        ctx->tev_used += kNEv;
        ctx->tev_split += split ? 1 : 0;
    }
    return M3E_OK;
}

}  // namespace

extern "C" {

const char* m3e_version(void) { return "m3e-b200 0.1 (sm_100a)"; }

int m3e_debug_check(m3e_context* ctx, uint32_t* line) {
    if (!ctx || !line) return fail(M3E_ERR_INVALID_ARGUMENT, "NULL argument");
    CK(cudaSetDevice(ctx->device));
    unsigned int l = 0;
    CK(read_check_line(&l));
    *line = l;
    return M3E_OK;
}
const char* m3e_last_error(void) { return g_err.c_str(); }

int m3e_create(m3e_context** out, int device, uint64_t max_frames, uint64_t max_hits) {
    if (!out) return fail(M3E_ERR_INVALID_ARGUMENT, "ctx is NULL");
    int n = 0;
    if (cudaGetDeviceCount(&n) != cudaSuccess || n == 0) return fail(M3E_ERR_NO_DEVICE, "no CUDA device");
    if (device < 0 || device >= n) return fail(M3E_ERR_INVALID_ARGUMENT, "bad device ordinal");
    CK(cudaSetDevice(device));
    cudaDeviceProp prop;
    CK(cudaGetDeviceProperties(&prop, device));
    if (prop.major != 10) return fail(M3E_ERR_NO_DEVICE, "libm3e is built for sm_100a (B200)");
    m3e_context* c = new m3e_context();
    c->device = device;
    c->sms = prop.multiProcessorCount;
    c->max_frames = max_frames;
    c->max_hits = max_hits;
    const char* fused = std::getenv("M3E_FUSED");
    c->split = !(fused && fused[0] == '1');
    if (const char* cs = std::getenv("M3E_CAND_STORE")) c->cand_per_frame = std::strtoull(cs, nullptr, 10);
    else c->cand_per_frame = kCandPerFrame;
    if (const char* tc = std::getenv("M3E_TRI_CAP")) c->tri_cap = std::strtoull(tc, nullptr, 10);
    for (int i = 0; i < 2; ++i) {
        if (cudaStreamCreateWithFlags(&c->st[i], cudaStreamNonBlocking) != cudaSuccess) {
            delete c;
            return fail(M3E_ERR_CUDA, "stream creation failed");
        }
    }
    *out = c;
    return M3E_OK;
}

int m3e_destroy(m3e_context* c) {
    if (!c) return M3E_OK;
    cudaSetDevice(c->device);
    for (int i = 0; i < 2; ++i) {
        if (c->st[i]) cudaStreamSynchronize(c->st[i]);
        free_ws(c->ws[i]);
        free_chunk(c->ch[i]);
        if (c->st[i]) cudaStreamDestroy(c->st[i]);
    }
    for (auto& e : c->tev) cudaEventDestroy(e);
    delete c;
    return M3E_OK;
}

uint64_t m3e_workspace_bytes(const m3e_context* c) { return c ? c->ws[0].bytes + c->ws[1].bytes : 0; }

int m3e_set_timing(m3e_context* c, int enable) {
    if (!c) return fail(M3E_ERR_INVALID_ARGUMENT, "ctx is NULL");
    CK(cudaSetDevice(c->device));
    if (enable && c->tev.empty()) {
        c->tev.resize(kNEv * 1024);   // up to 1024 timed calls between two m3e_kernel_times()
        for (auto& e : c->tev) CK(cudaEventCreate(&e));
    }
    c->timing = enable != 0;
    c->tev_used = 0;
    c->tev_split = 0;
    return M3E_OK;
}

int m3e_kernel_times(m3e_context* c, float ms[6]) {
    if (!c || !ms) return fail(M3E_ERR_INVALID_ARGUMENT, "NULL argument");
    if (c->tev_used == 0) return fail(M3E_ERR_INVALID_ARGUMENT, "no timed call since the last reset");
    double acc[kNEv - 1] = {};
    const size_t n = c->tev_used / kNEv;
    for (size_t i = 0; i < n; ++i) {
        CK(cudaEventSynchronize(c->tev[kNEv * i + kNEv - 1]));
        for (int k = 0; k < kNEv - 1; ++k) {
            float t = 0;
            CK(cudaEventElapsedTime(&t, c->tev[kNEv * i + k], c->tev[kNEv * i + k + 1]));
            acc[k] += t;
        }
    }
    for (int k = 0; k < kNEv - 1; ++k) ms[k] = (float)(acc[k] / n);
    if (c->tev_split == 0) ms[0] = ms[1] = ms[2] = ms[3] = 0.0f;   // fused path: only the filter kernel ran
    c->tev_used = 0;
    c->tev_split = 0;
    return M3E_OK;
}

int m3e_filter(m3e_context* ctx, const m3e_params* p, const float* x, const float* y, const float* z,
               const uint32_t* offsets, uint64_t F, uint64_t H, const m3e_outputs* out, void* stream) {
    if (!ctx || !out) return fail(M3E_ERR_INVALID_ARGUMENT, "ctx/out is NULL");
    cudaStream_t s = (cudaStream_t)stream;
    KArgs a{};
    a.out = *out;
    if (F == 0) {
        if (out->summary) CK(cudaMemsetAsync(out->summary, 0, sizeof(m3e_summary), s));
        return M3E_OK;
    }
    return run_mode(ctx, ctx->ws[0], kModeFull, p, x, y, z, offsets, F, H, a, s);
}

int m3e_select_triplets(m3e_context* ctx, const m3e_params* p, const float* x, const float* y, const float* z,
                        const uint32_t* offsets, uint64_t F, uint64_t H, uint32_t* cand, float* cand_rt,
                        m3e_frame_out* frames, void* stream) {
    if (!ctx || !cand || !cand_rt || !frames) return fail(M3E_ERR_INVALID_ARGUMENT, "NULL argument");
    cudaStream_t s = (cudaStream_t)stream;
    KArgs a{};
    a.s_cand = cand;
    a.s_rt = cand_rt;
    a.out.frames = frames;
    return run_mode(ctx, ctx->ws[0], kModeSelect, p, x, y, z, offsets, F, H, a, s);
}

int m3e_fit_tracks(m3e_context* ctx, const m3e_params* p, const float* x, const float* y, const float* z,
                   const uint32_t* offsets, uint64_t F, uint64_t H, const uint32_t* cand, const float* cand_rt,
                   const uint16_t* n_cand, m3e_fit_record* rec, m3e_track* tracks, m3e_frame_out* frames,
                   void* stream) {
    if (!ctx || !cand || !cand_rt || !n_cand || !rec || !tracks || !frames)
        return fail(M3E_ERR_INVALID_ARGUMENT, "NULL argument");
    cudaStream_t s = (cudaStream_t)stream;
    KArgs a{};
    a.s_cand = const_cast<uint32_t*>(cand);
    a.s_rt = const_cast<float*>(cand_rt);
    a.s_ncand = n_cand;
    a.s_rec = rec;
    a.s_trk = tracks;
    a.out.frames = frames;
    return run_mode(ctx, ctx->ws[0], kModeFit, p, x, y, z, offsets, F, H, a, s);
}

int m3e_vertex_select(m3e_context* ctx, const m3e_params* p, const float* x, const float* y, const float* z,
                      const uint32_t* offsets, uint64_t F, uint64_t H, const m3e_track* tracks, const uint16_t* n_tracks,
                      m3e_frame_out* frames, m3e_vertex* vertices, void* stream) {
    if (!ctx || !tracks || !n_tracks || !frames) return fail(M3E_ERR_INVALID_ARGUMENT, "NULL argument");
    cudaStream_t s = (cudaStream_t)stream;
    KArgs a{};
    a.s_trk = const_cast<m3e_track*>(tracks);
    a.s_ntrk = n_tracks;
    a.s_vtx = vertices;
    a.out.frames = frames;
    return run_mode(ctx, ctx->ws[0], kModeVertex, p, x, y, z, offsets, F, H, a, s);
}

int m3e_pack_frames(m3e_context* ctx, const float* x, const float* y, const float* z, const uint32_t* offsets,
                    uint64_t F, uint64_t H, const uint8_t* reason, const m3e_outputs* out, void* stream) {
    if (!ctx || !reason || !out) return fail(M3E_ERR_INVALID_ARGUMENT, "NULL argument");
    cudaStream_t s = (cudaStream_t)stream;
    // the packer needs no cut parameters; run with a valid default set
    m3e_params p{};
    const double R[4] = {23.3, 29.8, 73.9, 86.3};
    for (int l = 0; l < 4; ++l) p.layer_r[l] = R[l];
    p.b_field = 1.0; p.target_r = 19.0; p.target_half = 50.0; p.cuts_max = 768; p.max_tracks = 64;
    p.max_combs = 64; p.x_over_x0 = 1e-3;
    KArgs a{};
    a.s_reason = reason;
    a.out = *out;
    a.out.tracks = nullptr;
    if (F == 0) {
        if (out->summary) CK(cudaMemsetAsync(out->summary, 0, sizeof(m3e_summary), s));
        return M3E_OK;
    }
    return run_mode(ctx, ctx->ws[0], kModePack, &p, x, y, z, offsets, F, H, a, s);
}

// ------------------------------------------------------------ host path ----
static int ensure_chunk(Chunk& c, uint64_t frames, uint64_t hits, bool want_tracks, uint64_t max_tracks) {
    if (c.cap_frames >= frames && c.cap_hits >= hits && (!want_tracks || c.cap_tracks >= frames * max_tracks))
        return M3E_OK;
    free_chunk(c);
    c.cap_frames = frames;
    c.cap_hits = hits;
    const size_t hb = (hits + 8) * sizeof(float);
    CK(cudaMalloc(&c.x, hb)); CK(cudaMalloc(&c.y, hb)); CK(cudaMalloc(&c.z, hb));
    CK(cudaMalloc(&c.offsets, (4 * frames + 4) * sizeof(uint32_t)));
    CK(cudaMalloc(&c.reason, frames));
    CK(cudaMalloc(&c.frames, frames * sizeof(m3e_frame_out)));
    CK(cudaMalloc(&c.vertices, frames * sizeof(m3e_vertex)));
    CK(cudaMalloc(&c.kept_frame, frames * sizeof(uint32_t)));
    CK(cudaMalloc(&c.kept_offsets, (4 * frames + 1) * sizeof(uint32_t)));
    CK(cudaMalloc(&c.kx, hb)); CK(cudaMalloc(&c.ky, hb)); CK(cudaMalloc(&c.kz, hb));
    CK(cudaMalloc(&c.summary, sizeof(m3e_summary)));
    CK(cudaMallocHost(&c.h_summary, sizeof(m3e_summary)));
    if (want_tracks) {
        c.cap_tracks = frames * max_tracks;
        CK(cudaMalloc(&c.tracks, c.cap_tracks * sizeof(m3e_track)));
    }
    CK(cudaEventCreateWithFlags(&c.ev_summary, cudaEventDisableTiming));
    CK(cudaEventCreateWithFlags(&c.ev_free, cudaEventDisableTiming));
    return M3E_OK;
}

int m3e_filter_host(m3e_context* ctx, const m3e_params* p, const float* x, const float* y, const float* z,
                    const uint32_t* offsets, uint64_t F, const m3e_outputs* out) {
    if (!ctx || !out) return fail(M3E_ERR_INVALID_ARGUMENT, "ctx/out is NULL");
    int rc = validate(p);
    if (rc) return rc;
    CK(cudaSetDevice(ctx->device));
    m3e_summary total{};
    if (F == 0) {
        if (out->summary) *out->summary = total;
        return M3E_OK;
    }
    if (!x || !y || !z || !offsets) return fail(M3E_ERR_INVALID_ARGUMENT, "input pointer is NULL");
    // chunk size: bounded by the context limits, at most 2^20 frames per chunk
    const uint64_t cf = std::max<uint64_t>(1, std::min<uint64_t>({F, ctx->max_frames ? ctx->max_frames : F,
                                                                   (uint64_t)1 << 20}));
    uint64_t max_chunk_hits = 0;
    for (uint64_t a = 0; a < F; a += cf) {
        const uint64_t b = std::min(F, a + cf);
        max_chunk_hits = std::max<uint64_t>(max_chunk_hits, offsets[4 * b] - offsets[4 * a] + 8);
    }
    const bool want_tracks = out->tracks != nullptr || out->frames != nullptr;
    for (int i = 0; i < 2; ++i) {
        rc = ensure_chunk(ctx->ch[i], cf, max_chunk_hits, want_tracks, (uint64_t)p->max_tracks);
        if (rc) return rc;
        ctx->ch[i].used = false;
    }
    struct Done {
        uint64_t a, b;
        int set;
    };
    std::vector<Done> pending;
    uint64_t base_trk = 0, base_kept = 0, base_hits = 0;
    auto finish = [&](const Done& d) -> int {
        Chunk& c = ctx->ch[d.set];
        cudaStream_t s = ctx->st[d.set];
        CK(cudaEventSynchronize(c.ev_summary));
        const m3e_summary sm = *c.h_summary;
        uint64_t K = 0;
        for (int r = 1; r < 6; ++r) K += sm.kept_by_reason[r];
        const uint64_t Hk = sm.kept_hits, T = sm.track_slots;   // the chunk's track-array extent
        if (sm.overflow) return fail(M3E_ERR_CAPACITY, "device chunk capacity exceeded");
        if ((out->kept_frame || out->vertices || out->kept_offsets) && base_kept + K > out->kept_capacity)
            return fail(M3E_ERR_CAPACITY, "kept_capacity too small");
        if (out->kept_x && base_hits + Hk > out->kept_hit_capacity)
            return fail(M3E_ERR_CAPACITY, "kept_hit_capacity too small");
        if (out->tracks && base_trk + T > out->track_capacity)
            return fail(M3E_ERR_CAPACITY, "track_capacity too small");
        const uint64_t nfr = d.b - d.a;
        // chunk-local indices -> call-global, on the device before the copies
        // (frames' track_first / kept_index, tracks' and kept records' frame,
        // packed offsets)
        Rebase rb{};
        rb.frames = out->frames ? c.frames : nullptr;
        rb.n_frames = nfr;
        rb.tracks = out->tracks ? c.tracks : nullptr;
        rb.n_tracks = T;
        rb.kept_frame = out->kept_frame ? c.kept_frame : nullptr;
        rb.kept_offsets = out->kept_offsets ? c.kept_offsets : nullptr;
        rb.vertices = out->vertices ? c.vertices : nullptr;
        rb.n_kept = K;
        rb.frame0 = (uint32_t)d.a;
        rb.base_trk = (uint32_t)base_trk;
        rb.base_kept = (uint32_t)base_kept;
        rb.base_hits = (uint32_t)base_hits;
        if (d.a || base_trk || base_kept || base_hits) CK(launch_rebase(rb, ctx->sms, s));
        if (out->reason) CK(cudaMemcpyAsync(out->reason + d.a, c.reason, nfr, cudaMemcpyDeviceToHost, s));
        if (out->frames)
            CK(cudaMemcpyAsync(out->frames + d.a, c.frames, nfr * sizeof(m3e_frame_out), cudaMemcpyDeviceToHost, s));
        if (out->tracks && T)
            CK(cudaMemcpyAsync(out->tracks + base_trk, c.tracks, T * sizeof(m3e_track), cudaMemcpyDeviceToHost, s));
        if (K) {
            if (out->kept_frame)
                CK(cudaMemcpyAsync(out->kept_frame + base_kept, c.kept_frame, K * 4, cudaMemcpyDeviceToHost, s));
            if (out->kept_offsets)
                CK(cudaMemcpyAsync(out->kept_offsets + 4 * base_kept, c.kept_offsets, 4 * K * 4,
                                   cudaMemcpyDeviceToHost, s));
            if (out->vertices)
                CK(cudaMemcpyAsync(out->vertices + base_kept, c.vertices, K * sizeof(m3e_vertex),
                                   cudaMemcpyDeviceToHost, s));
        }
        if (Hk && out->kept_x) {
            CK(cudaMemcpyAsync(out->kept_x + base_hits, c.kx, Hk * 4, cudaMemcpyDeviceToHost, s));
            CK(cudaMemcpyAsync(out->kept_y + base_hits, c.ky, Hk * 4, cudaMemcpyDeviceToHost, s));
            CK(cudaMemcpyAsync(out->kept_z + base_hits, c.kz, Hk * 4, cudaMemcpyDeviceToHost, s));
        }
        CK(cudaEventRecord(c.ev_free, s));
        CK(cudaEventSynchronize(c.ev_free));
        total.frames += sm.frames;
        for (int r = 0; r < 6; ++r) total.kept_by_reason[r] += sm.kept_by_reason[r];
        total.candidates += sm.candidates;
        total.tracks += sm.tracks;
        total.track_slots += sm.track_slots;
        total.kept_hits += sm.kept_hits;
        total.vertices += sm.vertices;
        base_trk += T;
        base_kept += K;
        base_hits += Hk;
        return M3E_OK;
    };
    int ci = 0;
    for (uint64_t a = 0; a < F; a += cf, ++ci) {
        const uint64_t b = std::min(F, a + cf);
        const int set = ci & 1;
        Chunk& c = ctx->ch[set];
        cudaStream_t s = ctx->st[set];
        // the previous user of this set must have been drained (finish() syncs ev_free)
        if (pending.size() >= 2) {
            rc = finish(pending.front());
            if (rc) return rc;
            pending.erase(pending.begin());
        }
        const uint64_t h0 = offsets[4 * a], h1 = offsets[4 * b];
        const uint64_t h0a = h0 & ~3ull;           // keep 16 B alignment of the bulk copies
        const uint64_t nh = h1 - h0a;
        if (nh) {
            CK(cudaMemcpyAsync(c.x, x + h0a, nh * 4, cudaMemcpyHostToDevice, s));
            CK(cudaMemcpyAsync(c.y, y + h0a, nh * 4, cudaMemcpyHostToDevice, s));
            CK(cudaMemcpyAsync(c.z, z + h0a, nh * 4, cudaMemcpyHostToDevice, s));
        }
        CK(cudaMemcpyAsync(c.offsets, offsets + 4 * a, (4 * (b - a) + 1) * 4, cudaMemcpyHostToDevice, s));
        m3e_outputs o{};
        o.reason = c.reason;
        o.frames = c.frames;
        o.tracks = want_tracks ? c.tracks : nullptr;
        o.track_capacity = c.cap_tracks;
        o.vertices = c.vertices;
        o.kept_frame = c.kept_frame;
        o.kept_offsets = c.kept_offsets;
        o.kept_capacity = c.cap_frames;
        o.kept_x = c.kx; o.kept_y = c.ky; o.kept_z = c.kz;
        o.kept_hit_capacity = c.cap_hits;
        o.summary = c.summary;
        KArgs ka{};
        ka.out = o;
        // hit pointers shifted so that the (global) offsets index the chunk's copy
        rc = run_mode(ctx, ctx->ws[set], kModeFull, p, c.x - h0a, c.y - h0a, c.z - h0a, c.offsets, b - a,
                      h1 - h0, ka, s);
        if (rc) return rc;
        CK(cudaMemcpyAsync(c.h_summary, c.summary, sizeof(m3e_summary), cudaMemcpyDeviceToHost, s));
        CK(cudaEventRecord(c.ev_summary, s));
        pending.push_back({a, b, set});
    }
    for (const Done& d : pending) {
        rc = finish(d);
        if (rc) return rc;
    }
    if (out->kept_offsets) out->kept_offsets[4 * base_kept] = (uint32_t)base_hits;
    if (out->summary) *out->summary = total;
    return M3E_OK;
}

}  // extern "C"

static_assert(sizeof(m3e_frame_out) == 16, "m3e_frame_out layout");
static_assert(sizeof(m3e_track) == 32, "m3e_track layout");
static_assert(sizeof(m3e_vertex) == 56, "m3e_vertex layout");
static_assert(sizeof(m3e_fit_record) == 40, "m3e_fit_record layout");
static_assert(sizeof(m3e_summary) == 104, "m3e_summary layout");
