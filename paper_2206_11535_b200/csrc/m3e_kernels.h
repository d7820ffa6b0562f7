// m3e_kernels.h -- internal interface between the runtime (m3e_runtime.cu) and
// the filter kernel (m3e_kernels.cu).  Not part of the public ABI.
#pragma once
#include <cstddef>
#include <cstdint>
#include <cuda_runtime.h>

#include "m3e.h"
#include "m3e_device.cuh"

namespace m3e {

constexpr int kThreads = 256;        // 8 warps per CTA, each an independent pipeline
constexpr int kWarps = kThreads / 32;
constexpr int kFB = 16;              // frames per warp-batch (upper bound; runtime fb <= kFB)
constexpr int kHCap = 256;           // hits of a warp-batch staged in shared memory
constexpr int kMaxTracksCap = 128;   // upper bound accepted for params.max_tracks
constexpr int kMaxCombsCap = 128;    // upper bound accepted for params.max_combs + 1
constexpr int kMaxCutsCap = 1023;    // upper bound accepted for params.cuts_max
constexpr size_t kVScratchBytes = 4096;   // >= sizeof(VScratch), checked in m3e_kernels.cu
constexpr size_t kVResBytes = 56;         // sizeof(VRes) (phase-2 vertex result), checked in m3e_kernels.cu

// kModeSelectC: the Selection Cuts alone, candidates written compactly to the
// candidate store (first kernel of the split production path: select -> fit ->
// vertex -> fused kernel over the spilled warp-batches only -> pack)
enum { kModeFull = 0, kModeSelect = 1, kModeFit = 2, kModeVertex = 3, kModePack = 4, kModeSelectC = 5 };
constexpr uint32_t kSpilled = 0xFFFFFFFFu;   // bsel[] entry of a warp-batch whose candidates did not fit

// big frames (phase-II occupancy): pair-factorised selection with per-warp lists
constexpr long long kBigCombos = 4096;   // n0 n1 n2 above which the pair path is used
constexpr double kBigMeanHits = 60.0;    // calls with more hits per frame use the BIG kernel variant
constexpr int kPairCapG = 8192;          // entries of each pair list
constexpr size_t kPairWords = 4 * (size_t)kPairCapG + (kMaxLayerHits + 2) + (kPairCapG + 1);

constexpr int kPackTile = 256;       // warp-batches per CTA of the pack kernel (8 warps x 32)

// per warp-batch counts and staging offsets, written by the filter kernel and
// consumed by the pack kernel (32 B)
struct BatchStat {
    uint32_t n_trk, n_kept, n_hits;  // tracks, kept frames, hits of kept frames
    uint32_t s_trk, s_kept;          // staging offsets of its tracks / kept-frame records; s_trk =
                                     // kSpilled: its tracks are the front of its store segment
    uint32_t nf;                     // frames in the warp-batch
    uint32_t n_slot;                 // its track slots (sum over frames of min(stored candidates,
                                     // max_tracks)): the extent it takes in the output track array
    uint32_t pad;
};

// kept-frame record staged by the filter kernel (64 B)
struct KeptRec {
    uint32_t frame;
    uint32_t pad;
    m3e_vertex v;                    // v.frame = 0xFFFFFFFF unless the frame has a vertex
};

struct KArgs {
    DevParams P;
    const float* x;
    const float* y;
    const float* z;
    const uint32_t* offsets;
    uint32_t F;            // frames in this call
    int fb;                // frames per batch
    uint32_t nbatch;
    // workspace
    uint32_t* ticket;      // counters (zeroed before the launch): [0] select warp-batch ticket, [1] staged
                           // tracks, [2] staged kept frames, [3] pack-kernel tile ticket, [4] filter
                           // warp-batch ticket, [5] spilled warp-batches, [6..7] candidate-store fill (u64),
                           // [8] fit-kernel unit ticket, [9] vertex-list fill, [10] (unused)
                           // group ticket, [11] triple-list fill, [12] slot-scan tile ticket, [13] kept
                           // frames (pack kernel -> kept kernel)
    uint32_t* bticket;     // this launch's warp-batch ticket (ticket + 0 or ticket + 4)
    // candidate store of the split path (kModeSelectC writes, fit_kernel reads)
    uint32_t* spill_out;   // kModeSelectC: appends the warp-batches that did not fit (count in ticket[5])
    uint32_t* spill_list;  // kModeFull, non-NULL: process only these warp-batches
    uint4* cand_g;         // {first hit of the frame, frame, offsets of h1 | h2 << 16 and of h0 inside the
                           // frame}, warp-batch contiguous, frame order; frame = kSpilled marks an unused
                           // entry
    m3e_track* fit_g;      // fit_kernel: each warp-batch's output tracks (every frame's first
                           // max_tracks accepted, frame order) compacted to the front of its segment
    uint64_t cand_cap;     // entries of cand_g (< 2^32)
    uint32_t* sel;         // [F] per frame: n_cand | reason << 16
    uint32_t* fw;          // [F] per frame after the track stage: n_tracks | n_neg << 8 | n_combs << 16 |
                           // reason << 24 (fit_kernel writes, vertex_kernel updates, pack_kernel reads)
    uint32_t* vk;          // [F] vertex_kernel: list position of a frame's vertex (reason VERTEX only)
    uint2* vlist;          // frames for the vertex stage {frame, first store entry}, count in ticket[9]
    m3e_vertex* vrec;      // vertex of vlist entry k
    uint2* vtr;            // [vlist] its triples {first, count} in tri (count 0: decided without phase 2)
    uint4* tri;            // listed e+e+e- triples {vlist entry, store offsets a | b << 10 | e << 20,
                           // track indices a | b << 8 | e << 16, 0}, count in ticket[11]
    struct VRes* tres;     // phase-2 result of each listed triple
    uint64_t tri_cap;      // entries of tri / tres
    uint32_t* bsel;        // [nbatch] first store entry of the warp-batch, or kSpilled
    uint32_t* bcnt;        // [nbatch] its store entries
    uint32_t* bslot;       // [nbatch] its track slots: sum over its frames of min(stored candidates,
                           // max_tracks), an upper bound of its output tracks (selection kernel)
    uint32_t* tbase;       // [nbatch] exclusive prefix of bslot in warp-batch order (slot_scan_kernel): the
                           // warp-batch's first slot in out.tracks
    uint2* sstatus;        // slot_scan_kernel decoupled look-back, one 8 B word per tile
    uint4* status;         // pack-kernel decoupled look-back, one 16 B word per tile
    uint32_t epoch;        // launch epoch tag of the status words (never 0)
    BatchStat* bstat;      // [nbatch]
    m3e_track* stage_trk;  // staged tracks
    uint64_t stage_trk_cap;
    KeptRec* stage_kept;   // staged kept-frame records
    uint64_t stage_kept_cap;
    uint4* kept_rec;       // [out.kept_capacity] pack -> kept kernel: {frame, first packed hit, vertex
                           // source: reason, or 1 << 31 | stage_kept index}, count in ticket[13]
    // per-CTA scratch (MODE_FULL)
    uint32_t* pool_idx;
    float* pool_rt;
    m3e_fit_record* pool_rec;
    m3e_track* pool_trk;
    size_t pool_stride;    // candidate entries per warp >= fb * cuts_max
    uint32_t* pair_scratch;   // per-warp pair lists of the big-frame selection (kPairWords words per warp)
    void* vscratch;           // per-warp vertex-stage scratch (kVScratchBytes per warp)
    size_t trk_stride;     // track entries per warp >= fb * max_tracks
    // stage-mode fixed slots
    uint32_t* s_cand;
    float* s_rt;
    m3e_fit_record* s_rec;
    m3e_track* s_trk;
    const uint16_t* s_ncand;
    const uint16_t* s_ntrk;
    const uint8_t* s_reason;
    m3e_vertex* s_vtx;
    // outputs (device pointers; NULL entries are skipped)
    m3e_outputs out;
};

// host path: chunk-local output indices made call-global (m3e_filter_host)
struct Rebase {
    m3e_frame_out* frames;
    uint64_t n_frames;
    m3e_track* tracks;
    uint64_t n_tracks;
    uint32_t* kept_frame;
    uint32_t* kept_offsets;
    m3e_vertex* vertices;
    uint64_t n_kept;
    uint32_t frame0, base_trk, base_kept, base_hits;
};
cudaError_t launch_rebase(const Rebase& r, int sms, cudaStream_t s);

size_t smem_bytes();
cudaError_t launch_filter(int mode, bool big, const KArgs& a, int grid, cudaStream_t s);
cudaError_t launch_pack(const KArgs& a, int grid, cudaStream_t s);
cudaError_t launch_kept(const KArgs& a, int grid, cudaStream_t s);
cudaError_t read_check_line(unsigned int* line);   // check build: first failed index check (0: none)
constexpr int kScanItems = 8;                          // warp-batches per thread of slot_scan_kernel
constexpr int kScanTile = kThreads * kScanItems;       // warp-batches per tile (CTA iteration)
cudaError_t launch_slot_scan(const KArgs& a, int grid, cudaStream_t s);
cudaError_t launch_fit(const KArgs& a, bool big, int grid, cudaStream_t s);
int fit_blocks_per_sm();
cudaError_t launch_vertex(const KArgs& a, int grid, int sms, cudaStream_t s);
int vertex_blocks_per_sm();
int triple_blocks_per_sm();
int blocks_per_sm(int mode, bool big);

}  // namespace m3e
