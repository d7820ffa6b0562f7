/*
 * m3e.h -- C ABI of the B200 Mu3e online event selection library (libm3e.so).
 *
 * The library implements the data-parallel hot path of PAPER.md (arXiv
 * 2206.11535, "Online Event Selection for Mu3e using GPUs"): for every frame of
 * hits, Selection Cuts over layer-0/1/2 hit triplets (Sec. IV-A, Eq. 2-5,
 * Alg. 2), the multiple-scattering Triplet Fit extended to layer 3 (Sec. IV-B,
 * Eq. 6-8, Alg. 3) and the e+e+e- vertex selection (Sec. IV-C, Eq. 9-12,
 * Alg. 4), then packs the kept frames (Sec. V-A: kept frames are stored).
 * Frames are independent (Sec. V-B, Alg. 1).
 *
 * Conventions for every entry point
 *   - Pointers marked [dev] are device (HBM) pointers, [host] are host pointers
 *     (pinned memory gives full PCIe speed, pageable works).  The caller owns
 *     every buffer; the library never frees caller memory.
 *   - All work is enqueued on `stream` (a cudaStream_t, may be NULL = legacy
 *     default stream); calls return after enqueueing unless stated otherwise.
 *   - Return value: M3E_OK (0) or a negative M3E_ERR_*; m3e_last_error() gives
 *     a message (thread-local).  Errors never leave partial state in the
 *     context; outputs are undefined after an error.
 *   - Lengths: F = number of frames, H = number of hits = offsets[4F]
 *     (H < 2^32 per call; passed explicitly so no call reads it back).
 *   - Units: mm, MeV, tesla.  B along +z; a positive charge turns clockwise
 *     seen from +z, and has positive curvature (reading R5).
 *
 * HBM layout of one call's input: structure of arrays
 *   x, y, z   float32[H (+4 slack)]  hit coordinates, sorted by frame, then layer
 *   offsets   uint32[4F+1]           offsets[4f+l] = first hit of layer l (0..3)
 *                                    of frame f; offsets[4F] = H.
 * Limits: at most 1024 hits per layer per frame (larger frames get reason
 * M3E_REASON_INVALID); the x/y/z allocations must extend 16 bytes past the last
 * hit (bulk copies round the end up to 16 B).
 */
#ifndef M3E_H
#define M3E_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define M3E_OK 0
#define M3E_ERR_INVALID_ARGUMENT -1
#define M3E_ERR_CUDA -2
#define M3E_ERR_CAPACITY -3     /* an output buffer was too small (see summary) */
#define M3E_ERR_NO_DEVICE -4

/* keep reasons (Fig. 7 right legend "reason to keep") */
#define M3E_REASON_NONE 0              /* discarded */
#define M3E_REASON_TRIPLET_OVERFLOW 1  /* > cuts_max triplets survive the cuts (Sec. V-B, Sec. VI) */
#define M3E_REASON_TRACK_OVERFLOW 2    /* > max_tracks tracks accepted (Alg. 3) */
#define M3E_REASON_COMB_OVERFLOW 3     /* > max_combs e+e+e- triples pass the energy test (Alg. 4) */
#define M3E_REASON_VERTEX 4            /* a signal-compatible vertex was found (Alg. 4) */
#define M3E_REASON_INVALID 5           /* frame exceeds the layout limits; kept unprocessed */

/* Filter configuration.  Values from config/thresholds.json; the paper fixes
 * cuts_max = 768 (Sec. VI), chi2_max = 32 (Sec. IV-B), target radius 19 mm
 * (Sec. IV-C); the other thresholds are tuned on generated truth (R4). */
typedef struct m3e_params {
    double layer_r[4];       /* cylinder radii r_{t,0..3} [mm] (Sec. IV-A simplification) */
    double b_field;          /* [T] */
    double target_r;         /* double-cone target radius [mm] */
    double target_half;      /* double-cone target half length [mm] */
    double dlambda_max;      /* keep |tan l12 - tan l01| <= dlambda_max          (Eq. 2-3) */
    double cos_phi01_min;    /* keep cos Phi_01 >= cos_phi01_min                 (Eq. 4) */
    double cos_phi12_min;    /* keep cos Phi_12 >= cos_phi12_min                 (Eq. 4) */
    double rt_min, rt_max;   /* keep rt_min <= |r_tc| <= rt_max [mm]             (Eq. 5) */
    int32_t cuts_max;        /* 768 */
    double x_over_x0;        /* material per layer for sigma_MS (Highland) */
    double chi2_max;         /* 32 */
    int32_t max_tracks;      /* per frame */
    double e_window;         /* |E_a + E_b + E_e - m_mu| <= e_window [MeV] */
    double xy_margin;        /* intersections kept within target_r + xy_margin [mm] */
    double sigma_pixel;      /* [mm] (Eq. 10) */
    double chi2_vertex_max;  /* vertex chi2 (Eq. 12) */
    double target_dist_max;  /* distance of the vertex to the target surface [mm] */
    double p_total_max;      /* |sum of momenta at the points of closest approach| [MeV/c] */
    int32_t max_combs;       /* per frame */
} m3e_params;

/* per-frame result (16 B) */
typedef struct m3e_frame_out {
    uint16_t n_cand;         /* min(#triplets passing the cuts, cuts_max + 1) */
    uint16_t n_tracks;       /* min(#accepted tracks, max_tracks + 1) */
    uint16_t n_combs;        /* min(#energy-passing e+e+e- triples, max_combs + 1) */
    uint8_t reason;          /* M3E_REASON_* */
    uint8_t n_neg;           /* accepted negative tracks (saturating at 255) */
    uint32_t track_first;    /* index of this frame's first track in `tracks` */
    uint32_t kept_index;     /* index among kept frames, 0xFFFFFFFF if discarded */
} m3e_frame_out;

/* fitted track (32 B), Sec. IV-B "the track parameters are calculated" */
typedef struct m3e_track {
    uint32_t frame;          /* frame index within the call */
    uint16_t hit[4];         /* layer-local hit index in layers 0..3 */
    float kappa;             /* signed 3D curvature kappa-bar (Eq. 8) [1/mm]; > 0: e+ */
    float chi2;              /* chi2_global(kappa-bar) (Eq. 7) */
    float cos_theta01;       /* cos polar angle of the arc h0->h1 (= sin lambda_01 of Eq. 11) */
    float cx, cy;            /* centre of the transverse circle through h0, h1 [mm] */
} m3e_track;

/* vertex candidate of a frame kept with M3E_REASON_VERTEX (56 B) */
typedef struct m3e_vertex {
    uint32_t frame;          /* frame index (0xFFFFFFFF: kept frame without a vertex) */
    uint16_t track[3];       /* e+, e+, e-: indices into the frame's track list */
    uint16_t pad;
    float target_dist;       /* distance of the vertex to the target surface [mm] */
    double x, y, z;          /* estimated vertex mu = (mu_t, mu_z) [mm] (Eq. 9, 11) */
    double chi2;             /* Eq. 12 */
    float p_total;           /* |sum p| at the points of closest approach [MeV/c] */
    uint32_t pad2;
} m3e_vertex;

/* run summary, accumulated on the device (all uint64) */
typedef struct m3e_summary {
    uint64_t frames;
    uint64_t kept_by_reason[6];
    uint64_t candidates;     /* sum of stored candidates (<= cuts_max per frame) */
    uint64_t tracks;         /* tracks written */
    uint64_t kept_hits;      /* hits written to the packed output */
    uint64_t vertices;
    uint64_t overflow;       /* 1 if an output capacity was exceeded */
    uint64_t track_slots;    /* extent of the track array: slots used by `tracks` (>= tracks) */
} m3e_summary;

/* outputs of one filter call (all [dev] for m3e_filter, [host] for m3e_filter_host;
 * any pointer may be NULL to skip that output, capacities are element counts) */
typedef struct m3e_outputs {
    uint8_t* reason;              /* [F] M3E_REASON_* per frame (the accept flags) */
    m3e_frame_out* frames;        /* [F] */
    m3e_track* tracks;            /* [track_capacity] (device: 16-byte aligned), frame-ordered with
                                     unused slots: frame f's
                                     tracks are tracks[track_first .. track_first + min(n_tracks,
                                     max_tracks)); the frames are grouped in warp-batches of
                                     consecutive frames, each owning sum over its frames of
                                     min(n_cand, max_tracks) slots (0 for triplet-overflow /
                                     invalid frames) whose tail past its last track is marked unused
                                     (frame = 0xFFFFFFFF, other bytes 0).  The array's extent is
                                     summary.track_slots <= sum over frames of min(n_cand,
                                     max_tracks); track_capacity must cover it. */
    uint64_t track_capacity;
    m3e_vertex* vertices;         /* [kept_capacity], vertices[kept_index]; .frame = 0xFFFFFFFF
                                     for frames kept for another reason */
    /* packed kept frames (Sec. V-A layout, SoA): */
    uint32_t* kept_frame;         /* [kept_capacity] frame index of each kept frame */
    uint32_t* kept_offsets;       /* [4*kept_capacity+1] layer starts inside kept_x/y/z */
    uint64_t kept_capacity;
    float *kept_x, *kept_y, *kept_z;  /* [kept_hit_capacity] */
    uint64_t kept_hit_capacity;
    m3e_summary* summary;         /* [1] */
} m3e_outputs;

/* ---------------------------------------------------------------- runtime --- */
/* Library version string. */
const char* m3e_version(void);
/* Message of the last error on this thread (never NULL). */
const char* m3e_last_error(void);

/* Opaque context: device workspace, streams, CUDA graph, pinned staging.
 * max_frames / max_hits bound one call (device side); device = CUDA ordinal.
 * Environment read here (testing knobs, results never change): M3E_FUSED=1 runs
 * the single fused filter kernel; M3E_CAND_STORE=n sizes the candidate store at
 * n entries per frame (warp-batches that do not fit are re-selected by the fused
 * kernel); M3E_TRI_CAP=n caps the vertex stage's triple list (frames whose
 * triples do not fit are decided in place). */
typedef struct m3e_context m3e_context;
int m3e_create(m3e_context** ctx, int device, uint64_t max_frames, uint64_t max_hits);
int m3e_destroy(m3e_context* ctx);
/* Bytes of device workspace the context holds (informational). */
uint64_t m3e_workspace_bytes(const m3e_context* ctx);
/* Kernel timing: when enabled, every m3e_filter call records CUDA events on its
 * stream around each of its kernels (up to 1024 calls); m3e_kernel_times()
 * waits for them and returns the MEAN durations in ms over those calls, then
 * resets the record:
 *   ms[0] selection kernel, ms[1] fit kernel (with the per-frame track stage),
 *   ms[2] 0 (no separate track kernel), ms[3] vertex kernels (all four 0 when
 *   the call ran the single fused filter kernel), ms[4] the fused filter kernel
 *   over warp-batches the candidate store could not take (the whole path on the
 *   fused variant), ms[5] output kernel (frame records, tracks, kept frames).
 * The split path is the default; M3E_FUSED=1 in the environment at m3e_create
 * selects the single fused kernel (same results). */
int m3e_set_timing(m3e_context* ctx, int enable);
int m3e_kernel_times(m3e_context* ctx, float ms[6]);
/* Internal index checks (testing).  The check build of the library
 * (lib/libm3e_check.so, compiled with -DM3E_CHECK; same ABI and results) bounds-
 * checks the kernels' shared-memory and workspace indices and records the source
 * line of the first failed check instead of trapping.  Synchronises the device,
 * sets *line to that line (0: no check failed) and clears it; in the production
 * library *line = 0xFFFFFFFF (checks not compiled in). */
int m3e_debug_check(m3e_context* ctx, uint32_t* line);

/* Full hot path on device-resident input (the call bench.py times): Selection
 * Cuts -> triplet fit -> tracks -> vertex selection -> output staging -> pack for
 * frames [0, F), nine kernel launches on `stream`.
 * Outputs [dev]; frames, tracks, vertices and kept frames in frame order (the
 * track array with unused slots, see m3e_outputs.tracks: the fit kernel writes
 * every track straight into its final slot, no reordering copy). */
int m3e_filter(m3e_context* ctx, const m3e_params* p, const float* x, const float* y, const float* z,
               const uint32_t* offsets, uint64_t F, uint64_t H, const m3e_outputs* out, void* stream);

/* Same on HOST buffers: copies the input host->device in chunks overlapped with
 * compute on two streams, copies the requested outputs device->host, and
 * returns after synchronising.  Input and outputs [host]. */
int m3e_filter_host(m3e_context* ctx, const m3e_params* p, const float* x, const float* y,
                    const float* z, const uint32_t* offsets, uint64_t F, const m3e_outputs* out);

/* ------------------------------------------------------- stage entry points --- */
/* Each stage of the hot path on its own, with per-frame fixed-capacity slots, for
 * stage-isolated parity tests.  All pointers [dev]. */

/* (b)+(c) Selection Cuts (Eq. 2-5, Alg. 2) with ballot compaction.
 * cand[f*cuts_max + i] = i0 | i1 << 10 | i2 << 20 (layer-local indices) in the
 * row-major order of Alg. 2; cand_rt[...] = cached signed r_tc (Eq. 5);
 * frames[f].n_cand = min(#survivors, cuts_max + 1). */
int m3e_select_triplets(m3e_context* ctx, const m3e_params* p, const float* x, const float* y,
                        const float* z, const uint32_t* offsets, uint64_t F, uint64_t H, uint32_t* cand,
                        float* cand_rt, m3e_frame_out* frames, void* stream);

/* per-candidate fit record of the stage-(d) tap (40 B) */
typedef struct m3e_fit_record {
    uint8_t status;          /* 0 ok, 1 degenerate, 2 no reach, 3 layer 3 empty, 4 degenerate 2nd,
                                5 chi2 >= chi2_max, 6 circle domain (as the oracle's OR_FIT_*) */
    uint8_t pad;
    uint16_t hit3;           /* chosen layer-3 hit (0xFFFF if none) */
    float kappa1, kappa2;    /* single-triplet curvatures kappa_t (signed) */
    float var1, var2;        /* sigma^2_{kappa,t} */
    float kappa;             /* kappa-bar (Eq. 8) */
    float chi2;              /* chi2_global (Eq. 7) */
    float cos_theta01;       /* track parameters (valid when status == 0) */
    float cx, cy;
} m3e_fit_record;

/* (d) Triplet fit + layer-3 extension (Eq. 6-8, Alg. 3) of given candidates
 * (n_cand[f] <= cuts_max candidates per frame in the m3e_select_triplets slot
 * layout).  rec[f*cuts_max + i]: per-candidate record; tracks[f*max_tracks + j]:
 * accepted tracks in candidate order; frames[f].n_tracks. */
int m3e_fit_tracks(m3e_context* ctx, const m3e_params* p, const float* x, const float* y,
                   const float* z, const uint32_t* offsets, uint64_t F, uint64_t H, const uint32_t* cand,
                   const float* cand_rt, const uint16_t* n_cand, m3e_fit_record* rec,
                   m3e_track* tracks, m3e_frame_out* frames, void* stream);

/* (e) Vertex selection (Sec. IV-C, Alg. 4) on given tracks
 * (tracks[f*max_tracks + j], j < n_tracks[f] <= max_tracks): frames[f].reason,
 * n_combs, n_neg; vertices[f] valid when reason == M3E_REASON_VERTEX. */
int m3e_vertex_select(m3e_context* ctx, const m3e_params* p, const float* x, const float* y,
                      const float* z, const uint32_t* offsets, uint64_t F, uint64_t H, const m3e_track* tracks,
                      const uint16_t* n_tracks, m3e_frame_out* frames, m3e_vertex* vertices,
                      void* stream);

/* (f) Output packer: given per-frame reasons, pack the kept frames' hits (SoA)
 * and frame indices in frame order; summary counts. */
int m3e_pack_frames(m3e_context* ctx, const float* x, const float* y, const float* z,
                    const uint32_t* offsets, uint64_t F, uint64_t H, const uint8_t* reason,
                    const m3e_outputs* out, void* stream);

#ifdef __cplusplus
}
#endif
#endif
