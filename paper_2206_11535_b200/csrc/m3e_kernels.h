// m3e_kernels.h -- internal interface between the runtime (m3e_runtime.cu) and
// the filter kernel (m3e_kernels.cu).  Not part of the public ABI.
#pragma once
#include <cstddef>
#include <cstdint>
#include <cuda_runtime.h>

#include "m3e.h"
#include "m3e_device.cuh"

namespace m3e {

constexpr int kThreads = 256;        // 8 warps per CTA
constexpr int kWarps = kThreads / 32;
constexpr int kFB = 64;              // frames per batch (upper bound; runtime fb <= kFB)
constexpr int kHCap = 2048;          // hits of a batch staged in shared memory
constexpr int kMaxTracksCap = 128;   // upper bound accepted for params.max_tracks
constexpr int kMaxCombsCap = 256;    // upper bound accepted for params.max_combs + 1
constexpr int kMaxCutsCap = 1023;    // upper bound accepted for params.cuts_max

enum { kModeFull = 0, kModeSelect = 1, kModeFit = 2, kModeVertex = 3, kModePack = 4 };

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
    uint32_t* ticket;      // batch ticket counter (zeroed before the launch)
    uint4* status;         // decoupled look-back status, one 16 B word per batch
    uint32_t epoch;        // launch epoch tag of the status words (never 0)
    // per-CTA scratch (MODE_FULL)
    uint32_t* pool_idx;
    float* pool_rt;
    m3e_fit_record* pool_rec;
    m3e_track* pool_trk;
    size_t pool_stride;    // candidate entries per CTA = fb * cuts_max
    size_t trk_stride;     // track entries per CTA = fb * max_tracks
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

size_t smem_bytes();
cudaError_t launch_filter(int mode, const KArgs& a, int grid, cudaStream_t s);
int blocks_per_sm(int mode);

}  // namespace m3e
