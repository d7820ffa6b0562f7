/*
 * synth_host.c -- host driver of the synthetic frame generator (see synth_core.h).
 * Two-pass layout: synth_count() gives per-frame per-layer hit counts, the caller
 * builds the offsets array (4*F+1 entries: offsets[4f+l] = first hit of layer l of
 * frame f, offsets[4F] = total), synth_write() fills the SoA arrays.
 * Frames are independent, so both passes split the frame range over pthreads.
 */
#include "synth_core.h"
#include <pthread.h>
#include <stdlib.h>
#include <string.h>

typedef struct {
    const synth_cfg* c;
    uint64_t frame0, lo, hi;
    uint32_t* counts;
    const uint32_t* offsets;
    float *x, *y, *z;
    int32_t* hp;
} job_t;

static void* count_worker(void* arg) {
    job_t* j = (job_t*)arg;
    for (uint64_t i = j->lo; i < j->hi; ++i) {
        syn_sink s;
        memset(&s, 0, sizeof s);
        synth_frame(j->c, j->frame0 + i, &s, NULL);
        for (int l = 0; l < 4; ++l) j->counts[4 * i + l] = s.count[l];
    }
    return NULL;
}

static void* write_worker(void* arg) {
    job_t* j = (job_t*)arg;
    for (uint64_t i = j->lo; i < j->hi; ++i) {
        syn_sink s;
        memset(&s, 0, sizeof s);
        s.x = j->x; s.y = j->y; s.z = j->z; s.hit_particle = j->hp;
        for (int l = 0; l < 4; ++l) s.base[l] = j->offsets[4 * i + l];
        synth_frame(j->c, j->frame0 + i, &s, NULL);
    }
    return NULL;
}

static int run(job_t proto, uint64_t n, int nt, void* (*fn)(void*)) {
    if (nt < 1) nt = 1;
    if (nt > 256) nt = 256;
    if ((uint64_t)nt > n) nt = n ? (int)n : 1;
    pthread_t th[256];
    job_t jobs[256];
    for (int t = 0; t < nt; ++t) {
        jobs[t] = proto;
        jobs[t].lo = n * t / nt;
        jobs[t].hi = n * (t + 1) / nt;
        if (pthread_create(&th[t], NULL, fn, &jobs[t])) return -1;
    }
    for (int t = 0; t < nt; ++t) pthread_join(th[t], NULL);
    return 0;
}

int synth_count(const synth_cfg* c, uint64_t frame0, uint64_t n, uint32_t* counts, int nthreads) {
    job_t j;
    memset(&j, 0, sizeof j);
    j.c = c; j.frame0 = frame0; j.counts = counts;
    return run(j, n, nthreads, count_worker);
}

int synth_write(const synth_cfg* c, uint64_t frame0, uint64_t n, const uint32_t* offsets,
                float* x, float* y, float* z, int32_t* hit_particle, int nthreads) {
    job_t j;
    memset(&j, 0, sizeof j);
    j.c = c; j.frame0 = frame0; j.offsets = offsets; j.x = x; j.y = y; j.z = z; j.hp = hit_particle;
    return run(j, n, nthreads, write_worker);
}

/* truth particle table of one frame; returns the number of particles */
int synth_particles(const synth_cfg* c, uint64_t frame_id, synth_particle* out, int max_out) {
    static __thread synth_particle buf[SYN_MAX_PARTICLES];
    syn_sink s;
    memset(&s, 0, sizeof s);
    int n = synth_frame(c, frame_id, &s, buf);
    if (n > max_out) n = max_out;
    memcpy(out, buf, (size_t)n * sizeof(synth_particle));
    return n;
}

int synth_sizeof_cfg(void) { return (int)sizeof(synth_cfg); }
int synth_sizeof_particle(void) { return (int)sizeof(synth_particle); }
