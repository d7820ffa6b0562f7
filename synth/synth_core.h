/*
 * synth_core.h -- seeded synthetic Mu3e time-frame generator (input synthesis only).
 *
 * This module produces the INPUTS that both the CPU oracle (oracle/) and the CUDA
 * path (paper_2206_11535_b200/) consume.  It contains none of the filter's
 * arithmetic (no selection cuts, no triplet fit, no vertex estimate); it is a
 * forward simulation of charged particles in a solenoid:
 *
 *   - muons decay at rest on the surface of the double hollow-cone target
 *     (Sec. III-B "double hollow cone target"; Fig. 3 target polygon
 *     +-50 mm x 19 mm; Sec. IV-C "disk with a radius of 19mm");
 *   - background: Michel decays mu+ -> e+ nu nu (Sec. III-A,
 *     "Michel decay ... branching ratio of ~100%"), spectrum x^2(3-2x);
 *   - signal: mu+ -> e+ e- e+ with sum p = 0 and sum E = m_mu (Eq. 1),
 *     uniform three-body phase space;
 *   - helices in a 1 T field along +z (Sec. III-B "1T magnetic field");
 *   - four concentric cylindrical pixel layers (Sec. IV-A "a set of four
 *     concentric cylinders"), Gaussian multiple-scattering kink at every layer
 *     crossed (Highland, Sec. IV-B refs. [Highland1975, Lynch1991]),
 *     Gaussian pixel smearing along the cylinder surface;
 *   - uniform noise hits on the layer surfaces;
 *   - frames of 64 ns (Sec. VI "64 ns long frames"), Poisson number of
 *     decays with mean muon_rate * 64 ns.
 *
 * Every random number is drawn from a counter-based stream keyed by
 * (seed, frame_id), so any frame can be regenerated independently and in any
 * order (used for the two-pass count/write scheme and for thread parallelism).
 *
 * The code is plain C99 usable from gcc (host) and nvcc (device) through SYN_HD.
 */
#ifndef M3E_SYNTH_CORE_H
#define M3E_SYNTH_CORE_H

#include <stdint.h>
#include <math.h>

#ifdef __CUDACC__
#define SYN_HD __host__ __device__ static inline
#else
#define SYN_HD static inline
#endif

#define SYN_PI 3.14159265358979323846
#define SYN_M_MU 105.6583755      /* MeV, PDG */
#define SYN_M_E 0.51099895        /* MeV, PDG */
#define SYN_PT_CONV 0.299792458   /* MeV/c per (T mm) */
#define SYN_MAX_PARTICLES 512     /* per frame; far above 1e9 mu/s * 64 ns */

typedef struct synth_cfg {
    double muon_rate;        /* mu/s */
    double frame_ns;         /* frame length, ns */
    double signal_fraction;  /* probability that a frame carries one injected mu->eee */
    int fixed_michel;        /* >=0: exact number of Michel decays per frame, else Poisson */
    int fixed_signal;        /* >=0: exact number of signal decays per frame, else Bernoulli */
    double noise_per_layer;  /* mean number of noise hits per layer per frame */
    double x_over_x0;        /* material per layer crossing at normal incidence */
    double sigma_pixel;      /* mm, Gaussian smearing along the surface */
    int ms_on;               /* multiple scattering on/off */
    int normal_incidence;    /* 1: MS width ignores the crossing angle */
    uint64_t seed;
    double layer_r[4];       /* mm */
    double layer_half[4];    /* mm, half length of each layer */
    double b_field;          /* T, along +z */
    double target_r;         /* mm, cone base radius */
    double target_half;      /* mm, cone half length */
} synth_cfg;

/* one generated particle (truth) */
typedef struct synth_particle {
    int kind;        /* 0 michel e+, 1 signal e+, 2 signal e-, 3 noise (unused) */
    int charge;      /* +1 / -1 */
    int decay;       /* decay index within the frame */
    int layer_mask;  /* bit l set if the particle left a hit in layer l */
    double p[3];     /* momentum at production, MeV/c */
    double v[3];     /* production vertex, mm */
} synth_particle;

/* ---------------------------------------------------------------- RNG ---- */
typedef struct { uint64_t s; } syn_rng;

SYN_HD uint64_t syn_mix(uint64_t z) {
    z += 0x9E3779B97F4A7C15ull;
    z = (z ^ (z >> 30)) * 0xBF58476D1CE4E5B9ull;
    z = (z ^ (z >> 27)) * 0x94D049BB133111EBull;
    return z ^ (z >> 31);
}
SYN_HD syn_rng syn_rng_frame(uint64_t seed, uint64_t frame_id) {
    syn_rng r;
    r.s = syn_mix(syn_mix(seed) ^ (frame_id * 0xD1B54A32D192ED03ull + 0x632BE59BD9B4E019ull));
    return r;
}
SYN_HD uint64_t syn_next(syn_rng* r) {
    r->s += 0x9E3779B97F4A7C15ull;
    uint64_t z = r->s;
    z = (z ^ (z >> 30)) * 0xBF58476D1CE4E5B9ull;
    z = (z ^ (z >> 27)) * 0x94D049BB133111EBull;
    return z ^ (z >> 31);
}
/* uniform in [0,1) */
SYN_HD double syn_uniform(syn_rng* r) { return (double)(syn_next(r) >> 11) * (1.0 / 9007199254740992.0); }
/* uniform in (0,1] */
SYN_HD double syn_uniform_pos(syn_rng* r) { return 1.0 - syn_uniform(r); }
SYN_HD double syn_gauss(syn_rng* r) {
    double u1 = syn_uniform_pos(r), u2 = syn_uniform(r);
    return sqrt(-2.0 * log(u1)) * cos(2.0 * SYN_PI * u2);
}
SYN_HD int syn_poisson(syn_rng* r, double mean) {
    if (mean <= 0.0) return 0;
    if (mean < 200.0) { /* Knuth */
        double L = exp(-mean), p = 1.0;
        int k = 0;
        do { ++k; p *= syn_uniform(r); } while (p > L);
        return k - 1;
    }
    int k = (int)floor(mean + sqrt(mean) * syn_gauss(r) + 0.5); /* normal approx */
    return k < 0 ? 0 : k;
}

/* --------------------------------------------------------- kinematics ---- */
SYN_HD void syn_isotropic(syn_rng* r, double u[3]) {
    double c = 2.0 * syn_uniform(r) - 1.0, s = sqrt(fmax(0.0, 1.0 - c * c));
    double ph = 2.0 * SYN_PI * syn_uniform(r);
    u[0] = s * cos(ph); u[1] = s * sin(ph); u[2] = c;
}

/* decay point uniform on the lateral surface of the double cone
 * rho(z) = R (1 - |z|/L), |z| <= L (area element ~ rho(z) dz) */
SYN_HD void syn_target_point(syn_rng* r, const synth_cfg* c, double v[3]) {
    double a = c->target_half * (1.0 - sqrt(syn_uniform(r)));  /* |z| with density ~ (1-|z|/L) */
    double z = (syn_uniform(r) < 0.5) ? -a : a;
    double rho = c->target_r * (1.0 - a / c->target_half);
    double ph = 2.0 * SYN_PI * syn_uniform(r);
    v[0] = rho * cos(ph); v[1] = rho * sin(ph); v[2] = z;
}

/* Michel positron momentum: x = p/p_max with density ~ x^2 (3 - 2x) */
SYN_HD double syn_michel_p(syn_rng* r) {
    double emax = (SYN_M_MU * SYN_M_MU + SYN_M_E * SYN_M_E) / (2.0 * SYN_M_MU);
    double pmax = sqrt(emax * emax - SYN_M_E * SYN_M_E);
    for (;;) {
        double x = syn_uniform(r);
        if (syn_uniform(r) < x * x * (3.0 - 2.0 * x)) return x * pmax;
    }
}

/* uniform random rotation (Shoemake quaternion) applied to vector v in place */
SYN_HD void syn_random_rotate(syn_rng* r, double v[3][3]) {
    double u1 = syn_uniform(r), u2 = syn_uniform(r), u3 = syn_uniform(r);
    double a = sqrt(1.0 - u1), b = sqrt(u1);
    double qw = a * sin(2 * SYN_PI * u2), qx = a * cos(2 * SYN_PI * u2);
    double qy = b * sin(2 * SYN_PI * u3), qz = b * cos(2 * SYN_PI * u3);
    double R[3][3] = {
        {1 - 2 * (qy * qy + qz * qz), 2 * (qx * qy - qz * qw), 2 * (qx * qz + qy * qw)},
        {2 * (qx * qy + qz * qw), 1 - 2 * (qx * qx + qz * qz), 2 * (qy * qz - qx * qw)},
        {2 * (qx * qz - qy * qw), 2 * (qy * qz + qx * qw), 1 - 2 * (qx * qx + qy * qy)}};
    for (int i = 0; i < 3; ++i) {
        double t0 = v[i][0], t1 = v[i][1], t2 = v[i][2];
        v[i][0] = R[0][0] * t0 + R[0][1] * t1 + R[0][2] * t2;
        v[i][1] = R[1][0] * t0 + R[1][1] * t1 + R[1][2] * t2;
        v[i][2] = R[2][0] * t0 + R[2][1] * t1 + R[2][2] * t2;
    }
}

/* mu+ -> e+ e+ e- at rest: uniform Dalitz plot (E1,E2), then random orientation.
 * Output momenta p[0],p[1] (e+), p[2] (e-); sum p = 0, sum E = m_mu exactly
 * up to rounding (Eq. 1). */
SYN_HD void syn_signal_momenta(syn_rng* r, double p[3][3]) {
    const double M = SYN_M_MU, m = SYN_M_E;
    for (;;) {
        double E1 = m + syn_uniform(r) * (0.5 * M - m);
        double E2 = m + syn_uniform(r) * (0.5 * M - m);
        double E3 = M - E1 - E2;
        if (E3 < m) continue;
        double p1 = sqrt(E1 * E1 - m * m), p2 = sqrt(E2 * E2 - m * m), p3 = sqrt(E3 * E3 - m * m);
        if (p3 > p1 + p2 || p3 < fabs(p1 - p2) || p1 <= 0.0 || p2 <= 0.0) continue;
        double c12 = (p3 * p3 - p1 * p1 - p2 * p2) / (2.0 * p1 * p2);
        if (c12 > 1.0) c12 = 1.0;
        if (c12 < -1.0) c12 = -1.0;
        double s12 = sqrt(1.0 - c12 * c12);
        p[0][0] = 0; p[0][1] = 0; p[0][2] = p1;
        p[1][0] = p2 * s12; p[1][1] = 0; p[1][2] = p2 * c12;
        p[2][0] = -p[0][0] - p[1][0]; p[2][1] = -p[0][1] - p[1][1]; p[2][2] = -p[0][2] - p[1][2];
        syn_random_rotate(r, p);
        return;
    }
}

/* Highland width (PDG) for one layer crossing */
SYN_HD double syn_highland(double p, double x0frac) {
    double E = sqrt(p * p + SYN_M_E * SYN_M_E), beta = p / E;
    return 13.6 / (beta * p) * sqrt(x0frac) * (1.0 + 0.038 * log(x0frac));
}

/* ---------------------------------------------------------- transport ---- */
/* Sink for hits: count mode (hits == 0) or write mode. */
typedef struct syn_sink {
    uint32_t count[4];          /* hits emitted per layer so far */
    /* write mode: */
    float* x; float* y; float* z;   /* global SoA arrays (may be NULL in count mode) */
    uint32_t base[4];           /* global index of first hit of each layer of this frame */
    int32_t* hit_particle;      /* optional truth: particle index (-1 noise) per hit */
} syn_sink;

SYN_HD void syn_emit(syn_sink* s, int layer, double x, double y, double z, int particle) {
    uint32_t k = s->count[layer]++;
    if (s->x) {
        uint32_t g = s->base[layer] + k;
        s->x[g] = (float)x; s->y[g] = (float)y; s->z[g] = (float)z;
        if (s->hit_particle) s->hit_particle[g] = particle;
    }
}

/*
 * Transport one particle outward through the four layers.  Helix in B along +z:
 * a positive charge turns clockwise seen from +z.  Each layer crossing inside
 * the layer's z extent leaves a hit (smeared along the surface) and applies a
 * Gaussian MS kink.  Returns the layer mask of hits left; the hit positions
 * are returned in hx/hy/hz (valid where the mask bit is set).
 */
SYN_HD int syn_transport(syn_rng* r, const synth_cfg* c, int q, const double v0[3], const double p0[3],
                         double hx[4], double hy[4], double hz[4]) {
    double x = v0[0], y = v0[1], z = v0[2];
    double px = p0[0], py = p0[1], pz = p0[2];
    double pabs = sqrt(px * px + py * py + pz * pz);
    int mask = 0;
    for (int l = 0; l < 4; ++l) {
        double pt = sqrt(px * px + py * py);
        if (pt <= 1e-9) break;
        double Rt = pt / (SYN_PT_CONV * c->b_field);
        double psi = atan2(py, px);
        double cx = x + q * Rt * sin(psi), cy = y - q * Rt * cos(psi);
        double phi0 = atan2(y - cy, x - cx);
        double C = sqrt(cx * cx + cy * cy);
        double rho = c->layer_r[l];
        if (C < 1e-12) break;
        double arg = (rho * rho - C * C - Rt * Rt) / (2.0 * Rt * C);
        if (arg > 1.0 || arg < -1.0) break;              /* helix never reaches this layer */
        double phic = atan2(cy, cx), dphi = acos(arg);
        double best = 1e300;
        for (int s = -1; s <= 1; s += 2) {
            double ph = phic + s * dphi;
            double t = q * (phi0 - ph);                     /* turning angle, mod 2 pi */
            t = fmod(t, 2.0 * SYN_PI);
            if (t < 0) t += 2.0 * SYN_PI;
            if (t > 1e-12 && t < best) best = t;
        }
        if (best > 2.0 * SYN_PI) break;
        double ph = phi0 - q * best;
        double nx = cx + Rt * cos(ph), ny = cy + Rt * sin(ph);
        double nz = z + (pz / pt) * Rt * best;
        double npsi = psi - q * best;
        x = nx; y = ny; z = nz;
        px = pt * cos(npsi); py = pt * sin(npsi);
        if (fabs(z) > c->layer_half[l]) continue;          /* passes outside the layer's z extent */
        /* hit, smeared along the surface (keeps radius rho) */
        double phih = atan2(y, x) + (c->sigma_pixel > 0 ? c->sigma_pixel / rho * syn_gauss(r) : 0.0);
        double zh = z + (c->sigma_pixel > 0 ? c->sigma_pixel * syn_gauss(r) : 0.0);
        hx[l] = rho * cos(phih); hy[l] = rho * sin(phih); hz[l] = zh;
        mask |= 1 << l;
        /* multiple scattering kink */
        if (c->ms_on) {
            double ux = px / pabs, uy = py / pabs, uz = pz / pabs;
            double X = c->x_over_x0;
            if (!c->normal_incidence) {
                double cosinc = fabs(ux * x + uy * y) / rho;   /* cos of angle to the surface normal */
                if (cosinc < 0.05) cosinc = 0.05;
                X /= cosinc;
            }
            double sig = syn_highland(pabs, X);
            /* e1 = unit(z x u), e2 = u x e1 */
            double e1x = -uy, e1y = ux, e1n = sqrt(e1x * e1x + e1y * e1y);
            e1x /= e1n; e1y /= e1n;
            double e2x = uy * 0 - uz * e1y, e2y = uz * e1x - ux * 0, e2z = ux * e1y - uy * e1x;
            double g1 = sig * syn_gauss(r), g2 = sig * syn_gauss(r);
            double wx = ux + g1 * e1x + g2 * e2x, wy = uy + g1 * e1y + g2 * e2y, wz = uz + g2 * e2z;
            double wn = sqrt(wx * wx + wy * wy + wz * wz);
            px = pabs * wx / wn; py = pabs * wy / wn; pz = pabs * wz / wn;
        }
    }
    return mask;
}

/*
 * Generate frame `frame_id` into sink `s`.  Hits are emitted grouped by layer
 * (layer 0 first), inside a layer in particle order, noise hits last.
 * If `parts` is non-NULL the particle truth table is written there (returns
 * the number of particles, <= SYN_MAX_PARTICLES).
 */
SYN_HD int synth_frame(const synth_cfg* c, uint64_t frame_id, syn_sink* s, synth_particle* parts) {
    syn_rng r = syn_rng_frame(c->seed, frame_id);
    int n_sig = c->fixed_signal >= 0 ? c->fixed_signal : (syn_uniform(&r) < c->signal_fraction ? 1 : 0);
    int n_mich = c->fixed_michel >= 0 ? c->fixed_michel : syn_poisson(&r, c->muon_rate * c->frame_ns * 1e-9);
    int np = 0;
    /* Hits are written through per-layer cursors (base[l] + count[l]), so each
       particle's hits can be emitted as soon as it is transported: inside a layer
       the order is particle order, and noise hits (drawn last) come after them. */
    for (int d = 0; d < n_sig + n_mich; ++d) {
        double v[3];
        syn_target_point(&r, c, v);
        int is_sig = d < n_sig;
        double pm[3][3];
        int npart;
        if (is_sig) {
            syn_signal_momenta(&r, pm);
            npart = 3;
        } else {
            double u[3], p = syn_michel_p(&r);
            syn_isotropic(&r, u);
            pm[0][0] = p * u[0]; pm[0][1] = p * u[1]; pm[0][2] = p * u[2];
            npart = 1;
        }
        for (int k = 0; k < npart; ++k) {
            if (np >= SYN_MAX_PARTICLES) break;
            int q = (is_sig && k == 2) ? -1 : +1;
            double tx[4], ty[4], tz[4];
            int mask = syn_transport(&r, c, q, v, pm[k], tx, ty, tz);
            for (int l = 0; l < 4; ++l)
                if (mask >> l & 1) syn_emit(s, l, tx[l], ty[l], tz[l], np);
            if (parts) {
                synth_particle* P = &parts[np];
                P->kind = is_sig ? (q > 0 ? 1 : 2) : 0;
                P->charge = q;
                P->decay = d;
                P->layer_mask = mask;
                for (int i = 0; i < 3; ++i) { P->p[i] = pm[k][i]; P->v[i] = v[i]; }
            }
            ++np;
        }
    }
    for (int l = 0; l < 4; ++l) {
        int nn = syn_poisson(&r, c->noise_per_layer);
        for (int k = 0; k < nn; ++k) {
            double ph = 2.0 * SYN_PI * syn_uniform(&r);
            double zz = (2.0 * syn_uniform(&r) - 1.0) * c->layer_half[l];
            syn_emit(s, l, c->layer_r[l] * cos(ph), c->layer_r[l] * sin(ph), zz, -1);
        }
    }
    return np;
}

#endif
