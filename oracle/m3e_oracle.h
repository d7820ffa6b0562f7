/*
 * m3e_oracle.h -- CPU reference ("oracle") of the Mu3e online event selection
 * (PAPER.md = arXiv 2206.11535, Henkys, Schmidt, Berger).
 *
 * TEST INFRASTRUCTURE ONLY.  Plain, slow, fp64, single-threaded C written
 * from the paper.  Only tests/, __graft_entry__.smoke() and bench.py's
 * cpu_baseline / --impl reference leg may load it.  It shares no code, header,
 * table or constant with the CUDA path (paper_2206_11535_b200/), and the CUDA
 * path never calls it.
 *
 * Every function cites the PAPER.md passage it follows; where the paper is
 * silent or garbled the reading taken is named R<n> and listed in DESIGN.md
 * ("Readings of the paper").
 *
 * Parity status: every function is pinned by tests/test_oracle_*.py except
 * where a comment says "parity unpinned" (none at present).
 */
#ifndef M3E_ORACLE_H
#define M3E_ORACLE_H
#include <stdint.h>

#define OR_REASON_NONE 0
#define OR_REASON_TRIPLET_OVERFLOW 1 /* Sec. V-B "too many triplets ... marked for storage" */
#define OR_REASON_TRACK_OVERFLOW 2   /* Alg. 3 / Sec. V-B "too many tracks" */
#define OR_REASON_COMB_OVERFLOW 3    /* Alg. 4 "num_track_combs > max_tracks" */
#define OR_REASON_VERTEX 4           /* Alg. 4 "keep_frame <- true" */

typedef struct or_params {
    double layer_r[4];    /* mm, cylinder radii r_{t,i} (Sec. IV-A simplification) */
    double b_field;       /* T */
    double target_r;      /* mm, 19 (Sec. IV-C) */
    double target_half;   /* mm, 50 (Fig. 3 target polygon) */
    /* Selection Cuts, Sec. IV-A / Alg. 2 */
    double dlambda_max;   /* |Delta lambda| <= dlambda_max          (Eq. 3) */
    double cos_phi01_min; /* cos Phi_01 >= cos_phi01_min            (Eq. 4) */
    double cos_phi12_min; /* cos Phi_12 >= cos_phi12_min            (Eq. 4) */
    double rt_min;        /* rt_min <= |r_tc| <= rt_max             (Eq. 5) */
    double rt_max;
    int cuts_max;         /* 768 (Sec. VI) */
    /* Track reconstruction, Sec. IV-B / Alg. 3 */
    double x_over_x0;     /* material per layer for sigma_MS (Highland) */
    double chi2_max;      /* 32 (Sec. IV-B) */
    int max_tracks;
    /* Vertex fit, Sec. IV-C / Alg. 4 */
    double e_window;      /* |E_a + E_b + E_e - m_mu| <= e_window */
    double xy_margin;     /* intersections kept if |p| <= target_r + xy_margin */
    double sigma_pixel;   /* mm (Eq. 10) */
    double chi2_vertex_max;
    double target_dist_max;
    double p_total_max;
    int max_combs;
    double rel_band;      /* relative band for "near threshold" flags (north_star: 1e-5) */
} or_params;

typedef struct or_candidate {
    int32_t i0, i1, i2;   /* layer-local hit indices */
    int32_t marginal;     /* an evaluated cut variable lay within rel_band of its threshold */
    double rtc;           /* signed Eq. 5 radius, cached for the fit (Sec. IV-A last paragraph) */
} or_candidate;

/* one single-triplet fit (Sec. IV-B-1) */
typedef struct or_triplet_fit {
    int32_t ok;           /* 0: degenerate triplet */
    int32_t q;            /* +1 clockwise (e+ in B along +z), -1 counter-clockwise */
    double rtc;           /* signed circle radius (Eq. 5) */
    double phi_c[2];      /* circle-solution bending angle of arc 01 and 12 */
    double k_c[2];        /* circle-solution 3D curvature of each arc */
    double theta_c[2];    /* circle-solution polar angle of each arc */
    double dphi[2];       /* dPhi_ij/dk at k_c[ij] */
    double dtheta[2];     /* dtheta_ij/dk at k_c[ij] */
    double a_phi, b_phi;  /* linearised Phi_MS(k) = a_phi + b_phi k */
    double a_theta, b_theta; /* linearised Theta_MS(k) = a_theta + b_theta k */
    double sigma_ms, w_phi, w_theta;
    double k_hat;         /* minimiser of the linearised chi2 (|kappa|) */
    double kappa;         /* q * k_hat */
    double var_kappa;     /* sigma^2_{kappa,t} */
    double chi2;          /* chi2_t(k_hat) */
} or_triplet_fit;

#define OR_FIT_OK 0
#define OR_FIT_DEGENERATE1 1
#define OR_FIT_NO_REACH 2
#define OR_FIT_LAYER3_EMPTY 3
#define OR_FIT_DEGENERATE2 4
#define OR_FIT_CHI2 5
#define OR_FIT_DOMAIN 6

typedef struct or_track {
    int32_t cand;         /* candidate index */
    int32_t hit[4];       /* layer-local hit indices (layer 0..3) */
    int32_t status;       /* OR_FIT_* */
    int32_t accepted;     /* chi2_global < chi2_max */
    int32_t marginal;     /* a decision of this fit lay within rel_band of its threshold */
    int32_t q;            /* sign(kappa) */
    int32_t pad;
    or_triplet_fit t1, t2;
    double pred[3];       /* layer-3 point predicted from the first triplet */
    double kappa;         /* global kappa-bar (Eq. 8), signed */
    double var_kappa;
    double chi2;          /* chi2_global(kappa-bar) (Eq. 7) */
    double cos_theta01;   /* cos of polar angle of arc 01 at |kappa-bar| (= sin lambda_01) */
    double cx, cy, rt;    /* transverse circle of the track (Sec. IV-C) */
    double p, energy;     /* MeV/c, MeV */
} or_track;

/* vertex-stage view of one track (the inputs Sec. IV-C uses) */
typedef struct or_vtrack {
    double kappa;         /* signed 3D curvature, 1/mm */
    double cos_theta01;
    double cx, cy;
    double h0[3];         /* layer-0 hit */
} or_vtrack;

typedef struct or_vertex {
    int32_t a, b, e;      /* indices into the e+ / e+ / e- tracks (frame track list) */
    int32_t pass;         /* passed chi2, target and momentum tests */
    double x, y, z, chi2, target_dist, p_total;
} or_vertex;

typedef struct or_frame_result {
    int32_t reason;       /* OR_REASON_* */
    int32_t keep;
    int32_t n_cand;       /* min(#survivors, cuts_max + 1) */
    int32_t n_cand_marginal;
    int64_t funnel[5];    /* combos evaluated / passed d-lambda / phi01 / phi12 / r_t (Fig. 4) */
    int32_t n_fit;        /* candidates fitted */
    int32_t n_tracks;     /* min(#accepted, max_tracks + 1) */
    int32_t n_fit_marginal;
    int32_t n_pos, n_neg; /* accepted tracks by charge (stored ones) */
    int32_t n_combs;      /* min(#energy-passing triples, max_combs + 1) */
    int32_t n_vertex_marginal;
    int32_t has_vertex;
    or_vertex vertex;     /* best (lowest chi2) passing vertex if keep by reason 4 */
} or_frame_result;

#ifdef __cplusplus
extern "C" {
#endif
/* geometry primitives */
double or_tan_lambda(double zi, double zj, double ri, double rj);
double or_cos_phi(double xi, double yi, double xj, double yj, double ri, double rj);
double or_circle_radius(const double h0[3], const double h1[3], const double h2[3]);
double or_arc_phi(double d, double z, double k);
double or_highland(double p, double x_over_x0);
double or_target_distance(const or_params* P, double x, double y, double z);
int or_circle_intersections(double c1x, double c1y, double r1, double c2x, double c2y, double r2,
                            double out[4], double band, int* marginal);
/* exact (non-linearised) scattering angles of a hit triplet at 3D curvature k, charge sense q */
int or_scattering_angles(const double h0[3], const double h1[3], const double h2[3], int q, double k,
                         double* phi_ms, double* theta_ms);
/* stages */
int or_fit_triplet(const or_params* P, const double h0[3], const double h1[3], const double h2[3],
                   or_triplet_fit* out);
int or_extrapolate(const or_params* P, const double h1[3], const double h2[3], int q, double k,
                   double out[3]);
int or_select(const or_params* P, const float* x, const float* y, const float* z, const uint32_t start[5],
              or_candidate* cand, int cap, or_frame_result* res);
int or_fit_candidate(const or_params* P, const float* x, const float* y, const float* z,
                     const uint32_t start[5], const or_candidate* c, or_track* out);
/* reading R11 at a given signed kappa (used by or_fit_candidate; exported so the
 * tests can propagate the kappa tolerance through the vertex stage) */
int or_track_params(const or_params* P, const double h0[3], const double h1[3], double kappa, or_track* o);
int or_vertex_frame(const or_params* P, const or_vtrack* tracks, int n, or_frame_result* res,
                    or_vertex* all_out, int all_cap);
int or_process_frame(const or_params* P, const float* x, const float* y, const float* z,
                     const uint32_t start[5], or_frame_result* res, or_candidate* cand_buf,
                     or_track* track_buf);
int64_t or_process_frames(const or_params* P, const float* x, const float* y, const float* z,
                          const uint32_t* offsets, int64_t n_frames, or_frame_result* res);
int or_sizeof(int which);
#ifdef __cplusplus
}
#endif
#endif
