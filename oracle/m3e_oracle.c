/*
 * m3e_oracle.c -- CPU reference of the Mu3e online event selection, fp64.
 * TEST INFRASTRUCTURE ONLY (see m3e_oracle.h).  No blocking, fusion or
 * reordering beyond what the paper states; loops follow Alg. 2-4 literally.
 */
#include "m3e_oracle.h"

#include <math.h>
#include <stdlib.h>
#include <string.h>

#define PI 3.14159265358979323846
#define M_MU 105.6583755     /* MeV, PDG; m_mu c^2 of Eq. 1 */
#define M_E 0.51099895       /* MeV, PDG */
#define PT_CONV 0.299792458  /* p [MeV/c] = PT_CONV * B [T] * R [mm] */

static int near(double v, double thr, double band) { return fabs(v - thr) <= band * fabs(thr); }

static double wrap_pi(double a) { /* to (-pi, pi] */
    while (a > PI) a -= 2 * PI;
    while (a <= -PI) a += 2 * PI;
    return a;
}

/* ------------------------------------------------------------------------ */
/* Sec. IV-A, Eq. 2: tan lambda_ij = (z_j - z_i) / (r_{t,j} - r_{t,i}), with the
 * cylinder simplification h_{t,k} = r_{t,i} (layer radius, not hit radius). */
double or_tan_lambda(double zi, double zj, double ri, double rj) { return (zj - zi) / (rj - ri); }

/* Sec. IV-A, Eq. 4: cos Phi_ij = h_{t,i} . h_{t,j} / (r_{t,i} r_{t,j}). */
double or_cos_phi(double xi, double yi, double xj, double yj, double ri, double rj) {
    return (xi * xj + yi * yj) / (ri * rj);
}

/* Sec. IV-A, Eq. 5: r_{t,c} = d01 d12 d20 / (2 [(h0 - h1) x (h2 - h1)]_z), transverse
 * components only.  Signed: > 0 for clockwise h0 -> h1 -> h2 (a positive charge in
 * B along +z, reading R5).  Collinear -> +inf (fails every r_t window). */
double or_circle_radius(const double h0[3], const double h1[3], const double h2[3]) {
    double d01 = hypot(h0[0] - h1[0], h0[1] - h1[1]);
    double d12 = hypot(h1[0] - h2[0], h1[1] - h2[1]);
    double d20 = hypot(h2[0] - h0[0], h2[1] - h0[1]);
    double cz = (h0[0] - h1[0]) * (h2[1] - h1[1]) - (h0[1] - h1[1]) * (h2[0] - h1[0]);
    if (cz == 0.0) return INFINITY;
    return d01 * d12 * d20 / (2.0 * cz);
}

/* Highland width (Sec. IV-B "variances given by MS theory" [Highland1975, Lynch1991]);
 * reading R7: beta = 1, thickness x/X0 per layer at normal incidence. */
double or_highland(double p, double x_over_x0) {
    return 13.6 / p * sqrt(x_over_x0) * (1.0 + 0.038 * log(x_over_x0));
}

/* ------------------------------------------------------------------------ */
/* Helix arc between two hits (Fig. 5): a helix of 3D radius R = 1/k whose
 * transverse projection bends by Phi between hits with transverse chord d and
 * longitudinal distance z satisfies
 *     d = 2 R sin(theta) sin(Phi/2),   z = R cos(theta) Phi
 * so  R^2 = d^2 / (4 sin^2(Phi/2)) + z^2 / Phi^2          (reading R6)
 * The left side is strictly decreasing on (0, pi]; the short-arc root is returned,
 * NaN if 1/k^2 < d^2/4 + z^2/pi^2 (no short arc of that radius joins the hits). */
static double arc_f(double phi, double d, double z) {
    double s = sin(0.5 * phi);
    return d * d / (4.0 * s * s) + z * z / (phi * phi);
}
double or_arc_phi(double d, double z, double k) {
    if (!(k > 0.0) || !(d > 0.0)) return NAN;
    double R2 = 1.0 / (k * k);
    if (R2 < arc_f(PI, d, z)) return NAN;
    double lo = 0.0, hi = PI; /* f(lo) > R2 >= f(hi) */
    for (int it = 0; it < 200 && hi - lo > 1e-16 * hi; ++it) {
        double mid = 0.5 * (lo + hi);
        if (arc_f(mid, d, z) > R2) lo = mid; else hi = mid;
    }
    return 0.5 * (lo + hi);
}
static double arc_theta(double d, double z, double k) { /* cos theta = z k / Phi */
    double phi = or_arc_phi(d, z, k);
    double c = z * k / phi;
    if (c > 1.0) c = 1.0;
    if (c < -1.0) c = -1.0;
    return acos(c);
}

/* Exact scattering angles of Fig. 5 for a track of 3D curvature k and rotation
 * sense q through hits h0, h1, h2 (reading R6):
 *   Phi_MS   = heading of arc 12 at h1 - heading of arc 01 at h1
 *            = wrap(alpha_12 - alpha_01) + q (Phi_01 + Phi_12) / 2
 *              (alpha_ij = direction of the chord ij; a clockwise arc turns its
 *               heading by -Phi, so the chord sits half-way)
 *   Theta_MS = theta_12 - theta_01 (change of polar angle at h1). */
int or_scattering_angles(const double h0[3], const double h1[3], const double h2[3], int q, double k,
                         double* phi_ms, double* theta_ms) {
    double d01 = hypot(h1[0] - h0[0], h1[1] - h0[1]), d12 = hypot(h2[0] - h1[0], h2[1] - h1[1]);
    double z01 = h1[2] - h0[2], z12 = h2[2] - h1[2];
    double p01 = or_arc_phi(d01, z01, k), p12 = or_arc_phi(d12, z12, k);
    if (isnan(p01) || isnan(p12)) return -1;
    double a01 = atan2(h1[1] - h0[1], h1[0] - h0[0]), a12 = atan2(h2[1] - h1[1], h2[0] - h1[0]);
    *phi_ms = wrap_pi(a12 - a01) + q * 0.5 * (p01 + p12);
    *theta_ms = arc_theta(d12, z12, k) - arc_theta(d01, z01, k);
    return 0;
}

/*
 * Single Triplet Fit, Sec. IV-B-1, Eq. 6:
 *   chi2(k) = Phi_MS(k)^2 / sigma_Phi^2 + Theta_MS(k)^2 / sigma_Theta^2,
 *   sigma_Theta^2 = sigma_MS^2, sigma_Phi^2 = sigma_MS^2 / sin^2(theta)  (reading R8)
 * "linearize it around ... the solution where Phi_MS = 0. This solution forms a
 * circle in the transverse plane ... first order Taylor expansion around the
 * circle solution":
 *   circle solution of arc ij: Phi_C = 2 asin(d_ij / (2 r_tc)),
 *       k_C = 1 / sqrt(r_tc^2 + z_ij^2 / Phi_C^2), theta_C = acos(z_ij k_C / Phi_C);
 *   each arc's Phi_ij(k), theta_ij(k) is expanded to first order around its own
 *   k_C (derivatives by central differences of the exact arc relation);
 *   Phi_MS(k_C) = 0 at the circle solution, so
 *     Phi_MS(k)   ~ q/2 [Phi'_01 (k - k_C01) + Phi'_12 (k - k_C12)]
 *     Theta_MS(k) ~ (theta_C12 - theta_C01) + theta'_12 (k - k_C12) - theta'_01 (k - k_C01)
 *   and the quadratic chi2(k) is minimised in closed form; sigma_k^2 is the inverse
 *   curvature of chi2/2 (reading R6).
 * sigma_MS: Highland at the circle-solution momentum p = PT_CONV B / mean(k_C) (R7),
 * sin theta of the incoming arc 01 at the circle solution (R8).
 */
int or_fit_triplet(const or_params* P, const double h0[3], const double h1[3], const double h2[3],
                   or_triplet_fit* o) {
    memset(o, 0, sizeof *o);
    double rtc = or_circle_radius(h0, h1, h2);
    o->rtc = rtc;
    if (!isfinite(rtc)) return -1;
    o->q = rtc > 0 ? +1 : -1;
    double r = fabs(rtc);
    const double* H[3] = {h0, h1, h2};
    for (int a = 0; a < 2; ++a) {
        double d = hypot(H[a + 1][0] - H[a][0], H[a + 1][1] - H[a][1]);
        double z = H[a + 1][2] - H[a][2];
        double s = d / (2.0 * r);
        if (s > 1.0) s = 1.0;
        double phc = 2.0 * asin(s);
        double kc = 1.0 / sqrt(r * r + z * z / (phc * phc));
        double cth = z * kc / phc;
        o->phi_c[a] = phc;
        o->k_c[a] = kc;
        o->theta_c[a] = acos(cth > 1 ? 1 : (cth < -1 ? -1 : cth));
        double h = 1e-6 * kc;
        double pp = or_arc_phi(d, z, kc + h), pm = or_arc_phi(d, z, kc - h);
        if (isnan(pp) || isnan(pm)) return -1;
        o->dphi[a] = (pp - pm) / (2.0 * h);
        o->dtheta[a] = (arc_theta(d, z, kc + h) - arc_theta(d, z, kc - h)) / (2.0 * h);
    }
    int q = o->q;
    /* Phi_MS(k) = a_phi + b_phi k ; Theta_MS(k) = a_theta + b_theta k */
    o->b_phi = 0.5 * q * (o->dphi[0] + o->dphi[1]);
    o->a_phi = -0.5 * q * (o->dphi[0] * o->k_c[0] + o->dphi[1] * o->k_c[1]);
    o->b_theta = o->dtheta[1] - o->dtheta[0];
    o->a_theta = (o->theta_c[1] - o->theta_c[0]) - o->dtheta[1] * o->k_c[1] + o->dtheta[0] * o->k_c[0];
    double p0 = PT_CONV * P->b_field / (0.5 * (o->k_c[0] + o->k_c[1]));
    double sms = or_highland(p0, P->x_over_x0);
    double st = sin(o->theta_c[0]);
    o->sigma_ms = sms;
    o->w_theta = 1.0 / (sms * sms);
    o->w_phi = st * st / (sms * sms);
    double A = o->b_phi * o->b_phi * o->w_phi + o->b_theta * o->b_theta * o->w_theta;
    double B = o->a_phi * o->b_phi * o->w_phi + o->a_theta * o->b_theta * o->w_theta;
    if (!(A > 0.0)) return -1;
    o->k_hat = -B / A;
    o->kappa = q * o->k_hat;
    o->var_kappa = 1.0 / A;
    double fphi = o->a_phi + o->b_phi * o->k_hat, fth = o->a_theta + o->b_theta * o->k_hat;
    o->chi2 = fphi * fphi * o->w_phi + fth * fth * o->w_theta;
    o->ok = 1;
    return 0;
}

/* chi2_t of Eq. 6 in the linearised model at signed global curvature kappa (Eq. 7) */
static double triplet_chi2_at(const or_triplet_fit* t, double kappa) {
    double k = t->q * kappa;
    double fphi = t->a_phi + t->b_phi * k, fth = t->a_theta + t->b_theta * k;
    return fphi * fphi * t->w_phi + fth * fth * t->w_theta;
}

/*
 * Sec. IV-B-2: "Using this preliminary helix, the hit position in the fourth layer
 * is estimated."  Reading R9: the helix of 3D curvature k and sense q is continued
 * from h2 with the heading and polar angle the arc h1 -> h2 has at h2 (exact arc
 * relation at k); its transverse circle (radius sin(theta_12)/k) is intersected
 * with the layer-3 cylinder at the first crossing reached moving forward;
 * z grows by cos(theta_12)/k per radian turned.
 */
int or_extrapolate(const or_params* P, const double h1[3], const double h2[3], int q, double k,
                   double out[3]) {
    double d12 = hypot(h2[0] - h1[0], h2[1] - h1[1]), z12 = h2[2] - h1[2];
    double phi12 = or_arc_phi(d12, z12, k);
    if (isnan(phi12)) return -1;
    double cth = z12 * k / phi12;
    if (cth > 1) cth = 1;
    if (cth < -1) cth = -1;
    double sth = sqrt(1.0 - cth * cth);
    double a12 = atan2(h2[1] - h1[1], h2[0] - h1[0]);
    double psi = a12 - q * 0.5 * phi12;                    /* heading at h2 */
    double rt = sth / k;
    double cx = h2[0] + q * rt * sin(psi), cy = h2[1] - q * rt * cos(psi);
    double rho = P->layer_r[3];
    double C = hypot(cx, cy);
    if (C == 0.0) return -1;
    double arg = (rho * rho - C * C - rt * rt) / (2.0 * rt * C);
    if (arg > 1.0 || arg < -1.0) return -1;                /* never reaches layer 3 */
    double phic = atan2(cy, cx), dphi = acos(arg);
    double phi0 = atan2(h2[1] - cy, h2[0] - cx);
    double best = INFINITY;
    for (int s = -1; s <= 1; s += 2) {
        double t = fmod(q * (phi0 - (phic + s * dphi)), 2 * PI);
        if (t < 0) t += 2 * PI;
        if (t > 0 && t < best) best = t;
    }
    double ph = phi0 - q * best;
    out[0] = cx + rt * cos(ph);
    out[1] = cy + rt * sin(ph);
    out[2] = h2[2] + cth / k * best;
    return 0;
}

/* ------------------------------------------------------------------------ */
/* Selection Cuts, Sec. IV-A + Alg. 2: all n0 n1 n2 combinations in row-major
 * order (i0 outer, i2 inner), tests in the order Delta-lambda, Phi_01, Phi_12
 * ("test_Phi02(hit_1, hit_2)" in Alg. 2 read as Phi_12, reading R2), r_tc; a
 * survivor is stored while fewer than cuts_max are stored.  n_cand reports
 * min(#survivors, cuts_max + 1): overflow <=> n_cand > cuts_max (reading R3). */
int or_select(const or_params* P, const float* x, const float* y, const float* z, const uint32_t start[5],
              or_candidate* cand, int cap, or_frame_result* res) {
    const double* R = P->layer_r;
    int stored = 0, found = 0;
    double band = P->rel_band;
    for (uint32_t a = start[0]; a < start[1]; ++a)
        for (uint32_t b = start[1]; b < start[2]; ++b)
            for (uint32_t c = start[2]; c < start[3]; ++c) {
                if (found > P->cuts_max) goto done;
                res->funnel[0]++;
                double h0[3] = {x[a], y[a], z[a]}, h1[3] = {x[b], y[b], z[b]}, h2[3] = {x[c], y[c], z[c]};
                int marg = 0;
                /* Eq. 3: Delta lambda = tan lambda_12 - tan lambda_01 */
                double dl = or_tan_lambda(h1[2], h2[2], R[1], R[2]) - or_tan_lambda(h0[2], h1[2], R[0], R[1]);
                marg |= near(fabs(dl), P->dlambda_max, band);
                if (!(fabs(dl) <= P->dlambda_max)) goto next;
                res->funnel[1]++;
                /* Eq. 4, Phi_01 */
                double c01 = or_cos_phi(h0[0], h0[1], h1[0], h1[1], R[0], R[1]);
                marg |= near(c01, P->cos_phi01_min, band);
                if (!(c01 >= P->cos_phi01_min)) goto next;
                res->funnel[2]++;
                /* Eq. 4, Phi_12 */
                double c12 = or_cos_phi(h1[0], h1[1], h2[0], h2[1], R[1], R[2]);
                marg |= near(c12, P->cos_phi12_min, band);
                if (!(c12 >= P->cos_phi12_min)) goto next;
                res->funnel[3]++;
                /* Eq. 5 */
                double rt = or_circle_radius(h0, h1, h2);
                marg |= near(fabs(rt), P->rt_min, band) | near(fabs(rt), P->rt_max, band);
                if (!(fabs(rt) >= P->rt_min && fabs(rt) <= P->rt_max)) goto next;
                res->funnel[4]++;
                if (stored < P->cuts_max && stored < cap) {
                    cand[stored].i0 = (int)(a - start[0]);
                    cand[stored].i1 = (int)(b - start[1]);
                    cand[stored].i2 = (int)(c - start[2]);
                    cand[stored].marginal = marg;
                    cand[stored].rtc = rt;
                    ++stored;
                }
                ++found;
            next:
                if (marg) res->n_cand_marginal++;
            }
done:
    res->n_cand = found;  /* loop stops once found == cuts_max + 1 */
    return stored;
}

/* ------------------------------------------------------------------------ */
/* Track Reconstruction, Sec. IV-B-2 + Alg. 3 for one candidate:
 * fit (h0,h1,h2); predict the layer-3 point; take the closest layer-3 hit (3D
 * Euclidean, lowest index on ties, reading R10); fit (h1,h2,h3); kappa-bar by
 * Eq. 8; chi2_global = sum_t chi2_t(kappa-bar) (Eq. 7); keep iff chi2_global < 32. */
int or_fit_candidate(const or_params* P, const float* x, const float* y, const float* z,
                     const uint32_t start[5], const or_candidate* c, or_track* o) {
    memset(o, 0, sizeof *o);
    double band = P->rel_band;
    uint32_t g0 = start[0] + c->i0, g1 = start[1] + c->i1, g2 = start[2] + c->i2;
    double h0[3] = {x[g0], y[g0], z[g0]}, h1[3] = {x[g1], y[g1], z[g1]}, h2[3] = {x[g2], y[g2], z[g2]};
    o->hit[0] = c->i0; o->hit[1] = c->i1; o->hit[2] = c->i2; o->hit[3] = -1;
    if (or_fit_triplet(P, h0, h1, h2, &o->t1) != 0) { o->status = OR_FIT_DEGENERATE1; return 0; }
    if (or_extrapolate(P, h1, h2, o->t1.q, o->t1.k_hat, o->pred) != 0) { o->status = OR_FIT_NO_REACH; return 0; }
    if (start[4] == start[3]) { o->status = OR_FIT_LAYER3_EMPTY; return 0; }
    double best = INFINITY, second = INFINITY;
    int bi = -1;
    for (uint32_t g = start[3]; g < start[4]; ++g) {
        double dx = x[g] - o->pred[0], dy = y[g] - o->pred[1], dz = z[g] - o->pred[2];
        double d2 = dx * dx + dy * dy + dz * dz;
        if (d2 < best) { second = best; best = d2; bi = (int)(g - start[3]); }
        else if (d2 < second) second = d2;
    }
    if (isfinite(second) && second - best <= band * best) o->marginal = 1;
    o->hit[3] = bi;
    uint32_t g3 = start[3] + bi;
    double h3[3] = {x[g3], y[g3], z[g3]};
    if (or_fit_triplet(P, h1, h2, h3, &o->t2) != 0) { o->status = OR_FIT_DEGENERATE2; return 0; }
    /* Eq. 8 */
    double w1 = 1.0 / o->t1.var_kappa, w2 = 1.0 / o->t2.var_kappa;
    o->kappa = (o->t1.kappa * w1 + o->t2.kappa * w2) / (w1 + w2);
    o->var_kappa = 1.0 / (w1 + w2);
    /* Eq. 7 */
    o->chi2 = triplet_chi2_at(&o->t1, o->kappa) + triplet_chi2_at(&o->t2, o->kappa);
    if (near(o->chi2, P->chi2_max, band)) o->marginal = 1;
    if (!(o->chi2 < P->chi2_max)) { o->status = OR_FIT_CHI2; return 0; }
    if (or_track_params(P, h0, h1, o->kappa, o) != 0) { o->status = OR_FIT_DOMAIN; return 0; }
    o->status = OR_FIT_OK;
    o->accepted = 1;
    return 0;
}

/* Track parameters of an accepted track (Sec. IV-B last paragraph "the track
 * parameters are calculated", Sec. IV-C circles), reading R11, at signed global
 * curvature kappa: charge q = sign(kappa), polar angle of arc h0 -> h1 from the
 * exact arc relation at |kappa|, transverse circle of radius sin(theta01)/|kappa|
 * through h0 and h1, p = PT_CONV B / |kappa|, E = sqrt(p^2 + m_e^2).
 * Sets o->q, cos_theta01, cx, cy, rt, p, energy; -1 if no short arc of that
 * curvature joins h0 and h1. */
int or_track_params(const or_params* P, const double h0[3], const double h1[3], double kappa, or_track* o) {
    double k = fabs(kappa);
    o->q = kappa > 0 ? +1 : -1;
    double d01 = hypot(h1[0] - h0[0], h1[1] - h0[1]), z01 = h1[2] - h0[2];
    double phi01 = or_arc_phi(d01, z01, k);
    if (isnan(phi01)) return -1;
    double cth = z01 * k / phi01;
    if (cth > 1) cth = 1;
    if (cth < -1) cth = -1;
    o->cos_theta01 = cth;
    double rt = sqrt(1.0 - cth * cth) / k;
    double off = sqrt(fmax(0.0, rt * rt - 0.25 * d01 * d01));
    double ux = (h1[0] - h0[0]) / d01, uy = (h1[1] - h0[1]) / d01;
    /* clockwise (q = +1): centre to the right of the chord direction */
    o->cx = 0.5 * (h0[0] + h1[0]) + o->q * off * uy;
    o->cy = 0.5 * (h0[1] + h1[1]) - o->q * off * ux;
    o->rt = rt;
    o->p = PT_CONV * P->b_field / k;
    o->energy = sqrt(o->p * o->p + M_E * M_E);
    return 0;
}

/* ------------------------------------------------------------------------ */
/* Circle-circle intersections (Sec. IV-C "all circle-circle intersections between
 * all tracks are determined").  Returns 0 (no intersection, or concentric) or 2
 * points (tangency gives two coincident points). out = {x0, y0, x1, y1}:
 * p_{0/1} = c1 + a u +/- h n, u = (c2 - c1)/D, n = (-u_y, u_x). */
int or_circle_intersections(double c1x, double c1y, double r1, double c2x, double c2y, double r2,
                            double out[4], double band, int* marginal) {
    double dx = c2x - c1x, dy = c2y - c1y, D = hypot(dx, dy);
    if (marginal) {
        if (near(D, r1 + r2, band) || near(D, fabs(r1 - r2), band)) *marginal = 1;
    }
    if (D == 0.0 || D > r1 + r2 || D < fabs(r1 - r2)) return 0;
    double a = (r1 * r1 - r2 * r2 + D * D) / (2.0 * D);
    double h = sqrt(fmax(0.0, r1 * r1 - a * a));
    double ux = dx / D, uy = dy / D;
    out[0] = c1x + a * ux - h * uy; out[1] = c1y + a * uy + h * ux;
    out[2] = c1x + a * ux + h * uy; out[3] = c1y + a * uy - h * ux;
    return 2;
}

/* distance from (x, y, z) to the double hollow cone target surface
 * rho(z) = R (1 - |z|/L), |z| <= L (Sec. III-B, Fig. 3; reading R14):
 * distance in the (rho, z) half plane to the two generatrix segments. */
static double seg_dist(double px, double py, double ax, double ay, double bx, double by) {
    double vx = bx - ax, vy = by - ay;
    double t = ((px - ax) * vx + (py - ay) * vy) / (vx * vx + vy * vy);
    if (t < 0) t = 0;
    if (t > 1) t = 1;
    return hypot(px - ax - t * vx, py - ay - t * vy);
}
double or_target_distance(const or_params* P, double x, double y, double z) {
    double rho = hypot(x, y), R = P->target_r, L = P->target_half;
    double d1 = seg_dist(rho, z, 0.0, -L, R, 0.0), d2 = seg_dist(rho, z, R, 0.0, 0.0, L);
    return d1 < d2 ? d1 : d2;
}

typedef struct vt {
    int q;
    double k, cth, sth, cx, cy, rt, h0[3], p, energy, sms;
} vt;

/* path along the track circle from its layer-0 hit to point (px,py): signed turning
 * angle from the point to h0 in the direction of motion, wrapped to (-pi, pi]
 * (reading R12). */
static double turn_to_h0(const vt* t, double px, double py) {
    double fp = atan2(py - t->cy, px - t->cx), f0 = atan2(t->h0[1] - t->cy, t->h0[0] - t->cx);
    return wrap_pi(t->q * (fp - f0));
}

/*
 * Vertex Fit, Sec. IV-C + Alg. 4, for one frame's accepted tracks.
 * Phase 1: every (e+_a, e+_b, e-) with a < b in track order (Alg. 4 first loop)
 *   passing |E_a + E_b + E_e - m_mu| <= e_window is stored; more than max_combs
 *   stored -> frame kept (reason 3).
 * Phase 2, per stored triple (Alg. 4 second loop, Sec. IV-C-1/2):
 *   circle intersections of pairs (a,b), (a,e), (b,e); a pair without intersection
 *   skips the triple; intersections with |p| > target_r + xy_margin are dismissed;
 *   for each choice of one intersection per pair: sigma_i^2 (Eq. 10, R13),
 *   mu_t (Eq. 9), points of closest approach (Fig. 6), z by Eq. 11, mu_z weighted
 *   mean, chi2 (Eq. 12, squared-distance reading R15); the triple's vertex is its
 *   minimum-chi2 choice.  The triple passes iff chi2 <= chi2_vertex_max, target
 *   distance <= target_dist_max and |sum p| <= p_total_max (Alg. 4, R16).
 * Frame kept iff some triple passes; the reported vertex is the passing triple
 * of lowest chi2 (first in order on ties).
 */
int or_vertex_frame(const or_params* P, const or_vtrack* tracks, int n, or_frame_result* res,
                    or_vertex* all_out, int all_cap) {
    double band = P->rel_band;
    vt* T = (vt*)calloc(n > 0 ? n : 1, sizeof(vt));
    int* pos = (int*)calloc(n > 0 ? n : 1, sizeof(int));
    int* neg = (int*)calloc(n > 0 ? n : 1, sizeof(int));
    int npos = 0, nneg = 0;
    for (int i = 0; i < n; ++i) {
        vt* t = &T[i];
        t->q = tracks[i].kappa > 0 ? +1 : -1;
        t->k = fabs(tracks[i].kappa);
        t->cth = tracks[i].cos_theta01;
        t->sth = sqrt(fmax(0.0, 1.0 - t->cth * t->cth));
        t->cx = tracks[i].cx; t->cy = tracks[i].cy;
        t->rt = t->sth / t->k;
        for (int j = 0; j < 3; ++j) t->h0[j] = tracks[i].h0[j];
        t->p = PT_CONV * P->b_field / t->k;
        t->energy = sqrt(t->p * t->p + M_E * M_E);
        t->sms = or_highland(t->p, P->x_over_x0);
        if (t->q > 0) pos[npos++] = i; else neg[nneg++] = i;
    }
    res->n_pos = npos;
    res->n_neg = nneg;
    /* phase 1 */
    int cap = P->max_combs + 1;
    int (*comb)[3] = (int(*)[3])calloc(cap, sizeof *comb);
    int ncomb = 0;
    for (int ia = 0; ia < npos && ncomb <= P->max_combs; ++ia)
        for (int ib = ia + 1; ib < npos && ncomb <= P->max_combs; ++ib)
            for (int ie = 0; ie < nneg && ncomb <= P->max_combs; ++ie) {
                int a = pos[ia], b = pos[ib], e = neg[ie];
                double dE = T[a].energy + T[b].energy + T[e].energy - M_MU;
                if (near(fabs(dE), P->e_window, band)) res->n_vertex_marginal++;
                if (fabs(dE) <= P->e_window) {
                    comb[ncomb][0] = a; comb[ncomb][1] = b; comb[ncomb][2] = e;
                    ++ncomb;
                }
            }
    res->n_combs = ncomb;
    int nout = 0;
    if (ncomb > P->max_combs) {
        res->reason = OR_REASON_COMB_OVERFLOW;
        res->keep = 1;
        goto out;
    }
    /* phase 2 */
    double rlim = P->target_r + P->xy_margin;
    for (int ci = 0; ci < ncomb; ++ci) {
        int idx[3] = {comb[ci][0], comb[ci][1], comb[ci][2]};
        static const int pr[3][2] = {{0, 1}, {0, 2}, {1, 2}};
        double pts[3][2][2];
        int npt[3];
        int skip = 0;
        for (int pi = 0; pi < 3 && !skip; ++pi) {
            const vt* A = &T[idx[pr[pi][0]]];
            const vt* B = &T[idx[pr[pi][1]]];
            double o4[4];
            int m = 0;
            int ni = or_circle_intersections(A->cx, A->cy, A->rt, B->cx, B->cy, B->rt, o4, band, &m);
            if (m) res->n_vertex_marginal++;
            if (ni == 0) { skip = 1; break; }
            npt[pi] = 0;
            for (int s = 0; s < 2; ++s) {
                double rr = hypot(o4[2 * s], o4[2 * s + 1]);
                if (near(rr, rlim, band)) res->n_vertex_marginal++;
                if (rr <= rlim) {
                    pts[pi][npt[pi]][0] = o4[2 * s];
                    pts[pi][npt[pi]][1] = o4[2 * s + 1];
                    npt[pi]++;
                }
            }
            if (npt[pi] == 0) skip = 1;
        }
        if (skip) continue;
        double bestchi = INFINITY, second = INFINITY;
        or_vertex bv;
        memset(&bv, 0, sizeof bv);
        for (int s0 = 0; s0 < npt[0]; ++s0)
            for (int s1 = 0; s1 < npt[1]; ++s1)
                for (int s2 = 0; s2 < npt[2]; ++s2) {
                    int sel[3] = {s0, s1, s2};
                    /* Eq. 10 for each intersection point (R13) */
                    double mx = 0, my = 0, wsum = 0;
                    for (int pi = 0; pi < 3; ++pi) {
                        const double* pp = pts[pi][sel[pi]];
                        const vt* A = &T[idx[pr[pi][0]]];
                        const vt* B = &T[idx[pr[pi][1]]];
                        double sa = A->rt * fabs(turn_to_h0(A, pp[0], pp[1]));
                        double sb = B->rt * fabs(turn_to_h0(B, pp[0], pp[1]));
                        double s2 = 0.5 * (A->sms * A->sms * sa * sa + B->sms * B->sms * sb * sb) +
                                    P->sigma_pixel * P->sigma_pixel;
                        mx += pp[0] / s2; my += pp[1] / s2; wsum += 1.0 / s2;
                    }
                    mx /= wsum; my /= wsum;              /* Eq. 9 */
                    /* points of closest approach (Fig. 6) and Eq. 11 */
                    double pca[3][3], sig2[3], mz = 0, wz = 0;
                    int bad = 0;
                    for (int t = 0; t < 3; ++t) {
                        const vt* A = &T[idx[t]];
                        double dx = mx - A->cx, dy = my - A->cy, dn = hypot(dx, dy);
                        if (dn == 0.0) { bad = 1; break; }
                        pca[t][0] = A->cx + A->rt * dx / dn;
                        pca[t][1] = A->cy + A->rt * dy / dn;
                        double dphi = turn_to_h0(A, pca[t][0], pca[t][1]);
                        pca[t][2] = A->h0[2] - dphi * A->cth / A->k;   /* Eq. 11 */
                        double s = A->rt * fabs(dphi);
                        sig2[t] = A->sms * A->sms * s * s + P->sigma_pixel * P->sigma_pixel;
                        mz += pca[t][2] / sig2[t]; wz += 1.0 / sig2[t];
                    }
                    if (bad) continue;
                    mz /= wz;
                    double chi = 0;                       /* Eq. 12 (R15) */
                    for (int t = 0; t < 3; ++t) {
                        double ex = pca[t][0] - mx, ey = pca[t][1] - my, ez = pca[t][2] - mz;
                        chi += (ex * ex + ey * ey + ez * ez) / sig2[t];
                    }
                    if (chi < bestchi) {
                        second = bestchi;
                        bestchi = chi;
                        bv.x = mx; bv.y = my; bv.z = mz; bv.chi2 = chi;
                        double ptot[3] = {0, 0, 0};
                        for (int t = 0; t < 3; ++t) {
                            const vt* A = &T[idx[t]];
                            double ph = atan2(pca[t][1] - A->cy, pca[t][0] - A->cx);
                            /* direction of motion on the circle: q (sin ph, -cos ph) */
                            ptot[0] += A->p * A->sth * A->q * sin(ph);
                            ptot[1] += A->p * A->sth * (-A->q * cos(ph));
                            ptot[2] += A->p * A->cth;
                        }
                        bv.p_total = sqrt(ptot[0] * ptot[0] + ptot[1] * ptot[1] + ptot[2] * ptot[2]);
                    } else if (chi < second) {
                        second = chi;
                    }
                }
        if (!isfinite(bestchi)) continue;
        if (isfinite(second) && second - bestchi <= band * bestchi) res->n_vertex_marginal++;
        bv.a = idx[0]; bv.b = idx[1]; bv.e = idx[2];
        bv.target_dist = or_target_distance(P, bv.x, bv.y, bv.z);
        if (near(bv.chi2, P->chi2_vertex_max, band)) res->n_vertex_marginal++;
        if (near(bv.target_dist, P->target_dist_max, band)) res->n_vertex_marginal++;
        if (near(bv.p_total, P->p_total_max, band)) res->n_vertex_marginal++;
        bv.pass = bv.chi2 <= P->chi2_vertex_max && bv.target_dist <= P->target_dist_max &&
                  bv.p_total <= P->p_total_max;
        if (all_out && nout < all_cap) all_out[nout] = bv;
        ++nout;
        if (bv.pass && (!res->has_vertex || bv.chi2 < res->vertex.chi2)) {
            res->has_vertex = 1;
            res->vertex = bv;
        }
    }
    if (res->has_vertex) {
        res->keep = 1;
        res->reason = OR_REASON_VERTEX;
    }
out:
    free(T); free(pos); free(neg); free(comb);
    return nout;
}

/* ------------------------------------------------------------------------ */
/* Alg. 1 for one frame: selection cuts -> track reconstruction -> vertex fit,
 * each overflow short-circuiting to "keep" (Sec. V-B). */
int or_process_frame(const or_params* P, const float* x, const float* y, const float* z,
                     const uint32_t start[5], or_frame_result* res, or_candidate* cand_buf,
                     or_track* track_buf) {
    memset(res, 0, sizeof *res);
    int ns = or_select(P, x, y, z, start, cand_buf, P->cuts_max, res);
    if (res->n_cand > P->cuts_max) {
        res->reason = OR_REASON_TRIPLET_OVERFLOW;
        res->keep = 1;
        return 0;
    }
    int nacc = 0;
    for (int i = 0; i < ns; ++i) {
        or_track tr;
        or_fit_candidate(P, x, y, z, start, &cand_buf[i], &tr);
        tr.cand = i;
        res->n_fit++;
        if (tr.marginal || cand_buf[i].marginal) res->n_fit_marginal++;
        if (tr.accepted) {
            if (nacc < P->max_tracks) track_buf[nacc] = tr;
            ++nacc;
        }
    }
    res->n_tracks = nacc > P->max_tracks ? P->max_tracks + 1 : nacc;  /* min(#accepted, max_tracks + 1) */
    if (nacc > P->max_tracks) {
        res->reason = OR_REASON_TRACK_OVERFLOW;
        res->keep = 1;
        return 0;
    }
    or_vtrack* vtr = (or_vtrack*)calloc(nacc > 0 ? nacc : 1, sizeof(or_vtrack));
    for (int i = 0; i < nacc; ++i) {
        vtr[i].kappa = track_buf[i].kappa;
        vtr[i].cos_theta01 = track_buf[i].cos_theta01;
        vtr[i].cx = track_buf[i].cx;
        vtr[i].cy = track_buf[i].cy;
        uint32_t g0 = start[0] + track_buf[i].hit[0];
        vtr[i].h0[0] = x[g0]; vtr[i].h0[1] = y[g0]; vtr[i].h0[2] = z[g0];
    }
    or_vertex_frame(P, vtr, nacc, res, NULL, 0);
    free(vtr);
    return 0;
}

int64_t or_process_frames(const or_params* P, const float* x, const float* y, const float* z,
                          const uint32_t* offsets, int64_t n_frames, or_frame_result* res) {
    or_candidate* cb = (or_candidate*)malloc(sizeof(or_candidate) * (P->cuts_max + 1));
    or_track* tb = (or_track*)malloc(sizeof(or_track) * (P->max_tracks + 1));
    int64_t kept = 0;
    for (int64_t f = 0; f < n_frames; ++f) {
        or_process_frame(P, x, y, z, offsets + 4 * f, &res[f], cb, tb);
        kept += res[f].keep;
    }
    free(cb);
    free(tb);
    return kept;
}

int or_sizeof(int which) {
    switch (which) {
        case 0: return (int)sizeof(or_params);
        case 1: return (int)sizeof(or_candidate);
        case 2: return (int)sizeof(or_triplet_fit);
        case 3: return (int)sizeof(or_track);
        case 4: return (int)sizeof(or_vtrack);
        case 5: return (int)sizeof(or_vertex);
        case 6: return (int)sizeof(or_frame_result);
    }
    return -1;
}
