// fit_numerics.cu -- host build of the CUDA path's fp32 fit math (m3e_device.cuh)
// for numerics studies against the oracle on the CPU.  Not part of the product.
#include "m3e_device.cuh"
using namespace m3e;
extern "C" int fit_numerics(const m3e_params* p, const float* x, const float* y, const float* z,
                            const uint32_t* start, int i0, int i1, int i2, float rtc, float* out) {
    DevParams d{};
    for (int l = 0; l < 4; ++l) d.R[l] = (float)p->layer_r[l];
    const double X = p->x_over_x0;
    d.chl = (float)(13.6 * sqrt(X) * (1.0 + 0.038 * log(X)) / (kPtConv * p->b_field));
    d.chi2_max = (float)p->chi2_max;
    d.R3sq = (float)(p->layer_r[3] * p->layer_r[3]);
    Frame F;
    F.x = x + start[0]; F.y = y + start[0]; F.z = z + start[0];
    for (int l = 0; l < 4; ++l) { F.s[l] = start[l] - start[0]; F.n[l] = start[l + 1] - start[l]; }
    FitOut o = fit_candidate(d, F, i0, i1, i2, rtc);
    out[0] = o.status; out[1] = o.hit3; out[2] = o.kappa1; out[3] = o.kappa2; out[4] = o.var1;
    out[5] = o.var2; out[6] = o.kappa; out[7] = o.chi2; out[8] = o.cth01; out[9] = o.cx; out[10] = o.cy;
    return 0;
}
