// K2 at the reference's compiled plug point: `_sweep` (pkg/src/macetomo/icd.py:67-139)
// with its exact argument list and float64 arithmetic, pixels in raster order
// [s_begin, s_end), one warp (lanes stride the column; warp-shuffle theta1).  The
// neighbour tables are honoured as given (icd.py:106-127), so any neighbourhood works.
// This is the binding a maintainer uses to run the reference package itself on a
// B200; the production path is k_icd_sv / k_icd_raster.
#pragma once
#include <cuda_runtime.h>
#include <stdint.h>

namespace mace {

__device__ __forceinline__ double qg_influence64(double d, double p, double q, double T, double sx)
{
    const double ad = fabs(d);
    if (ad == 0.0) return 0.0;
    const double um = pow(ad / (T * sx), q - p);
    const double val = (pow(ad, p - 1.0) / pow(sx, p)) * um * (q / p + um) / ((1.0 + um) * (1.0 + um));
    return d > 0.0 ? val : -val;
}

__device__ __forceinline__ double qg_coef64(double d, double p, double q, double T, double sx)
{
    double ad = fabs(d);
    const double fl = 1e-9 * T * sx;
    if (ad <= fl) {
        if (p == 2.0) return 1.0 / (sx * sx);
        ad = fl;
    }
    const double um = pow(ad / (T * sx), q - p);
    return (pow(ad, p - 2.0) / pow(sx, p)) * um * (q / p + um) / ((1.0 + um) * (1.0 + um));
}

struct Sweep64 {
    double *z, *e, *dsq;
    const double *v, *a_val, *lam, *curv, *nbr_w;
    const int64_t *col_ptr, *row_idx, *nbr_idx;
    double beta_eff, eps_reg, inv_sigma2, p, q, T, sx;
    int quad, clamp;
    int64_t s_begin, s_end;
};

__global__ void __launch_bounds__(32) k_sweep64(Sweep64 P)
{
    const int lane = threadIdx.x;
    double delta_sq = 0.0;
    for (int64_t s = P.s_begin; s < P.s_end; ++s) {
        const double zs = __ldcg(P.z + s);
        double t1 = 0.0;
        for (int64_t jj = P.col_ptr[s] + lane; jj < P.col_ptr[s + 1]; jj += 32) {
            const int64_t r = P.row_idx[jj];
            t1 += P.a_val[jj] * P.lam[r] * __ldcg(P.e + r);
        }
        double g = 0.0, c = 0.0;
        if (lane < 8 && P.beta_eff > 0.0) {
            const int64_t r = P.nbr_idx[s * 8 + lane];
            if (r >= 0) {
                const double w = P.nbr_w[s * 8 + lane];
                const double zr = __ldcg(P.z + r);
                if (P.quad) {
                    g = w * (zs - zr);
                    c = w;
                } else {
                    const double d = zs - zr;
                    g = w * qg_influence64(d, P.p, P.q, P.T, P.sx);
                    c = w * qg_coef64(d, P.p, P.q, P.T, P.sx);
                }
            }
        }
#pragma unroll
        for (int o = 16; o; o >>= 1) {
            t1 += __shfl_xor_sync(0xffffffffu, t1, o);
            g += __shfl_xor_sync(0xffffffffu, g, o);
            c += __shfl_xor_sync(0xffffffffu, c, o);
        }
        double gp = 0.0, cp = 0.0;
        if (P.beta_eff > 0.0) {
            if (P.quad) {
                gp = P.beta_eff * (g + 2.0 * P.eps_reg * zs);
                cp = P.beta_eff * (c + 2.0 * P.eps_reg);
            } else {
                gp = P.beta_eff * g;
                cp = P.beta_eff * c;
            }
        }
        const double num = t1 - gp - P.inv_sigma2 * (zs - P.v[s]);
        const double den = P.curv[s] + cp + P.inv_sigma2;
        if (den <= 0.0) continue;
        double alpha = num / den;
        if (P.clamp && zs + alpha < 0.0) alpha = -zs;
        if (lane == 0) __stcg(P.z + s, zs + alpha);
        // red.add: a column may repeat a row (scipy keeps duplicates); both must land
        for (int64_t jj = P.col_ptr[s] + lane; jj < P.col_ptr[s + 1]; jj += 32)
            atomicAdd(P.e + P.row_idx[jj], -alpha * P.a_val[jj]);
        delta_sq += alpha * alpha;
        __syncwarp();
    }
    if (lane == 0) *P.dsq = delta_sq;
}

}  // namespace mace
