/*
 * TEST INFRASTRUCTURE ONLY — CPU oracle for the partial-update ICD pass.
 *
 * Plain-C float64 restatement of the reference's numba hot loop so that the
 * parity tests (and bench.py's cpu_baseline / --impl reference legs) have a
 * compiled CPU checker.  Nothing in the product package links or calls this.
 *
 *   orc_qg_influence  <- pkg/src/macetomo/icd.py:45-52   (_qg_influence)
 *   orc_qg_coef       <- pkg/src/macetomo/icd.py:55-64   (_qg_coef)
 *   orc_sweep         <- pkg/src/macetomo/icd.py:67-139  (_sweep, raster order)
 *   orc_csr_residual  <- pkg/src/macetomo/icd.py:210-211 (refresh_error: e = y - A z)
 *
 * Pinned against the reference itself through tests/golden/ (vectors written
 * by tests/golden/make_golden.py, which imports the reference package).
 */
#include <math.h>
#include <stdint.h>

static double orc_qg_influence(double d, double p, double q, double T, double sx)
{
    double ad = fabs(d);
    if (ad == 0.0) return 0.0;
    double u = ad / (T * sx);
    double um = pow(u, q - p);
    double val = (pow(ad, p - 1.0) / pow(sx, p)) * um * (q / p + um) / ((1.0 + um) * (1.0 + um));
    return d > 0.0 ? val : -val;
}

static double orc_qg_coef(double d, double p, double q, double T, double sx)
{
    double ad = fabs(d);
    double floor_ = 1e-9 * T * sx;
    if (ad <= floor_) {
        if (p == 2.0) return 1.0 / (sx * sx);
        ad = floor_;
    }
    double u = ad / (T * sx);
    double um = pow(u, q - p);
    return (pow(ad, p - 2.0) / pow(sx, p)) * um * (q / p + um) / ((1.0 + um) * (1.0 + um));
}

/* Exported twins so the tests can check the potential math point-wise. */
double orc_influence(double d, double p, double q, double T, double sx) { return orc_qg_influence(d, p, q, T, sx); }
double orc_coef(double d, double p, double q, double T, double sx) { return orc_qg_coef(d, p, q, T, sx); }

/*
 * Raster pass over pixels [s_begin, s_end).  Same argument list and meaning
 * as the reference _sweep; mutates z and e, returns sum(alpha^2).
 */
double orc_sweep(double *z, const double *v, double *e,
                 const int64_t *col_ptr, const int64_t *row_idx, const double *a_val,
                 const double *lam, const double *curv_data,
                 const int64_t *nbr_idx, const double *nbr_w,
                 double beta_eff, double eps_reg, double inv_sigma2, int quad_prior,
                 double p, double q, double T, double sx, int clamp,
                 int64_t s_begin, int64_t s_end)
{
    double delta_sq = 0.0;
    for (int64_t s = s_begin; s < s_end; ++s) {
        double zs = z[s];
        double t1 = 0.0;
        for (int64_t jj = col_ptr[s]; jj < col_ptr[s + 1]; ++jj) {
            int64_t r = row_idx[jj];
            t1 += a_val[jj] * lam[r] * e[r];
        }
        double gp = 0.0, cp = 0.0;
        if (beta_eff > 0.0) {
            double acc_g = 0.0, acc_c = 0.0;
            if (quad_prior) {
                for (int k = 0; k < 8; ++k) {
                    int64_t r = nbr_idx[s * 8 + k];
                    if (r >= 0) {
                        double w = nbr_w[s * 8 + k];
                        acc_g += w * (zs - z[r]);
                        acc_c += w;
                    }
                }
                gp = beta_eff * (acc_g + 2.0 * eps_reg * zs);
                cp = beta_eff * (acc_c + 2.0 * eps_reg);
            } else {
                for (int k = 0; k < 8; ++k) {
                    int64_t r = nbr_idx[s * 8 + k];
                    if (r >= 0) {
                        double w = nbr_w[s * 8 + k];
                        double d = zs - z[r];
                        acc_g += w * orc_qg_influence(d, p, q, T, sx);
                        acc_c += w * orc_qg_coef(d, p, q, T, sx);
                    }
                }
                gp = beta_eff * acc_g;
                cp = beta_eff * acc_c;
            }
        }
        double num = t1 - gp - inv_sigma2 * (zs - v[s]);
        double den = curv_data[s] + cp + inv_sigma2;
        if (den <= 0.0) continue;
        double alpha = num / den;
        if (clamp && zs + alpha < 0.0) alpha = -zs;
        z[s] = zs + alpha;
        for (int64_t jj = col_ptr[s]; jj < col_ptr[s + 1]; ++jj)
            e[row_idx[jj]] -= alpha * a_val[jj];
        delta_sq += alpha * alpha;
    }
    return delta_sq;
}

/* e[r] = y[r] - sum_j A[r, j] z[j] for a CSR operator (refresh_error). */
void orc_csr_residual(int64_t n_rows, const int64_t *row_ptr, const int64_t *cols,
                      const double *vals, const double *y, const double *z, double *e)
{
    for (int64_t r = 0; r < n_rows; ++r) {
        double acc = 0.0;
        for (int64_t j = row_ptr[r]; j < row_ptr[r + 1]; ++j) acc += vals[j] * z[cols[j]];
        e[r] = y[r] - acc;
    }
}
