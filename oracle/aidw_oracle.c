/*
 * aidw_oracle.c -- plain, slow, obviously-correct CPU oracle for the AIDW hot path
 * (arXiv 1511.02186, "GPU-accelerated Adaptive IDW").
 *
 * TEST INFRASTRUCTURE ONLY.  Only tests/, __graft_entry__.smoke() and bench.py's
 * cpu_baseline / --impl reference legs may load this library.  It shares no code,
 * header, table or constant with the CUDA path (paper_1511_02186_b200/csrc/).
 *
 * Precision: fp64 throughout ("CPU ... in double"), except the
 * oracle_knn_f32 instantiation, which reproduces the fp32 kNN decision in the
 * precision the paper's single-precision kernels take it in (REAL = float,
 * PAPER.md:402-405) so the fp32 GPU kNN can be checked bit for bit.
 * Compile with -ffp-contract=off (no silent FMA contraction); fmaf() is explicit
 * where the documented canonical sequence (reading R16) uses a fused op.
 *
 * Every function cites the passage it follows.  Functions are OpenMP-parallel over
 * queries only; each query is computed sequentially, so results do not depend on
 * the thread count.
 */
#include <math.h>
#include <stddef.h>
#include <stdint.h>

#ifdef _OPENMP
#include <omp.h>
#endif

/* ------------------------------------------------------------------------- */
/* §3.1.2 Step 3: insert one distance into the ascending    */
/* buffer of the k nearest so far.  "if dist < the kth distance, then replace  */
/* the kth distance with the dist", then "iteratively compare and swap the      */
/* neighboring two distances from the kth distance to the 1st distance".       */
/* ------------------------------------------------------------------------- */
void oracle_knn_insert(double *buf, int k, double dist)
{
    if (!(dist < buf[k - 1]))
        return;
    buf[k - 1] = dist;
    for (int i = k - 1; i > 0; --i) {
        if (buf[i] < buf[i - 1]) {
            double t = buf[i];
            buf[i] = buf[i - 1];
            buf[i - 1] = t;
        }
    }
}

static void knn_insert_f(float *buf, int k, float dist)
{
    if (!(dist < buf[k - 1]))
        return;
    buf[k - 1] = dist;
    for (int i = k - 1; i > 0; --i) {
        if (buf[i] < buf[i - 1]) {
            float t = buf[i];
            buf[i] = buf[i - 1];
            buf[i - 1] = t;
        }
    }
}

/* §3.1.2 Steps 1-2: the first k distances, sorted ascending. */
static void sort_ascending(double *a, int k)
{
    for (int i = 1; i < k; ++i) /* insertion sort */
        for (int j = i; j > 0 && a[j] < a[j - 1]; --j) {
            double t = a[j];
            a[j] = a[j - 1];
            a[j - 1] = t;
        }
}

static void sort_ascending_f(float *a, int k)
{
    for (int i = 1; i < k; ++i)
        for (int j = i; j > 0 && a[j] < a[j - 1]; --j) {
            float t = a[j];
            a[j] = a[j - 1];
            a[j - 1] = t;
        }
}

/* Squared Euclidean distance in the plane, Eq. 1's d(x, x_i)^2,
 * in the canonical sequence of DESIGN.md reading R16 (the paper's
 * REAL arithmetic, fixes no operation order):
 *   dx = qx - px; dy = qy - py; s = fma(dx, dx, dy*dy)   (each op rounded to nearest). */
static double dist2d_sq(double qx, double qy, double px, double py)
{
    double dx = qx - px;
    double dy = qy - py;
    return fma(dx, dx, dy * dy);
}

/* Euclidean distance d = sqrt_RN(s) (R16). */
static double dist2d(double qx, double qy, double px, double py)
{
    return sqrt(dist2d_sq(qx, qy, px, py));
}

#define KMAX 64

/*
 * Per-query kNN and r_obs, fp64.
 *   §3.1.2 Steps 1-3 give the k nearest distances d_1..d_k,
 *   Eq. 3: r_obs = (1/k) * sum_i d_i, summed in ascending order.
 * dists_out (nullable): [nq*k] ascending distances per query.
 * d1sq_out (nullable): [nq] squared distance to the nearest data point, min_i s_i
 *   (R16's s; the weighting pass scales Eq. 1's weights by it, R20).
 * Returns 0, or -1 if k is out of range / nd < k.
 */
int oracle_knn_f64(const double *x, const double *y, int64_t nd,
                   const double *qx, const double *qy, int64_t nq, int k,
                   double *dists_out, double *robs_out, double *d1sq_out)
{
    if (k < 1 || k > KMAX || nd < k)
        return -1;
#pragma omp parallel for schedule(static)
    for (int64_t q = 0; q < nq; ++q) {
        double buf[KMAX];
        double m = INFINITY;
        for (int64_t i = 0; i < nd; ++i) {
            double s = dist2d_sq(qx[q], qy[q], x[i], y[i]);
            if (s < m)
                m = s;
            double d = sqrt(s);
            if (i < k) { /* Step 1: the first k distances */
                buf[i] = d;
                if (i == k - 1)
                    sort_ascending(buf, k); /* Step 2 */
            } else {
                oracle_knn_insert(buf, k, d); /* Step 3 */
            }
        }
        double sum = 0.0;
        for (int i = 0; i < k; ++i)
            sum += buf[i];
        robs_out[q] = sum / (double)k;
        if (d1sq_out)
            d1sq_out[q] = m;
        if (dists_out)
            for (int i = 0; i < k; ++i)
                dists_out[q * k + i] = buf[i];
    }
    return 0;
}

/*
 * fp32 instantiation of the same steps: the kNN decision in REAL = float
 * (PAPER.md:402-405), with the canonical distance sequence of DESIGN.md R16:
 *   dx = qx - px; dy = qy - py; s = fma(dx, dx, dy*dy); d = sqrt(s)  (all float, RN).
 * r_obs = (sum of the ascending float d_i, sequential, in float) / (float)k.
 * d1sq_out (nullable): [nq] min_i s_i in float (the nearest squared distance).
 */
int oracle_knn_f32(const float *x, const float *y, int64_t nd,
                   const float *qx, const float *qy, int64_t nq, int k,
                   float *dists_out, float *robs_out, float *d1sq_out)
{
    if (k < 1 || k > KMAX || nd < k)
        return -1;
#pragma omp parallel for schedule(static)
    for (int64_t q = 0; q < nq; ++q) {
        float buf[KMAX];
        float m = INFINITY;
        for (int64_t i = 0; i < nd; ++i) {
            float dx = qx[q] - x[i];
            float dy = qy[q] - y[i];
            float dy2 = dy * dy;
            float s = fmaf(dx, dx, dy2);
            if (s < m)
                m = s;
            float d = sqrtf(s);
            if (i < k) {
                buf[i] = d;
                if (i == k - 1)
                    sort_ascending_f(buf, k);
            } else {
                knn_insert_f(buf, k, d);
            }
        }
        float sum = 0.0f;
        for (int i = 0; i < k; ++i)
            sum += buf[i];
        robs_out[q] = sum / (float)k;
        if (d1sq_out)
            d1sq_out[q] = m;
        if (dists_out)
            for (int i = 0; i < k; ++i)
                dists_out[q * k + i] = buf[i];
    }
    return 0;
}

/* Study area A for Eq. 2: the data's axis-aligned bounding box (R5). */
double oracle_bbox_area(const double *x, const double *y, int64_t nd)
{
    double x0 = x[0], x1 = x[0], y0 = y[0], y1 = y[0];
    for (int64_t i = 1; i < nd; ++i) {
        if (x[i] < x0) x0 = x[i];
        if (x[i] > x1) x1 = x[i];
        if (y[i] < y0) y0 = y[i];
        if (y[i] > y1) y1 = y[i];
    }
    return (x1 - x0) * (y1 - y0);
}

/* Eq. 2: r_exp = 1 / (2 sqrt(n / A)), n = number of data points. */
double oracle_r_exp(int64_t nd, double area)
{
    return 1.0 / (2.0 * sqrt((double)nd / area));
}

/*
 * Eq. 5: fuzzy membership mu_R of R.
 * form 0 (NORMALIZED, R8): 0.5 - 0.5 cos(pi (R - Rmin) / (Rmax - Rmin))
 * form 1 (PRINTED, as typeset):      0.5 - 0.5 cos(pi / Rmax * (R - Rmin))
 * Overlapping closed intervals resolve by first match in printed order (R9):
 * R <= Rmin -> 0; else R <= Rmax -> cosine; else 1.
 */
double oracle_mu(double R, double rmin, double rmax, int form)
{
    const double pi = 3.14159265358979323846;
    if (R <= rmin)
        return 0.0;
    if (R <= rmax) {
        if (form == 0)
            return 0.5 - 0.5 * cos(pi * ((R - rmin) / (rmax - rmin)));
        return 0.5 - 0.5 * cos(pi / rmax * (R - rmin));
    }
    return 1.0;
}

/*
 * Eq. 6: triangular membership alpha(mu), first match in the
 * printed row order (R12).  lv = alpha_1..alpha_5.
 */
double oracle_alpha_of_mu(double mu, const double *lv)
{
    if (mu <= 0.1)
        return lv[0];
    if (mu <= 0.3)
        return lv[0] * (1.0 - 5.0 * (mu - 0.1)) + 5.0 * lv[1] * (mu - 0.1);
    if (mu <= 0.5)
        return 5.0 * lv[2] * (mu - 0.3) + lv[1] * (1.0 - 5.0 * (mu - 0.3));
    if (mu <= 0.7)
        return lv[2] * (1.0 - 5.0 * (mu - 0.5)) + 5.0 * lv[3] * (mu - 0.5);
    if (mu <= 0.9)
        return 5.0 * lv[4] * (mu - 0.7) + lv[3] * (1.0 - 5.0 * (mu - 0.7));
    return lv[4];
}

/*
 * Steps 1-3 of §2.2 after the kNN: Eq. 4 R = r_obs / r_exp,
 * Eq. 5 mu, Eq. 6 alpha.  rmin/rmax are bounds on R (FIXED values, or the global
 * min/max of R over all queries in GLOBAL mode -- computed by the caller).
 * R_out / mu_out nullable.
 */
void oracle_alpha(const double *robs, int64_t nq, double r_exp, const double *lv,
                  double rmin, double rmax, int form,
                  double *alpha_out, double *R_out, double *mu_out)
{
#pragma omp parallel for schedule(static)
    for (int64_t q = 0; q < nq; ++q) {
        double R = robs[q] / r_exp;
        double mu = oracle_mu(R, rmin, rmax, form);
        alpha_out[q] = oracle_alpha_of_mu(mu, lv);
        if (R_out) R_out[q] = R;
        if (mu_out) mu_out[q] = mu;
    }
}

/*
 * Eq. 1: Z(x) = sum_i w_i z_i / sum_j w_j, w_i = d(x, x_i)^-alpha,
 * over ALL data points, in ascending index order, with the
 * per-query alpha.  d = 0 (exact coincidence, R19): Z = arithmetic mean
 * of z over the coincident data points (the limit of Eq. 1).
 */
void oracle_idw(const double *x, const double *y, const double *z, int64_t nd,
                const double *qx, const double *qy, const double *alpha, int64_t nq,
                double *z_out)
{
#pragma omp parallel for schedule(static)
    for (int64_t q = 0; q < nq; ++q) {
        double num = 0.0, den = 0.0, zc = 0.0;
        int64_t nc = 0;
        for (int64_t i = 0; i < nd; ++i) {
            double d = dist2d(qx[q], qy[q], x[i], y[i]);
            if (d == 0.0) {
                zc += z[i];
                nc += 1;
                continue;
            }
            double w = pow(d, -alpha[q]);
            num += w * z[i];
            den += w;
        }
        z_out[q] = nc > 0 ? zc / (double)nc : num / den;
    }
}

int oracle_num_threads(void)
{
#ifdef _OPENMP
    return omp_get_max_threads();
#else
    return 1;
#endif
}

void oracle_set_num_threads(int n)
{
#ifdef _OPENMP
    if (n > 0)
        omp_set_num_threads(n);
#else
    (void)n;
#endif
}
