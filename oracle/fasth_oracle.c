/*
 * TEST INFRASTRUCTURE ONLY — the CPU oracle.  Never linked into, loaded by, or
 * called from the product library (paper_2009_13977_b200/).  Only tests/,
 * __graft_entry__.smoke() and bench.py's cpu_baseline leg use it, and only as
 * the checker.
 *
 * A plain-C, f64, single-threaded restatement of the reference FastH path
 * (/root/reference/proj/include/fasth/).  Each function cites the reference
 * lines it restates.  Parity of this restatement is PINNED two ways:
 *   - against golden vectors produced by the unmodified reference
 *     (tests/golden/*.npz, generator tests/golden/make_golden.py), and
 *   - live against oracle/_ref/libfasth_ref.so (the reference headers
 *     compiled by oracle/Makefile) when that library is present.
 *
 * Layouts (C order, f64):
 *   chain  : n x d   (row k = v_k, chain order: applying = H_1 (H_2 (... H_n X)))
 *   matrix : rows x cols row-major (as fasth::Matrix, matrix.hpp:66)
 * Return codes: 0 ok, 1 dimension, 2 degenerate vector, 3 singular, 4 error.
 */
#include <math.h>
#include <stdlib.h>
#include <string.h>

#define ORC_OK 0
#define ORC_DIM 1
#define ORC_DEGENERATE 2
#define ORC_SINGULAR 3
#define ORC_ERROR 4

/* householder.hpp:15 */
static const double kDegeneracy = 1e-30;

static double norm_sq(const double* v, size_t d) {
    double s = 0.0;
    for (size_t i = 0; i < d; ++i) s += v[i] * v[i];
    return s;
}

/* householder.hpp:109-126: X <- X - (2/||v||^2) v (v^T X), X d x m row-major. */
static void reflect_inplace(const double* v, double vv, size_t d, size_t m, double* X,
                            double* t /* m scratch */) {
    const double s = 2.0 / vv;
    memset(t, 0, m * sizeof(double));
    for (size_t i = 0; i < d; ++i)
        for (size_t l = 0; l < m; ++l) t[l] += v[i] * X[i * m + l];
    for (size_t i = 0; i < d; ++i) {
        const double c = s * v[i];
        for (size_t l = 0; l < m; ++l) X[i * m + l] -= c * t[l];
    }
}

static int check_chain(const double* V, size_t d, size_t n) {
    for (size_t k = 0; k < n; ++k) {
        const double s = norm_sq(V + k * d, d);
        if (!isfinite(s)) return ORC_ERROR;
        if (s <= kDegeneracy) return ORC_DEGENERATE;
    }
    return ORC_OK;
}

/* householder.hpp:130-137: H_1 ... H_n X, factor-at-a-time from H_n inward. */
int orc_chain_apply(size_t d, size_t n, size_t m, const double* V, const double* X, double* Y) {
    int rc = check_chain(V, d, n);
    if (rc) return rc;
    double* t = (double*)malloc((m ? m : 1) * sizeof(double));
    memcpy(Y, X, d * m * sizeof(double));
    for (size_t k = n; k-- > 0;) reflect_inplace(V + k * d, norm_sq(V + k * d, d), d, m, Y, t);
    free(t);
    return ORC_OK;
}

/* householder.hpp:148-179, Eq. (5): gradient of one reflection vector given
 * A_next (its input activation) and G (gradient at its output), summed over
 * the batch columns. */
int orc_householder_grad(size_t d, size_t m, const double* v, const double* A, const double* G,
                         double* grad) {
    const double vv = norm_sq(v, d);
    if (vv <= kDegeneracy) return ORC_DEGENERATE;
    const double s = 2.0 / vv;
    double* alpha = (double*)calloc(2 * (m ? m : 1), sizeof(double));
    double* beta = alpha + (m ? m : 1);
    for (size_t i = 0; i < d; ++i)
        for (size_t l = 0; l < m; ++l) {
            alpha[l] += v[i] * A[i * m + l];
            beta[l] += v[i] * G[i * m + l];
        }
    double ab = 0.0;
    for (size_t l = 0; l < m; ++l) ab += alpha[l] * beta[l];
    for (size_t i = 0; i < d; ++i) {
        double acc = 0.0;
        for (size_t l = 0; l < m; ++l) acc += alpha[l] * G[i * m + l] + beta[l] * A[i * m + l];
        grad[i] = -s * (acc - s * ab * v[i]);
    }
    free(alpha);
    return ORC_OK;
}

/* reference.hpp:17-47: sequential forward (chain_apply_sequential) then the
 * factor-at-a-time backward that reconstructs A_{j+1} = H_j A_j. */
int orc_sequential_fwd_bwd(size_t d, size_t n, size_t m, const double* V, const double* X,
                           const double* G, double* Y, double* dX, double* dV) {
    int rc = orc_chain_apply(d, n, m, V, X, Y);
    if (rc) return rc;
    double* a = (double*)malloc((d * m ? d * m : 1) * sizeof(double));
    double* t = (double*)malloc((m ? m : 1) * sizeof(double));
    memcpy(a, Y, d * m * sizeof(double));
    memcpy(dX, G, d * m * sizeof(double));
    for (size_t j = 0; j < n; ++j) {
        const double* v = V + j * d;
        const double vv = norm_sq(v, d);
        reflect_inplace(v, vv, d, m, a, t);
        orc_householder_grad(d, m, v, a, dX, dV + j * d);
        reflect_inplace(v, vv, d, m, dX, t);
    }
    free(a);
    free(t);
    return ORC_OK;
}

/* wy.hpp:56-100: W, Y (stored b x d, column j contiguous) with
 * I - 2 W Y^T = H_1 ... H_b, built by b sequential prepends from the last
 * factor: W' = [u_j | H_j W], Y' = [u_j | Y]. */
int orc_wy_compact(size_t d, size_t b, const double* V, double* W, double* Y) {
    if (b == 0) return ORC_ERROR;
    int rc = check_chain(V, d, b);
    if (rc) return rc;
    double* t = (double*)malloc(b * sizeof(double));
    for (size_t step = 0; step < b; ++step) {
        const size_t j = b - 1 - step;
        const double* v = V + j * d;
        const double vv = norm_sq(v, d);
        const double s = 2.0 / vv, inv = 1.0 / sqrt(vv);
        /* H_j applied to columns j+1..b-1 of W */
        for (size_t k = j + 1; k < b; ++k) {
            double acc = 0.0;
            for (size_t i = 0; i < d; ++i) acc += v[i] * W[k * d + i];
            t[k] = acc;
        }
        for (size_t k = j + 1; k < b; ++k)
            for (size_t i = 0; i < d; ++i) W[k * d + i] -= s * v[i] * t[k];
        for (size_t i = 0; i < d; ++i) W[j * d + i] = Y[j * d + i] = v[i] * inv;
    }
    free(t);
    return ORC_OK;
}

/* wy.hpp:104-133 (transpose=0: X - 2 W (Y^T X)) and wy.hpp:137-146
 * (transpose=1: X - 2 Y (W^T X)); W, Y stored b x d. In place on X (d x m). */
static void wy_apply_inplace(const double* W, const double* Y, size_t d, size_t b, size_t m,
                             int transpose, double* X, double* T /* b*m */) {
    const double* L = transpose ? W : Y; /* contracted with X */
    const double* R = transpose ? Y : W; /* expands the update */
    memset(T, 0, b * m * sizeof(double));
    for (size_t k = 0; k < b; ++k)
        for (size_t i = 0; i < d; ++i) {
            const double y = L[k * d + i];
            for (size_t l = 0; l < m; ++l) T[k * m + l] += y * X[i * m + l];
        }
    for (size_t i = 0; i < d; ++i)
        for (size_t k = 0; k < b; ++k) {
            const double c = 2.0 * R[k * d + i];
            for (size_t l = 0; l < m; ++l) X[i * m + l] -= c * T[k * m + l];
        }
}

/* fasth.hpp:40-61 (Algorithm 1) and fasth.hpp:69-109 (Algorithm 2).
 * b is clamped to [1, n] (fasth.hpp:52).  G, dX, dV may be NULL for a
 * forward-only call. */
int orc_fasth_fwd_bwd(size_t d, size_t n, size_t m, size_t b, const double* V, const double* X,
                      const double* G, double* Y, double* dX, double* dV) {
    int rc = check_chain(V, d, n);
    if (rc) return rc;
    if (n == 0) {
        memcpy(Y, X, d * m * sizeof(double));
        if (G) memcpy(dX, G, d * m * sizeof(double));
        return ORC_OK;
    }
    if (b < 1) b = 1;
    if (b > n) b = n;
    const size_t q = (n + b - 1) / b;
    double* W = (double*)malloc(n * d * sizeof(double));
    double* Yw = (double*)malloc(n * d * sizeof(double));
    for (size_t i = 0; i < q; ++i) { /* Step 1: compact_chain (wy.hpp:151-170) */
        const size_t lo = i * b, w = (lo + b <= n ? b : n - lo);
        orc_wy_compact(d, w, V + lo * d, W + lo * d, Yw + lo * d);
    }
    const size_t dm = d * m ? d * m : 1;
    double* act = (double*)malloc((q + 1) * dm * sizeof(double)); /* activations */
    double* T = (double*)malloc(b * (m ? m : 1) * sizeof(double));
    memcpy(act + q * dm, X, d * m * sizeof(double));
    for (size_t i = q; i-- > 0;) { /* Step 2: A_i = P_i A_{i+1} */
        const size_t lo = i * b, w = (lo + b <= n ? b : n - lo);
        memcpy(act + i * dm, act + (i + 1) * dm, d * m * sizeof(double));
        wy_apply_inplace(W + lo * d, Yw + lo * d, d, w, m, 0, act + i * dm, T);
    }
    memcpy(Y, act, d * m * sizeof(double));
    if (G) {
        /* Algorithm 2 step 1: dA[i+1] = P_i^T dA[i] (sequential). */
        double* dA = (double*)malloc((q + 1) * dm * sizeof(double));
        memcpy(dA, G, d * m * sizeof(double));
        for (size_t i = 0; i < q; ++i) {
            const size_t lo = i * b, w = (lo + b <= n ? b : n - lo);
            memcpy(dA + (i + 1) * dm, dA + i * dm, d * m * sizeof(double));
            wy_apply_inplace(W + lo * d, Yw + lo * d, d, w, m, 1, dA + (i + 1) * dm, T);
        }
        memcpy(dX, dA + q * dm, d * m * sizeof(double));
        /* Step 2 (fasth.hpp:97-108): per block, reconstruct within the block
         * and apply Eq. (5) per reflection. */
        double* a = (double*)malloc(dm * sizeof(double));
        double* g = (double*)malloc(dm * sizeof(double));
        double* t = (double*)malloc((m ? m : 1) * sizeof(double));
        for (size_t i = 0; i < q; ++i) {
            const size_t lo = i * b, w = (lo + b <= n ? b : n - lo);
            memcpy(a, act + i * dm, d * m * sizeof(double));
            memcpy(g, dA + i * dm, d * m * sizeof(double));
            for (size_t j = 0; j < w; ++j) {
                const double* v = V + (lo + j) * d;
                const double vv = norm_sq(v, d);
                reflect_inplace(v, vv, d, m, a, t);
                orc_householder_grad(d, m, v, a, g, dV + (lo + j) * d);
                reflect_inplace(v, vv, d, m, g, t);
            }
        }
        free(a);
        free(g);
        free(t);
        free(dA);
    }
    free(W);
    free(Yw);
    free(act);
    free(T);
    return ORC_OK;
}

static void reverse_chain(const double* V, size_t d, size_t n, double* R) {
    for (size_t k = 0; k < n; ++k) memcpy(R + k * d, V + (n - 1 - k) * d, d * sizeof(double));
}

/* svd_layer.hpp:106-117 (forward) and :122-154 (backward).  U chain has
 * length nu in dimension out, V chain nv in dimension in; sigma has
 * min(out, in) entries.  G == NULL -> forward only. */
int orc_svd_fwd_bwd(size_t out, size_t in, size_t nu, size_t nv, size_t m, size_t b,
                    const double* U, const double* V, const double* sigma, const double* X,
                    const double* G, double* Y, double* dX, double* dU, double* dV,
                    double* dsigma) {
    const size_t k = out < in ? out : in;
    for (size_t i = 0; i < k; ++i)
        if (!isfinite(sigma[i])) return ORC_ERROR;
    double* Vr = (double*)malloc((nv * in ? nv * in : 1) * sizeof(double));
    reverse_chain(V, in, nv, Vr);
    double* T1 = (double*)malloc((in * m ? in * m : 1) * sizeof(double));
    double* T2 = (double*)calloc(out * m ? out * m : 1, sizeof(double));
    double* dT2 = (double*)malloc((out * m ? out * m : 1) * sizeof(double));
    double* dT1 = (double*)calloc(in * m ? in * m : 1, sizeof(double));
    double* dVr = (double*)malloc((nv * in ? nv * in : 1) * sizeof(double));
    int rc = orc_fasth_fwd_bwd(in, nv, m, b, Vr, X, NULL, T1, NULL, NULL);
    if (!rc) {
        for (size_t i = 0; i < k; ++i) /* apply_sigma, svd_layer.hpp:92-101 */
            for (size_t l = 0; l < m; ++l) T2[i * m + l] = sigma[i] * T1[i * m + l];
        rc = orc_fasth_fwd_bwd(out, nu, m, b, U, T2, G, Y, dT2, dU);
    }
    if (!rc && G) {
        for (size_t i = 0; i < k; ++i) { /* svd_layer.hpp:131-145 */
            double acc = 0.0;
            for (size_t l = 0; l < m; ++l) acc += dT2[i * m + l] * T1[i * m + l];
            dsigma[i] = acc;
            for (size_t l = 0; l < m; ++l) dT1[i * m + l] = sigma[i] * dT2[i * m + l];
        }
        double* Yv = (double*)malloc((in * m ? in * m : 1) * sizeof(double));
        rc = orc_fasth_fwd_bwd(in, nv, m, b, Vr, X, dT1, Yv, dX, dVr);
        free(Yv);
        reverse_chain(dVr, in, nv, dV); /* undo the reversal, :150-151 */
    }
    free(Vr);
    free(T1);
    free(T2);
    free(dT2);
    free(dT1);
    free(dVr);
    return rc;
}

/* svd_layer.hpp:158-192 (svd_step) then :196-202 (clamp_sigma) when
 * clamp_eps >= 0.  On a degenerate update returns ORC_DEGENERATE and sets
 * *bad_chain (0 = U, 1 = V) and *bad_index like the reference message. */
int orc_svd_step(size_t out, size_t in, size_t nu, size_t nv, const double* U, const double* V,
                 const double* sigma, const double* dU, const double* dV, const double* dsigma,
                 double eta, double clamp_eps, double* U_out, double* V_out, double* sigma_out,
                 int* bad_chain, long* bad_index) {
    if (!isfinite(eta)) return ORC_ERROR;
    const size_t k = out < in ? out : in;
    for (int c = 0; c < 2; ++c) {
        const size_t dim = c ? in : out, n = c ? nv : nu;
        const double* P = c ? V : U;
        const double* D = c ? dV : dU;
        double* O = c ? V_out : U_out;
        for (size_t j = 0; j < n; ++j) {
            double s = 0.0;
            for (size_t i = 0; i < dim; ++i) {
                const double x = P[j * dim + i] - eta * D[j * dim + i];
                O[j * dim + i] = x;
                s += x * x;
            }
            if (!isfinite(s)) return ORC_ERROR;
            if (s <= kDegeneracy) {
                if (bad_chain) *bad_chain = c;
                if (bad_index) *bad_index = (long)j;
                return ORC_DEGENERATE;
            }
        }
    }
    if (clamp_eps >= 0.0 && clamp_eps >= 1.0) return ORC_ERROR;
    for (size_t i = 0; i < k; ++i) {
        double s = sigma[i] - eta * dsigma[i];
        if (clamp_eps >= 0.0) {
            if (s < 1.0 - clamp_eps) s = 1.0 - clamp_eps;
            if (s > 1.0 + clamp_eps) s = 1.0 + clamp_eps;
        }
        sigma_out[i] = s;
    }
    return ORC_OK;
}

/* matops.hpp:69-85 (kind 0: V Sigma^{-1} U^T X), :98-103 (kind 1:
 * U e^Sigma U^T X) and :107-117 (kind 2: U (1-s)/(1+s) U^T X).  Kinds 1, 2
 * need the symmetric form (nv == 0). */
int orc_matop(int kind, size_t d, size_t nu, size_t nv, size_t m, size_t b, const double* U,
              const double* V, const double* sigma, const double* X, double* Y) {
    if (kind != 0 && nv != 0) return ORC_ERROR;
    for (size_t i = 0; i < d; ++i) {
        if (kind == 0 && sigma[i] == 0.0) return ORC_SINGULAR;
        if (kind == 2 && sigma[i] == -1.0) return ORC_ERROR;
    }
    double* Ur = (double*)malloc((nu * d ? nu * d : 1) * sizeof(double));
    double* t = (double*)malloc((d * m ? d * m : 1) * sizeof(double));
    reverse_chain(U, d, nu, Ur);
    int rc = orc_fasth_fwd_bwd(d, nu, m, b, Ur, X, NULL, t, NULL, NULL);
    if (!rc) {
        for (size_t i = 0; i < d; ++i) {
            const double s = sigma[i];
            const double f = kind == 0 ? 1.0 / s : kind == 1 ? exp(s) : (1.0 - s) / (1.0 + s);
            for (size_t l = 0; l < m; ++l) t[i * m + l] *= f;
        }
        rc = kind == 0 ? orc_fasth_fwd_bwd(d, nv, m, b, V, t, NULL, Y, NULL, NULL)
                       : orc_fasth_fwd_bwd(d, nu, m, b, U, t, NULL, Y, NULL, NULL);
    }
    free(Ur);
    free(t);
    return rc;
}

/* matops.hpp:57-66 */
int orc_log_abs_det(size_t d, const double* sigma, double* out) {
    double acc = 0.0;
    for (size_t i = 0; i < d; ++i) {
        if (sigma[i] == 0.0) return ORC_SINGULAR;
        acc += log(fabs(sigma[i]));
    }
    *out = acc;
    return ORC_OK;
}
