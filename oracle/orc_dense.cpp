// ORACLE — TEST INFRASTRUCTURE ONLY (see orc_core.h header).
// Restates proj/src/dense_kernels.cpp.  Eigen's HouseholderQR is restated as
// the unblocked Householder sweep with Eigen's makeHouseholder convention
// (third-party algorithm, Eigen3 >= 3.3; reflector v = [1; x_tail/(c0-beta)],
// beta = -sign(c0)*||x|| (beta = -||x|| when c0 >= 0), tau = (beta-c0)/beta,
// tau = 0 and beta = c0 when ||x_tail||^2 <= DBL_MIN).  Sign rule shared with the
// GPU kernels (csrc/dev.h hh_beta_negative): when c0 is roundoff-sized
// (c0^2 <= 1e-20 ||x_tail||^2) its sign is not a property of the data — Eigen's
// blocked arithmetic decides it by roundoff — so beta = -||x|| is taken there too.
#include <algorithm>
#include <cassert>
#include <limits>

#include "orc_core.h"

namespace orc {

namespace {

// Eigen MatrixBase::makeHouseholder on x = A(k:m, k); returns tau, beta and
// writes the essential part into A(k+1:m, k).
void make_householder(Mat& A, Index k, double& tau, double& beta) {
    const Index m = A.r;
    double tail2 = 0.0;
    for (Index i = k + 1; i < m; ++i) tail2 += A(i, k) * A(i, k);
    const double c0 = A(k, k);
    if (tail2 <= std::numeric_limits<double>::min()) {
        tau = 0.0;
        beta = c0;
        for (Index i = k + 1; i < m; ++i) A(i, k) = 0.0;
        return;
    }
    beta = std::sqrt(c0 * c0 + tail2);
    if (c0 >= 0.0 || c0 * c0 <= 1e-20 * tail2) beta = -beta;
    const double den = c0 - beta;
    for (Index i = k + 1; i < m; ++i) A(i, k) /= den;
    tau = (beta - c0) / beta;
}

}  // namespace

// dense_kernels.cpp:11-35
void block_householder_qr(const Mat& B, ReflectorSet& H, Mat& R) {
    const Index m = B.r, n = B.c;
    assert(m >= n);
    Mat A = B;
    Vec hc(n, 0.0);
    for (Index k = 0; k < n; ++k) {
        double tau, beta;
        make_householder(A, k, tau, beta);
        A(k, k) = beta;
        hc[k] = tau;
        if (tau == 0.0) continue;
        // applyHouseholderOnTheLeft to A(k:m, k+1:n)
        for (Index j = k + 1; j < n; ++j) {
            double w = A(k, j);
            for (Index i = k + 1; i < m; ++i) w += A(i, k) * A(i, j);
            A(k, j) -= tau * w;
            const double tw = tau * w;
            for (Index i = k + 1; i < m; ++i) A(i, j) -= tw * A(i, k);
        }
    }
    H.T = Mat();
    H.V = Mat::zeros(m, n);
    H.tau = hc;
    H.sign.assign(n, 1.0);
    R = Mat::zeros(n, n);
    for (Index j = 0; j < n; ++j) {
        H.V(j, j) = 1.0;
        for (Index i = j + 1; i < m; ++i) H.V(i, j) = A(i, j);
        for (Index i = 0; i <= j; ++i) R(i, j) = A(i, j);
    }
    for (Index i = 0; i < n; ++i)
        if (R(i, i) < 0.0) {
            H.sign[i] = -1.0;
            for (Index j = 0; j < n; ++j) R(i, j) = -R(i, j);
        }
}

namespace {

// dense_kernels.cpp:41-53 — upper-triangular T with H_0..H_{k-1} = I - V T V^T.
Mat accumulate_wy(const ReflectorSet& H) {
    const Index k = H.count(), m = H.rows();
    Mat T = Mat::zeros(k, k);
    for (Index j = 0; j < k; ++j) {
        if (H.tau[j] == 0.0) continue;
        if (j > 0) {
            Vec w(j, 0.0);
            for (Index a = 0; a < j; ++a) {
                double s = 0.0;
                for (Index i = 0; i < m; ++i) s += H.V(i, a) * H.V(i, j);
                w[a] = s;
            }
            for (Index a = 0; a < j; ++a) {
                double s = 0.0;
                for (Index b = a; b < j; ++b) s += T(a, b) * w[b];
                T(a, j) = -H.tau[j] * s;
            }
        }
        T(j, j) = H.tau[j];
    }
    return T;
}

// dense_kernels.cpp:56-87
void apply_raw(const ReflectorSet& H, View X, bool transpose) {
    const Index m = H.rows(), k = H.count();
    assert(X.r == m);
    if (k == 0) return;
    if (k >= 4 && X.c >= 4) {
        if (H.T.size() == 0) H.T = accumulate_wy(H);
        Mat W(k, X.c);  // V^T X
        for (Index j = 0; j < X.c; ++j)
            for (Index a = 0; a < k; ++a) {
                double s = 0.0;
                for (Index i = 0; i < m; ++i) s += H.V(i, a) * X(i, j);
                W(a, j) = s;
            }
        Mat W2(k, X.c);
        for (Index j = 0; j < X.c; ++j)
            for (Index a = 0; a < k; ++a) {
                double s = 0.0;
                if (transpose)  // T^T (lower)
                    for (Index b = 0; b <= a; ++b) s += H.T(b, a) * W(b, j);
                else  // T (upper)
                    for (Index b = a; b < k; ++b) s += H.T(a, b) * W(b, j);
                W2(a, j) = s;
            }
        for (Index j = 0; j < X.c; ++j)
            for (Index i = 0; i < m; ++i) {
                double s = 0.0;
                for (Index a = 0; a < k; ++a) s += H.V(i, a) * W2(a, j);
                X(i, j) -= s;
            }
        return;
    }
    auto one = [&](Index j) {
        if (H.tau[j] == 0.0) return;
        for (Index c = 0; c < X.c; ++c) {
            double w = 0.0;
            for (Index i = j; i < m; ++i) w += X(i, c) * H.V(i, j);
            const double tw = H.tau[j] * w;
            for (Index i = j; i < m; ++i) X(i, c) -= tw * H.V(i, j);
        }
    };
    if (transpose)
        for (Index j = 0; j < k; ++j) one(j);
    else
        for (Index j = k - 1; j >= 0; --j) one(j);
}

void flip_rows(const ReflectorSet& H, View X) {  // :89-92
    for (Index i = 0; i < H.count(); ++i)
        if (H.sign[i] < 0.0)
            for (Index c = 0; c < X.c; ++c) X(i, c) = -X(i, c);
}

}  // namespace

void apply_left_t(const ReflectorSet& H, View X) {
    apply_raw(H, X, true);
    flip_rows(H, X);
}
void apply_left(const ReflectorSet& H, View X) {
    flip_rows(H, X);
    apply_raw(H, X, false);
}
void apply_right(const ReflectorSet& H, Mat& X) {
    Mat Xt = X.transpose();
    apply_left_t(H, view(Xt));
    X = Xt.transpose();
}
void apply_right_t(const ReflectorSet& H, Mat& X) {
    Mat Xt = X.transpose();
    apply_left(H, view(Xt));
    X = Xt.transpose();
}
Mat reflectors_to_dense(const ReflectorSet& H) {
    Mat Q = Mat::identity(H.rows());
    apply_left(H, view(Q));
    return Q;
}

namespace {
double col_tail_norm(const Mat& A, Index j, Index r0) {
    double s = 0.0;
    for (Index i = r0; i < A.r; ++i) s += A(i, j) * A(i, j);
    return std::sqrt(s);
}
}  // namespace

// dense_kernels.cpp:124-232 — greedy column-norm pivoting with the exact-norm
// stop rule (refresh all trailing norms and retry once before stopping) and
// LAPACK-style norm downdating (recompute when t*ratio^2 <= sqrt(eps_mach)).
TruncatedQR truncated_cpqr(const Mat& B, double eps) {
    const Index m = B.r, n = B.c, kmax = std::min(m, n);
    TruncatedQR out;
    if (kmax == 0) {
        out.H.V = Mat::zeros(m, 0);
        out.R = Mat::zeros(0, n);
        return out;
    }
    Mat A = B;
    std::vector<Index> colid(n);
    for (Index j = 0; j < n; ++j) colid[j] = j;
    Vec vn1(n), vn2(n);
    for (Index j = 0; j < n; ++j) vn1[j] = vn2[j] = col_tail_norm(A, j, 0);
    const double tol3z = std::sqrt(std::numeric_limits<double>::epsilon());
    Mat Vfull = Mat::zeros(m, kmax);
    Vec tau(kmax, 0.0), sgn(kmax, 1.0);

    Index k = 0;
    while (k < kmax) {
        Index piv = k;
        for (Index j = k + 1; j < n; ++j)
            if (vn1[j] > vn1[piv]) piv = j;
        double exact = col_tail_norm(A, piv, k);
        bool stop = (k == 0) ? !(exact > 0.0) : (eps > 0.0 && exact < eps * out.r11);
        if (stop && k > 0) {
            Index best = k;
            double bn = -1.0;
            for (Index j = k; j < n; ++j) {
                vn1[j] = vn2[j] = col_tail_norm(A, j, k);
                if (vn1[j] > bn) {
                    bn = vn1[j];
                    best = j;
                }
            }
            piv = best;
            exact = bn;
            stop = eps > 0.0 && exact < eps * out.r11;
        }
        if (stop) break;
        if (piv != k) {
            for (Index i = 0; i < m; ++i) std::swap(A(i, piv), A(i, k));
            std::swap(colid[piv], colid[k]);
            std::swap(vn1[piv], vn1[k]);
            std::swap(vn2[piv], vn2[k]);
        }
        // Householder on x = A(k:m, k): alpha = -sign+(x0)||x||, v = x - alpha e1.
        const Index len = m - k;
        Vec v(len);
        for (Index i = 0; i < len; ++i) v[i] = A(k + i, k);
        double alpha = 0.0;
        for (Index i = 0; i < len; ++i) alpha += v[i] * v[i];
        alpha = std::sqrt(alpha);
        if (v[0] > 0.0) alpha = -alpha;
        v[0] -= alpha;
        double vns = 0.0;
        for (Index i = 0; i < len; ++i) vns += v[i] * v[i];
        Vfull(k, k) = 1.0;
        if (vns > 0.0) {
            const double t = 2.0 / vns;
            for (Index j = k + 1; j < n; ++j) {
                double w = 0.0;
                for (Index i = 0; i < len; ++i) w += A(k + i, j) * v[i];
                const double tw = t * w;
                for (Index i = 0; i < len; ++i) A(k + i, j) -= tw * v[i];
            }
            for (Index i = 0; i < len; ++i) A(k + i, k) = 0.0;
            A(k, k) = alpha;
            for (Index i = 0; i < len; ++i) Vfull(k + i, k) = v[i] / v[0];
            tau[k] = t * v[0] * v[0];
        }
        if (A(k, k) < 0.0) {
            sgn[k] = -1.0;
            for (Index j = k; j < n; ++j) A(k, j) = -A(k, j);
        }
        if (k == 0) out.r11 = A(0, 0);
        out.perm.push_back(colid[k]);
        ++k;
        if (k < kmax) {
            for (Index j = k; j < n; ++j) {
                if (vn1[j] == 0.0) continue;
                double t = std::abs(A(k - 1, j)) / vn1[j];
                t = std::max(0.0, (1.0 - t) * (1.0 + t));
                const double ratio = vn1[j] / vn2[j];
                if (t * ratio * ratio <= tol3z)
                    vn1[j] = vn2[j] = col_tail_norm(A, j, k);
                else
                    vn1[j] *= std::sqrt(t);
            }
        }
    }
    out.rank = k;
    out.H.V = Vfull.block(0, 0, m, k);
    out.H.tau.assign(tau.begin(), tau.begin() + k);
    out.H.sign.assign(sgn.begin(), sgn.begin() + k);
    out.R = Mat::zeros(k, n);
    for (Index j = 0; j < n; ++j)
        for (Index i = 0; i < k; ++i) out.R(i, colid[j]) = A(i, j);
    return out;
}

// :234-240
void check_diag_invertible(const Mat& R) {
    for (Index i = 0; i < std::min(R.r, R.c); ++i) {
        const double d = std::abs(R(i, i));
        if (!(d >= std::numeric_limits<double>::min()))
            throw SingularFrontError(-1, "pivot " + std::to_string(i) + " is zero or denormal");
    }
}

// :242-257 — U X = B / U^T X = B (left), X U = B / X U^T = B (right).
void tri_solve_upper(const Mat& R, View B, Side side, bool transpose) {
    check_diag_invertible(R);
    const Index n = R.r;
    if (side == Side::Left) {
        for (Index c = 0; c < B.c; ++c) {
            if (!transpose) {
                for (Index i = n - 1; i >= 0; --i) {
                    double s = B(i, c);
                    for (Index j = i + 1; j < n; ++j) s -= R(i, j) * B(j, c);
                    B(i, c) = s / R(i, i);
                }
            } else {
                for (Index i = 0; i < n; ++i) {
                    double s = B(i, c);
                    for (Index j = 0; j < i; ++j) s -= R(j, i) * B(j, c);
                    B(i, c) = s / R(i, i);
                }
            }
        }
    } else {
        for (Index r = 0; r < B.r; ++r) {
            if (!transpose) {  // x U = b: x_j = (b_j - sum_{i<j} x_i U_ij) / U_jj
                for (Index j = 0; j < n; ++j) {
                    double s = B(r, j);
                    for (Index i = 0; i < j; ++i) s -= B(r, i) * R(i, j);
                    B(r, j) = s / R(j, j);
                }
            } else {  // x U^T = b: x_j = (b_j - sum_{i>j} x_i U_ji) / U_jj
                for (Index j = n - 1; j >= 0; --j) {
                    double s = B(r, j);
                    for (Index i = j + 1; i < n; ++i) s -= B(r, i) * R(j, i);
                    B(r, j) = s / R(j, j);
                }
            }
        }
    }
}

}  // namespace orc
