// ORACLE — TEST INFRASTRUCTURE ONLY.
//
// A from-scratch restatement of the small subset of the Eigen 3 C++ API that the
// spaQR reference sources (/root/reference/proj/src/*.cpp) call, so that those
// sources compile UNMODIFIED here into oracle/_ref/libspaqr_ref.so (see
// oracle/Makefile.ref).  Eigen3 itself (third-party, >= 3.3, unpinned: the
// reference's CMakeLists.txt:15-20 falls back to /usr/include/eigen3) is absent from
// this image and there is no network, so its published algorithms are restated:
//
//  * dense storage: column-major double, dynamic size (Eigen::MatrixXd / VectorXd);
//    block expressions are strided views, every arithmetic expression is evaluated
//    eagerly into a temporary (aliasing-safe, like Eigen's default products);
//  * products: natural order — C(i,j) = sum_k A(i,k) B(k,j), k ascending;
//    squaredNorm/norm: sequential sum of squares (Eigen's redux order is
//    vectorised and not reproducible anyway);
//  * HouseholderQR: the unblocked Householder sweep with Eigen's
//    MatrixBase::makeHouseholder convention (v = [1; x_tail/(c0-beta)],
//    beta = -sign(c0)*||x|| with beta = -||x|| for c0 >= 0, tau = (beta-c0)/beta;
//    tau = 0, beta = c0 when ||x_tail||^2 <= DBL_MIN) and applyHouseholderOnTheLeft
//    for the trailing columns — the same restatement as oracle/orc_dense.cpp,
//    including its documented sign rule: a roundoff-sized c0 (c0^2 <= 1e-20
//    ||x_tail||^2), whose sign real Eigen leaves to roundoff, takes beta = -||x||;
//  * triangular solves: substitution in natural order;
//  * SparseMatrix<double>: compressed column storage (int indices), setFromTriplets
//    sums duplicates and sorts rows, prune(0,0) drops exact zeros, A*x accumulates
//    column by column (j ascending), A^T*y takes per-column dots (rows ascending).
//
// Nothing in the product package includes this file.
#pragma once

#include <algorithm>
#include <cassert>
#include <cmath>
#include <cstddef>
#include <cstring>
#include <limits>
#include <type_traits>
#include <vector>

namespace Eigen {

using Index = std::ptrdiff_t;
enum { Dynamic = -1 };
enum UpLoType { Lower = 1, Upper = 2 };
enum SideType { OnTheLeft = 1, OnTheRight = 2 };
enum NoChange_t { NoChange };

class Matrix;
class View;
template <int Mode>
struct TriView;

// ---------------------------------------------------------------- View ---
// A strided view: element (i, j) lives at p[i*rs + j*cs].  Copy construction is
// shallow; assignment copies ELEMENTS (as an Eigen block expression does).
class View {
public:
    double* p = nullptr;
    Index r = 0, c = 0, rs = 1, cs = 0;

    View() = default;
    View(double* p_, Index r_, Index c_, Index rs_, Index cs_) : p(p_), r(r_), c(c_), rs(rs_), cs(cs_) {}
    View(const View&) = default;

    Index rows() const { return r; }
    Index cols() const { return c; }
    Index size() const { return r * c; }
    double& operator()(Index i, Index j) const { return p[i * rs + j * cs]; }
    double& operator()(Index i) const { return c == 1 ? p[i * rs] : p[i * cs]; }
    double& operator[](Index i) const { return (*this)(i); }

    View block(Index i, Index j, Index nr, Index nc) const { return View(p + i * rs + j * cs, nr, nc, rs, cs); }
    View row(Index i) const { return block(i, 0, 1, c); }
    View col(Index j) const { return block(0, j, r, 1); }
    View topRows(Index n) const { return block(0, 0, n, c); }
    View bottomRows(Index n) const { return block(r - n, 0, n, c); }
    View middleRows(Index i, Index n) const { return block(i, 0, n, c); }
    View leftCols(Index n) const { return block(0, 0, r, n); }
    View rightCols(Index n) const { return block(0, c - n, r, n); }
    View middleCols(Index j, Index n) const { return block(0, j, r, n); }
    View topLeftCorner(Index nr, Index nc) const { return block(0, 0, nr, nc); }
    View bottomRightCorner(Index nr, Index nc) const { return block(r - nr, c - nc, nr, nc); }
    // vector segments: along the columns of a row vector, else along the rows
    View segment(Index i, Index n) const { return r == 1 && c != 1 ? block(0, i, 1, n) : block(i, 0, n, 1); }
    View head(Index n) const { return segment(0, n); }
    View tail(Index n) const { return segment(size() - n, n); }
    View transpose() const { return View(p, c, r, cs, rs); }
    View noalias() const { return *this; }

    template <int Mode>
    TriView<Mode> triangularView() const;

    double squaredNorm() const {
        double s = 0.0;
        for (Index j = 0; j < c; ++j)
            for (Index i = 0; i < r; ++i) s += (*this)(i, j) * (*this)(i, j);
        return s;
    }
    double norm() const { return std::sqrt(squaredNorm()); }
    double maxCoeff() const {
        double m = -std::numeric_limits<double>::infinity();
        for (Index j = 0; j < c; ++j)
            for (Index i = 0; i < r; ++i) m = std::max(m, (*this)(i, j));
        return m;
    }
    double sum() const {
        double s = 0.0;
        for (Index j = 0; j < c; ++j)
            for (Index i = 0; i < r; ++i) s += (*this)(i, j);
        return s;
    }
    // isZero(prec) / isIdentity(prec) with prec = 0: exact comparisons.
    bool isZero(double prec = 0.0) const {
        for (Index j = 0; j < c; ++j)
            for (Index i = 0; i < r; ++i)
                if (std::abs((*this)(i, j)) > prec) return false;
        return true;
    }
    bool isIdentity(double prec = 0.0) const {
        for (Index j = 0; j < c; ++j)
            for (Index i = 0; i < r; ++i)
                if (std::abs((*this)(i, j) - (i == j ? 1.0 : 0.0)) > prec) return false;
        return true;
    }
    Matrix cwiseAbs() const;
    Matrix cwiseProduct(const View& o) const;
    void setZero() const {
        for (Index j = 0; j < c; ++j)
            for (Index i = 0; i < r; ++i) (*this)(i, j) = 0.0;
    }
    void setIdentity() const {
        for (Index j = 0; j < c; ++j)
            for (Index i = 0; i < r; ++i) (*this)(i, j) = i == j ? 1.0 : 0.0;
    }
    void swap(View o) const {
        assert(o.r == r && o.c == c);
        for (Index j = 0; j < c; ++j)
            for (Index i = 0; i < r; ++i) std::swap((*this)(i, j), o(i, j));
    }

    bool overlaps(const View& o) const;
    const View& operator=(const View& o) const;
    const View& operator=(const Matrix& o) const;
    View& operator=(const View& o) {
        static_cast<const View&>(*this) = o;
        return *this;
    }
    View& operator=(const Matrix& o) {
        static_cast<const View&>(*this) = o;
        return *this;
    }
    const View& operator+=(const View& o) const;
    const View& operator-=(const View& o) const;
    const View& operator*=(double s) const {
        for (Index j = 0; j < c; ++j)
            for (Index i = 0; i < r; ++i) (*this)(i, j) *= s;
        return *this;
    }
    const View& operator/=(double s) const {
        for (Index j = 0; j < c; ++j)
            for (Index i = 0; i < r; ++i) (*this)(i, j) /= s;
        return *this;
    }
};

// -------------------------------------------------------------- Matrix ---
// Column-major dynamic matrix; VectorXd is the same class with one column.
class Matrix {
public:
    std::vector<double> a;
    Index r = 0, c = 0;

    Matrix() = default;
    template <class I, class = std::enable_if_t<std::is_integral_v<I>>>
    explicit Matrix(I n) : a(static_cast<size_t>(n), 0.0), r(static_cast<Index>(n)), c(1) {}
    template <class I, class J, class = std::enable_if_t<std::is_integral_v<I> && std::is_integral_v<J>>>
    Matrix(I nr, J nc) : a(static_cast<size_t>(nr) * static_cast<size_t>(nc), 0.0), r(static_cast<Index>(nr)), c(static_cast<Index>(nc)) {}
    Matrix(const View& v) : a(static_cast<size_t>(v.r * v.c)), r(v.r), c(v.c) {
        for (Index j = 0; j < c; ++j)
            for (Index i = 0; i < r; ++i) a[j * r + i] = v(i, j);
    }
    template <class Sparse, class = decltype(std::declval<const Sparse&>().outerIndexPtr())>
    explicit Matrix(const Sparse& S) : a(static_cast<size_t>(S.rows()) * S.cols(), 0.0), r(S.rows()), c(S.cols()) {
        for (Index j = 0; j < c; ++j)
            for (int k = S.outerIndexPtr()[j]; k < S.outerIndexPtr()[j + 1]; ++k)
                a[j * r + S.innerIndexPtr()[k]] = S.valuePtr()[k];
    }
    Matrix(const Matrix&) = default;
    Matrix(Matrix&&) = default;
    Matrix& operator=(const Matrix&) = default;
    Matrix& operator=(Matrix&&) = default;
    Matrix& operator=(const View& v) {
        Matrix t(v);
        *this = std::move(t);
        return *this;
    }

    View view() const { return View(const_cast<double*>(a.data()), r, c, 1, r); }
    operator View() const { return view(); }

    Index rows() const { return r; }
    Index cols() const { return c; }
    Index size() const { return r * c; }
    double* data() { return a.data(); }
    const double* data() const { return a.data(); }
    double& operator()(Index i, Index j) { return a[j * r + i]; }
    double operator()(Index i, Index j) const { return a[j * r + i]; }
    double& operator()(Index i) { return a[i]; }
    double operator()(Index i) const { return a[i]; }
    double& operator[](Index i) { return a[i]; }
    double operator[](Index i) const { return a[i]; }

    static Matrix Zero(Index n) { return Matrix(n); }
    static Matrix Zero(Index nr, Index nc) { return Matrix(nr, nc); }
    static Matrix Ones(Index n) {
        Matrix m(n);
        std::fill(m.a.begin(), m.a.end(), 1.0);
        return m;
    }
    static Matrix Identity(Index nr, Index nc) {
        Matrix m(nr, nc);
        for (Index i = 0; i < std::min(nr, nc); ++i) m(i, i) = 1.0;
        return m;
    }

    void resize(Index n) { resize(n, 1); }
    void resize(Index nr, Index nc) {
        if (nr * nc != r * c) a.assign(static_cast<size_t>(nr * nc), 0.0);
        r = nr;
        c = nc;
    }
    void conservativeResize(Index n) { conservativeResize(n, c == 0 ? 1 : c); }
    void conservativeResize(Index nr, NoChange_t) { conservativeResize(nr, c); }
    void conservativeResize(Index nr, Index nc) {
        Matrix m(nr, nc);
        for (Index j = 0; j < std::min(nc, c); ++j)
            for (Index i = 0; i < std::min(nr, r); ++i) m(i, j) = (*this)(i, j);
        *this = std::move(m);
    }
    Matrix& noalias() { return *this; }
    void setZero() { std::fill(a.begin(), a.end(), 0.0); }
    void setIdentity() { view().setIdentity(); }

    // views
    View block(Index i, Index j, Index nr, Index nc) const { return view().block(i, j, nr, nc); }
    View row(Index i) const { return view().row(i); }
    View col(Index j) const { return view().col(j); }
    View topRows(Index n) const { return view().topRows(n); }
    View bottomRows(Index n) const { return view().bottomRows(n); }
    View middleRows(Index i, Index n) const { return view().middleRows(i, n); }
    View leftCols(Index n) const { return view().leftCols(n); }
    View rightCols(Index n) const { return view().rightCols(n); }
    View middleCols(Index j, Index n) const { return view().middleCols(j, n); }
    View topLeftCorner(Index nr, Index nc) const { return view().topLeftCorner(nr, nc); }
    View bottomRightCorner(Index nr, Index nc) const { return view().bottomRightCorner(nr, nc); }
    View segment(Index i, Index n) const { return view().segment(i, n); }
    View head(Index n) const { return view().head(n); }
    View tail(Index n) const { return view().tail(n); }
    View transpose() const { return view().transpose(); }
    template <int Mode>
    TriView<Mode> triangularView() const;

    double squaredNorm() const { return view().squaredNorm(); }
    double norm() const { return view().norm(); }
    double maxCoeff() const { return view().maxCoeff(); }
    double sum() const { return view().sum(); }
    bool isZero(double prec = 0.0) const { return view().isZero(prec); }
    bool isIdentity(double prec = 0.0) const { return view().isIdentity(prec); }
    Matrix cwiseAbs() const { return view().cwiseAbs(); }
    Matrix cwiseProduct(const View& o) const { return view().cwiseProduct(o); }

    Matrix& operator+=(const View& o) {
        view() += o;
        return *this;
    }
    Matrix& operator-=(const View& o) {
        view() -= o;
        return *this;
    }
    Matrix& operator*=(double s) {
        for (double& x : a) x *= s;
        return *this;
    }
    Matrix& operator/=(double s) {
        for (double& x : a) x /= s;
        return *this;
    }
};

using MatrixXd = Matrix;
using VectorXd = Matrix;

// --------------------------------------------------- View out-of-line ---
inline bool View::overlaps(const View& o) const {
    if (size() == 0 || o.size() == 0) return false;
    auto span = [](const View& v, const double*& lo, const double*& hi) {
        const double* a = v.p;
        const double* b = v.p + (v.r - 1) * v.rs + (v.c - 1) * v.cs;
        lo = std::min(a, b);
        hi = std::max(a, b);
    };
    const double *l1, *h1, *l2, *h2;
    span(*this, l1, h1);
    span(o, l2, h2);
    return !(h1 < l2 || h2 < l1);
}
inline const View& View::operator=(const View& o) const {
    assert(o.r == r && o.c == c);
    if (overlaps(o)) {
        Matrix t(o);
        return *this = t;
    }
    for (Index j = 0; j < c; ++j)
        for (Index i = 0; i < r; ++i) (*this)(i, j) = o(i, j);
    return *this;
}
inline const View& View::operator=(const Matrix& o) const {
    assert(o.r == r && o.c == c);
    for (Index j = 0; j < c; ++j)
        for (Index i = 0; i < r; ++i) (*this)(i, j) = o(i, j);
    return *this;
}
inline const View& View::operator+=(const View& o) const {
    assert(o.r == r && o.c == c);
    Matrix t(o);
    for (Index j = 0; j < c; ++j)
        for (Index i = 0; i < r; ++i) (*this)(i, j) += t(i, j);
    return *this;
}
inline const View& View::operator-=(const View& o) const {
    assert(o.r == r && o.c == c);
    Matrix t(o);
    for (Index j = 0; j < c; ++j)
        for (Index i = 0; i < r; ++i) (*this)(i, j) -= t(i, j);
    return *this;
}
inline Matrix View::cwiseAbs() const {
    Matrix m(*this);
    for (double& x : m.a) x = std::abs(x);
    return m;
}
inline Matrix View::cwiseProduct(const View& o) const {
    Matrix m(*this);
    for (Index j = 0; j < c; ++j)
        for (Index i = 0; i < r; ++i) m(i, j) *= o(i, j);
    return m;
}

// ----------------------------------------------------------- arithmetic ---
inline Matrix operator*(const View& A, const View& B) {
    assert(A.c == B.r);
    Matrix C(A.r, B.c);
    for (Index j = 0; j < B.c; ++j)
        for (Index i = 0; i < A.r; ++i) {
            double s = 0.0;
            for (Index k = 0; k < A.c; ++k) s += A(i, k) * B(k, j);
            C(i, j) = s;
        }
    return C;
}
inline Matrix operator*(const Matrix& A, const Matrix& B) { return A.view() * B.view(); }
inline Matrix operator*(const Matrix& A, const View& B) { return A.view() * B; }
inline Matrix operator*(const View& A, const Matrix& B) { return A * B.view(); }
inline Matrix operator*(double s, const View& A) {
    Matrix m(A);
    for (double& x : m.a) x = s * x;
    return m;
}
inline Matrix operator*(double s, const Matrix& A) { return s * A.view(); }
inline Matrix operator*(const View& A, double s) {
    Matrix m(A);
    for (double& x : m.a) x = x * s;
    return m;
}
inline Matrix operator*(const Matrix& A, double s) { return A.view() * s; }
inline Matrix operator/(const View& A, double s) {
    Matrix m(A);
    for (double& x : m.a) x = x / s;
    return m;
}
inline Matrix operator/(const Matrix& A, double s) { return A.view() / s; }
inline Matrix operator-(const View& A) {
    Matrix m(A);
    for (double& x : m.a) x = -x;
    return m;
}
inline Matrix operator-(const Matrix& A) { return -A.view(); }
inline Matrix operator+(const View& A, const View& B) {
    Matrix m(A);
    for (Index j = 0; j < m.c; ++j)
        for (Index i = 0; i < m.r; ++i) m(i, j) += B(i, j);
    return m;
}
inline Matrix operator+(const Matrix& A, const Matrix& B) { return A.view() + B.view(); }
inline Matrix operator+(const Matrix& A, const View& B) { return A.view() + B; }
inline Matrix operator+(const View& A, const Matrix& B) { return A + B.view(); }
inline Matrix operator-(const View& A, const View& B) {
    Matrix m(A);
    for (Index j = 0; j < m.c; ++j)
        for (Index i = 0; i < m.r; ++i) m(i, j) -= B(i, j);
    return m;
}
inline Matrix operator-(const Matrix& A, const Matrix& B) { return A.view() - B.view(); }
inline Matrix operator-(const Matrix& A, const View& B) { return A.view() - B; }
inline Matrix operator-(const View& A, const Matrix& B) { return A - B.view(); }

// ------------------------------------------------------ triangularView ---
template <int Mode>
struct TriView {
    View t;
    bool in(Index i, Index j) const { return Mode == Upper ? i <= j : i >= j; }
    Matrix operator*(const View& B) const {
        Matrix C(t.r, B.c);
        for (Index j = 0; j < B.c; ++j)
            for (Index i = 0; i < t.r; ++i) {
                double s = 0.0;
                for (Index k = 0; k < t.c; ++k)
                    if (in(i, k)) s += t(i, k) * B(k, j);
                C(i, j) = s;
            }
        return C;
    }
    Matrix operator*(const Matrix& B) const { return (*this) * B.view(); }
    // T X = B (OnTheLeft) or X T = B (OnTheRight), in place in B.
    template <int Side = OnTheLeft>
    void solveInPlace(View B) const {
        const Index n = t.r;
        if (Side == OnTheLeft) {
            for (Index j = 0; j < B.c; ++j) {
                if (Mode == Upper)
                    for (Index i = n - 1; i >= 0; --i) {
                        double s = B(i, j);
                        for (Index k = i + 1; k < n; ++k) s -= t(i, k) * B(k, j);
                        B(i, j) = s / t(i, i);
                    }
                else
                    for (Index i = 0; i < n; ++i) {
                        double s = B(i, j);
                        for (Index k = 0; k < i; ++k) s -= t(i, k) * B(k, j);
                        B(i, j) = s / t(i, i);
                    }
            }
        } else {  // X T = B  <=>  T^T X^T = B^T
            for (Index i = 0; i < B.r; ++i) {
                if (Mode == Upper)
                    for (Index j = 0; j < n; ++j) {
                        double s = B(i, j);
                        for (Index k = 0; k < j; ++k) s -= B(i, k) * t(k, j);
                        B(i, j) = s / t(j, j);
                    }
                else
                    for (Index j = n - 1; j >= 0; --j) {
                        double s = B(i, j);
                        for (Index k = j + 1; k < n; ++k) s -= B(i, k) * t(k, j);
                        B(i, j) = s / t(j, j);
                    }
            }
        }
    }
    template <int Side = OnTheLeft>
    void solveInPlace(Matrix& B) const {
        solveInPlace<Side>(B.view());
    }
};
template <int Mode>
TriView<Mode> View::triangularView() const {
    return TriView<Mode>{*this};
}
template <int Mode>
TriView<Mode> Matrix::triangularView() const {
    return TriView<Mode>{view()};
}

// ------------------------------------------------------- Ref and Map ---
template <class M>
class Ref : public View {
public:
    Ref(const View& v) : View(v) {}
    Ref(Matrix& m) : View(m.view()) {}
    Ref(const Ref&) = default;
    using View::operator=;
    Ref& operator=(const Ref& o) {
        static_cast<const View&>(*this) = static_cast<const View&>(o);
        return *this;
    }
};

template <class M>
class Map : public View {
public:
    Map(double* p, Index n) : View(p, n, 1, 1, n) {}
    Map(double* p, Index nr, Index nc) : View(p, nr, nc, 1, nr) {}
};

// -------------------------------------------------------- HouseholderQR ---
template <class M>
class HouseholderQR {
public:
    explicit HouseholderQR(const Matrix& B) : qr_(B), h_(std::min(B.rows(), B.cols())) {
        const Index m = qr_.r, n = qr_.c;
        for (Index k = 0; k < std::min(m, n); ++k) {
            double tail2 = 0.0;
            for (Index i = k + 1; i < m; ++i) tail2 += qr_(i, k) * qr_(i, k);
            const double c0 = qr_(k, k);
            double tau, beta;
            if (tail2 <= std::numeric_limits<double>::min()) {
                tau = 0.0;
                beta = c0;
                for (Index i = k + 1; i < m; ++i) qr_(i, k) = 0.0;
            } else {
                beta = std::sqrt(c0 * c0 + tail2);
                if (c0 >= 0.0 || c0 * c0 <= 1e-20 * tail2) beta = -beta;
                const double den = c0 - beta;
                for (Index i = k + 1; i < m; ++i) qr_(i, k) /= den;
                tau = (beta - c0) / beta;
            }
            qr_(k, k) = beta;
            h_(k) = tau;
            if (tau == 0.0) continue;
            for (Index j = k + 1; j < n; ++j) {  // applyHouseholderOnTheLeft
                double w = qr_(k, j);
                for (Index i = k + 1; i < m; ++i) w += qr_(i, k) * qr_(i, j);
                qr_(k, j) -= tau * w;
                const double tw = tau * w;
                for (Index i = k + 1; i < m; ++i) qr_(i, j) -= tw * qr_(i, k);
            }
        }
    }
    const Matrix& matrixQR() const { return qr_; }
    const Matrix& hCoeffs() const { return h_; }

private:
    Matrix qr_, h_;
};

// ----------------------------------------------------------- sparse ---
template <class T>
class Triplet {
public:
    Triplet(int r = 0, int c = 0, T v = T(0)) : r_(r), c_(c), v_(v) {}
    int row() const { return r_; }
    int col() const { return c_; }
    T value() const { return v_; }

private:
    int r_, c_;
    T v_;
};

template <class T>
class SparseMatrix;

template <class T>
struct SparseTranspose {
    const SparseMatrix<T>& s;
};

template <class T>
class SparseMatrix {
public:
    SparseMatrix() : outer_(1, 0) {}
    SparseMatrix(Index nr, Index nc) : r_(nr), c_(nc), outer_(static_cast<size_t>(nc) + 1, 0) {}

    Index rows() const { return r_; }
    Index cols() const { return c_; }
    Index nonZeros() const { return static_cast<Index>(val_.size()); }
    void makeCompressed() {}
    const int* outerIndexPtr() const { return outer_.data(); }
    const int* innerIndexPtr() const { return inner_.data(); }
    const T* valuePtr() const { return val_.data(); }
    int* outerIndexPtr() { return outer_.data(); }
    int* innerIndexPtr() { return inner_.data(); }
    T* valuePtr() { return val_.data(); }

    // Duplicates are summed in input order; rows end up strictly increasing per column.
    template <class It>
    void setFromTriplets(It b, It e) {
        std::vector<int> cnt(static_cast<size_t>(c_) + 1, 0);
        for (It it = b; it != e; ++it) ++cnt[it->col() + 1];
        for (Index j = 0; j < c_; ++j) cnt[j + 1] += cnt[j];
        const size_t nt = static_cast<size_t>(cnt[c_]);
        std::vector<int> ri(nt);
        std::vector<T> rv(nt);
        std::vector<size_t> seq(nt);
        std::vector<int> pos(cnt.begin(), cnt.end() - 1);
        size_t s = 0;
        for (It it = b; it != e; ++it, ++s) {
            const int q = pos[it->col()]++;
            ri[q] = it->row();
            rv[q] = it->value();
            seq[q] = s;
        }
        outer_.assign(static_cast<size_t>(c_) + 1, 0);
        inner_.clear();
        val_.clear();
        std::vector<size_t> ord;
        for (Index j = 0; j < c_; ++j) {
            ord.resize(static_cast<size_t>(cnt[j + 1] - cnt[j]));
            for (size_t k = 0; k < ord.size(); ++k) ord[k] = static_cast<size_t>(cnt[j]) + k;
            std::stable_sort(ord.begin(), ord.end(), [&](size_t x, size_t y) { return ri[x] < ri[y]; });
            for (size_t k = 0; k < ord.size(); ++k) {
                if (k > 0 && ri[ord[k]] == ri[ord[k - 1]])
                    val_.back() += rv[ord[k]];
                else {
                    inner_.push_back(ri[ord[k]]);
                    val_.push_back(rv[ord[k]]);
                }
            }
            outer_[j + 1] = static_cast<int>(val_.size());
        }
        (void)seq;
    }
    // prune(ref, eps): keep entries that are not much smaller than ref (|v| > |ref|*eps).
    void prune(T ref, T eps) {
        const T thr = std::abs(ref) * eps;
        std::vector<int> no(outer_.size(), 0);
        size_t w = 0;
        for (Index j = 0; j < c_; ++j) {
            for (int k = outer_[j]; k < outer_[j + 1]; ++k)
                if (std::abs(val_[k]) > thr) {
                    inner_[w] = inner_[k];
                    val_[w] = val_[k];
                    ++w;
                }
            no[j + 1] = static_cast<int>(w);
        }
        inner_.resize(w);
        val_.resize(w);
        outer_ = std::move(no);
    }

    class InnerIterator {
    public:
        InnerIterator(const SparseMatrix& m, Index j)
            : m_(const_cast<SparseMatrix&>(m)), k_(m.outer_[j]), e_(m.outer_[j + 1]), j_(j) {}
        explicit operator bool() const { return k_ < e_; }
        InnerIterator& operator++() {
            ++k_;
            return *this;
        }
        Index row() const { return m_.inner_[k_]; }
        Index col() const { return j_; }
        Index index() const { return row(); }
        T value() const { return m_.val_[k_]; }
        T& valueRef() { return m_.val_[k_]; }

    private:
        SparseMatrix& m_;
        int k_, e_;
        Index j_;
    };

    SparseTranspose<T> transpose() const { return {*this}; }

private:
    Index r_ = 0, c_ = 0;
    std::vector<int> outer_, inner_;
    std::vector<T> val_;
    friend class InnerIterator;
};

// A x: columns accumulated in ascending order.
inline Matrix operator*(const SparseMatrix<double>& A, const Matrix& x) {
    Matrix y(A.rows());
    const int* p = A.outerIndexPtr();
    const int* ii = A.innerIndexPtr();
    const double* v = A.valuePtr();
    for (Index j = 0; j < A.cols(); ++j) {
        const double xj = x(j);
        for (int k = p[j]; k < p[j + 1]; ++k) y(ii[k]) += v[k] * xj;
    }
    return y;
}
// A^T y: one dot per column, rows ascending.
inline Matrix operator*(const SparseTranspose<double>& At, const Matrix& y) {
    const SparseMatrix<double>& A = At.s;
    Matrix x(A.cols());
    const int* p = A.outerIndexPtr();
    const int* ii = A.innerIndexPtr();
    const double* v = A.valuePtr();
    for (Index j = 0; j < A.cols(); ++j) {
        double s = 0.0;
        for (int k = p[j]; k < p[j + 1]; ++k) s += v[k] * y(ii[k]);
        x(j) = s;
    }
    return x;
}

}  // namespace Eigen
