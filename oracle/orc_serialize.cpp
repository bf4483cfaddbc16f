// ORACLE — test infrastructure only (see oracle/orc_core.h).
//
// Restatement of the reference's factorization file format "SPQRFW01"
// (proj/src/transforms.cpp:129-289, save_factorization / load_factorization):
// little-endian, every integer a signed 64-bit field, every real an IEEE
// double.  Layout:
//   "SPQRFW01" | M | N | eps | ivec pivot_row | ivec dropped_rows |
//   ivec trailing_rows | nW | nW x factor | has_q | [nQ | nQ x (ivec rows, refl)]
//   ivec   = n, then n integers
//   mat    = rows, cols, then the entries column by column
//   vec    = n, then n reals
//   refl   = mat V, vec tau, vec sign
//   factor = tag 0: ivec cols, mat R, ivec coupled, mat C   (TriangularScale)
//            tag 1: ivec cols, refl Q                       (ColumnRotation)
// A negative size is a corrupt file; unknown tags, a bad magic or a short read
// raise std::runtime_error with the reference's messages.
#include <cstdint>
#include <cstring>
#include <fstream>
#include <stdexcept>
#include <string>

#include "orc_core.h"

namespace orc {

namespace {

const char kMagic[8] = {'S', 'P', 'Q', 'R', 'F', 'W', '0', '1'};

struct Writer {
    std::ofstream& o;
    void i64(std::int64_t v) { o.write(reinterpret_cast<const char*>(&v), 8); }
    void f64(double v) { o.write(reinterpret_cast<const char*>(&v), 8); }
    void ivec(const std::vector<Index>& v) {
        i64(static_cast<std::int64_t>(v.size()));
        for (Index x : v) i64(x);
    }
    void mat(const Mat& m) {
        i64(m.r);
        i64(m.c);
        for (Index j = 0; j < m.c; ++j)
            for (Index i = 0; i < m.r; ++i) f64(m(i, j));
    }
    void vec(const Vec& v) {
        i64(static_cast<std::int64_t>(v.size()));
        for (double x : v) f64(x);
    }
    void refl(const ReflectorSet& h) {
        mat(h.V);
        vec(h.tau);
        vec(h.sign);
    }
};

struct Reader {
    std::ifstream& in;
    std::int64_t i64() {
        std::int64_t v = 0;
        in.read(reinterpret_cast<char*>(&v), 8);
        return in ? v : 0;
    }
    double f64() {
        double v = 0.0;
        in.read(reinterpret_cast<char*>(&v), 8);
        return v;
    }
    std::int64_t size() {
        const std::int64_t n = i64();
        if (n < 0) throw std::runtime_error("corrupt size field in factorization file");
        return n;
    }
    std::vector<Index> ivec() {
        std::vector<Index> v(static_cast<size_t>(size()));
        for (auto& x : v) x = static_cast<Index>(i64());
        return v;
    }
    Mat mat() {
        const std::int64_t r = size(), c = size();
        Mat m(static_cast<Index>(r), static_cast<Index>(c));
        for (Index j = 0; j < c; ++j)
            for (Index i = 0; i < r; ++i) m(i, j) = f64();
        return m;
    }
    Vec vec() {
        Vec v(static_cast<size_t>(size()));
        for (auto& x : v) x = f64();
        return v;
    }
    ReflectorSet refl() {
        ReflectorSet h;
        h.V = mat();
        h.tau = vec();
        h.sign = vec();
        return h;
    }
};

}  // namespace

void save_factorization(const Factorization& f, const std::string& path) {
    std::ofstream o(path, std::ios::binary);
    if (!o) throw std::runtime_error("cannot open " + path + " for writing");
    Writer w{o};
    o.write(kMagic, 8);
    w.i64(f.M);
    w.i64(f.N);
    w.f64(f.eps);
    w.ivec(f.pivot_row);
    w.ivec(f.dropped_rows);
    w.ivec(f.trailing_rows);
    w.i64(static_cast<std::int64_t>(f.W.size()));
    for (const WFactor& x : f.W) {
        if (const auto* t = std::get_if<TriangularScale>(&x)) {
            w.i64(0);
            w.ivec(t->cols);
            w.mat(t->R);
            w.ivec(t->coupled);
            w.mat(t->C);
        } else {
            const auto& r = std::get<ColumnRotation>(x);
            w.i64(1);
            w.ivec(r.cols);
            w.refl(r.Q);
        }
    }
    w.i64(f.has_q ? 1 : 0);
    if (f.has_q) {
        w.i64(static_cast<std::int64_t>(f.Q.size()));
        for (const RowReflect& q : f.Q) {
            w.ivec(q.rows);
            w.refl(q.H);
        }
    }
    if (!o) throw std::runtime_error("write failed: " + path);
}

Factorization load_factorization(const std::string& path) {
    std::ifstream in(path, std::ios::binary);
    if (!in) throw std::runtime_error("cannot open " + path);
    char magic[8];
    in.read(magic, 8);
    if (!in || std::memcmp(magic, kMagic, 8) != 0) throw std::runtime_error(path + ": not a factorization file (bad magic)");
    Reader r{in};
    Factorization f;
    f.M = static_cast<Index>(r.i64());
    f.N = static_cast<Index>(r.i64());
    f.eps = r.f64();
    f.pivot_row = r.ivec();
    f.dropped_rows = r.ivec();
    f.trailing_rows = r.ivec();
    const std::int64_t nw = r.size();
    for (std::int64_t i = 0; i < nw; ++i) {
        const std::int64_t tag = r.i64();
        if (tag == 0) {
            TriangularScale t;
            t.cols = r.ivec();
            t.R = r.mat();
            t.coupled = r.ivec();
            t.C = r.mat();
            f.W.emplace_back(std::move(t));
        } else if (tag == 1) {
            ColumnRotation c;
            c.cols = r.ivec();
            c.Q = r.refl();
            f.W.emplace_back(std::move(c));
        } else {
            throw std::runtime_error(path + ": unknown factor tag");
        }
    }
    f.has_q = r.i64() != 0;
    if (f.has_q) {
        const std::int64_t nq = r.size();
        for (std::int64_t i = 0; i < nq; ++i) {
            RowReflect q;
            q.rows = r.ivec();
            q.H = r.refl();
            f.Q.push_back(std::move(q));
        }
    }
    if (!in) throw std::runtime_error(path + ": truncated file");
    return f;
}

}  // namespace orc
