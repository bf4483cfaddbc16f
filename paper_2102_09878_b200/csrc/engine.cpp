// GPU spaQR engine (Algorithm 1, proj/src/factorize.cpp:17-791).
//
// Division of labour.  The host owns STRUCTURE: cluster ids, row-id lists,
// the key sets of every front, holders, and every decision that the
// reference takes (row selection, keysets, pivots, reassignment targets,
// coupling pruning, ranks) — taken from small statistics vectors computed on
// the GPU.  The GPU owns all FP64 front data.  Each phase of a stage is a
// fixed number of batched launches:
//   eliminate : stats -> [sync] -> gather stacks, QR + Q^T apply, post stats
//               -> [sync] -> scatter/append/W copies as ONE assemble launch
//   scale     : identity test -> [sync] -> QR + U^T apply + [I;0], TRSM
//   sparsify  : gather + truncated CPQR -> [sync] -> write-back (rows);
//               per dependency wave: gather G + CPQR -> [sync] -> assemble (cols)
//   merge     : one assemble launch into the next stage's arena.
// Within one eliminate batch the host replays the reference's sequential
// bookkeeping exactly, on symbolic rows (a row's values are "row r of old
// front f, overridden by row s of stack S_c for the stack's keys"); the
// gathers then materialise every touched front once.
#include "engine.h"

#include <algorithm>
#include <climits>
#include <cmath>
#include <cstdarg>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <iterator>
#include <condition_variable>
#include <deque>
#include <functional>
#ifdef _OPENMP
#include <omp.h>
#endif
#include <map>
#include <mutex>
#include <thread>
#include <string>

#include "dev.h"

namespace spqr {

long long DeviceFactorization::nnz_w() const {  // transforms.cpp:25-38
    long long s = 0;
    for (const auto& f : W) {
        const long long c = f.c, k = f.k;
        if (f.kind == 0)
            s += c * (c + 1) / 2 + c * k;
        else
            s += k * c - k * (k - 1) / 2 + k;
    }
    return s;
}

namespace {

struct KeyRef {
    int key, width, col;
};

struct Front {
    bool live = false;
    std::vector<int> rows;
    std::vector<KeyRef> keys;  // ascending key; device layout: own key first, then ascending
    double* mat = nullptr;
    bool big = false;  // mat from cudaMallocAsync (released stream-ordered when superseded)
    int ld = 0, ncols = 0;
    bool scaled_ok = false;
    std::vector<long long> soff;  // pre-stage row statistics offset per key (eliminate)
    std::vector<int> tag;         // per row append tag within the current stage (empty: all -1)
    int find(int key) const {
        auto it = std::lower_bound(keys.begin(), keys.end(), key, [](const KeyRef& a, int k) { return a.key < k; });
        return (it != keys.end() && it->key == key) ? static_cast<int>(it - keys.begin()) : -1;
    }
    int nrows() const { return static_cast<int>(rows.size()); }
    // dead after a merge: emptied but keeps its storage (freed with the engine, off the
    // critical path) — freeing ~10^5 small vectors per merge contended on malloc's locks
    void retire() {
        live = false;
        rows.clear();
        keys.clear();
        mat = nullptr;
        big = false;
        ld = ncols = 0;
        scaled_ok = false;
        soff.clear();
        tag.clear();
    }
};

// symbolic row: values of old front `base` row `brow`, overridden by stack
// `sidx` row `srow` on that stack's neighbour keys.
struct PRow {
    int gid, base, brow, sidx, srow, tag;  // tag: cluster whose move_extras appended the row this stage (-1: none)
};
struct KW {
    int key, width;
};
struct PFront {
    std::vector<PRow> rows;
    std::vector<KW> keys;  // ascending
    int find(int key) const {
        auto it = std::lower_bound(keys.begin(), keys.end(), key, [](const KW& a, int k) { return a.key < k; });
        return (it != keys.end() && it->key == key) ? static_cast<int>(it - keys.begin()) : -1;
    }
    void add(int key, int w) {
        auto it = std::lower_bound(keys.begin(), keys.end(), key, [](const KW& a, int k) { return a.key < k; });
        if (it == keys.end() || it->key != key) keys.insert(it, KW{key, w});
    }
    void erase(int key) {
        auto it = std::lower_bound(keys.begin(), keys.end(), key, [](const KW& a, int k) { return a.key < k; });
        if (it != keys.end() && it->key == key) keys.erase(it);
    }
};

// holders[key]: fronts holding a block of key.  Appends are O(1); the set is
// sorted/deduplicated lazily when read (reads need ascending order).
struct HolderSet {
    std::vector<int> v;
    bool dirty = false;
    void add(int x) {
        v.push_back(x);
        dirty = true;
    }
    void remove(int x) {
        norm();
        auto it = std::lower_bound(v.begin(), v.end(), x);
        if (it != v.end() && *it == x) v.erase(it);
    }
    void clear() {
        v.clear();
        dirty = false;
    }
    const std::vector<int>& get() {
        norm();
        return v;
    }
    void norm() {
        if (!dirty) return;
        std::sort(v.begin(), v.end());
        v.erase(std::unique(v.begin(), v.end()), v.end());
        dirty = false;
    }
};

void sorted_insert(std::vector<int>& v, int x) {
    auto it = std::lower_bound(v.begin(), v.end(), x);
    if (it == v.end() || *it != x) v.insert(it, x);
}

// Host-side profile (SPQR_PROF=1 prints it to stderr after the factorization).
struct HostProf {
    enum { INIT, STATS, SYNC, PASS1, SBUILD, PASS2, MATER, SCALE, SROWS, SCOLS, MERGE, UPLOAD, DEPS, FETCH, N };
    double t[N] = {0};
    long long n[N] = {0};
    static const char* name(int i) {
        static const char* s[N] = {"init", "stats", "sync_wait", "pass1", "stack_build", "pass2", "materialize",
                                   "scale", "sparsify_rows", "sparsify_cols", "merge", "upload", "deps", "fetch"};
        return s[i];
    }
};
// named fine-grained scopes (string literals as keys)
struct NamedProf {
    std::vector<std::pair<const char*, double>> v;
    double& slot(const char* n) {
        for (auto& p : v)
            if (p.first == n) return p.second;
        v.emplace_back(n, 0.0);
        return v.back().second;
    }
};
// the host-profile scopes only read the clock when SPQR_PROF is set (they are on
// every wave's path)
inline bool host_prof_on() {
    static const bool on = std::getenv("SPQR_PROF") != nullptr;
    return on;
}
struct NScope {
    double& t;
    double t0;
    NScope(NamedProf& p, const char* n) : t(p.slot(n)), t0(host_prof_on() ? now_s() : 0.0) {}
    ~NScope() {
        if (host_prof_on()) t += now_s() - t0;
    }
};
struct ProfScope {
    HostProf& p;
    int i;
    double t0;
    ProfScope(HostProf& p_, int i_) : p(p_), i(i_), t0(host_prof_on() ? now_s() : 0.0) {}
    ~ProfScope() {
        if (!host_prof_on()) return;
        p.t[i] += now_s() - t0;
        p.n[i]++;
    }
};

// CUDA-event accounting per kernel family; resolved at every host sync.
class KTimer {
public:
    ~KTimer() {
        for (auto e : pool_) cudaEventDestroy(e);
    }
    cudaEvent_t begin(cudaStream_t st) {
        cudaEvent_t e = take();
        CK(cudaEventRecord(e, st));
        return e;
    }
    // route >= 0: also accumulated per CPQR route (SPQR_PROF breakdown), with `probs` problems
    void end(int tag, cudaEvent_t e0, cudaStream_t st, double bytes, int route = -1, double probs = 0) {
        cudaEvent_t e1 = take();
        CK(cudaEventRecord(e1, st));
        pend_.push_back({tag, e0, e1, bytes, route, probs});
    }
    void resolve(EngineCounters& c) {
        for (auto& p : pend_) {
            float ms = 0.f;
            CK(cudaEventElapsedTime(&ms, p.e0, p.e1));
            c.k_ms[p.tag] += ms;
            c.k_bytes[p.tag] += p.bytes;
            c.k_launches[p.tag] += 1;
            if (p.route >= 0) {
                c.route_ms[p.route] += ms;
                c.route_probs[p.route] += p.probs;
                c.route_launches[p.route] += 1;
            }
        }
        pend_.clear();
        used_ = 0;
    }

private:
    struct P {
        int tag;
        cudaEvent_t e0, e1;
        double bytes;
        int route;
        double probs;
    };
    std::vector<cudaEvent_t> pool_;
    std::vector<P> pend_;
    size_t used_ = 0;
    cudaEvent_t take() {
        if (used_ == pool_.size()) {
            cudaEvent_t e;
            CK(cudaEventCreate(&e));
            pool_.push_back(e);
        }
        return pool_[used_++];
    }
};

// One elimination of the current batch.
struct Elim {
    int c = -1, cs = 0;
    std::vector<int> parts;
    std::vector<int> keys;  // [c, keyset...]
    std::vector<int> off;   // column offsets in S
    std::vector<PRow> srows;
    int total_rows = 0, tcols = 0, nsel_c = 0;
    double* S = nullptr;
    bool sbig = false;
    int* flag = nullptr;  // device
    // deferred effects of the parallel host passes
    std::vector<std::pair<int, int>> hadd;  // holders_[key].add(front)
    std::string err;                        // error text raised inside a parallel pass
    bool logic = false;                     // err is an internal logic error
    std::vector<int> keepk, coupled;        // pruned coupling (W factor)
    int kept = 0;
    std::vector<std::pair<int, int>> dest;  // move_extras: (target, local row), ascending target
    std::vector<int> trail;                 // move_extras: rows to the trailing set
    int color = 0;
    double cmax2 = 0.0;  // largest squared row norm of the c blocks (move_extras noise floor scale)
    void reset(int c_, int cs_) {
        c = c_;
        cs = cs_;
        cmax2 = 0.0;
        hadd.clear();
        err.clear();
        logic = false;
        keepk.clear();
        coupled.clear();
        kept = 0;
        dest.clear();
        trail.clear();
        parts.clear();
        keys.clear();
        off.clear();
        srows.clear();
        total_rows = tcols = nsel_c = 0;
        S = nullptr;
        sbig = false;
        flag = nullptr;
        post_off = -1;
    }
    // post statistics (host): block max / nz of pivot rows; own non-pivot row sums per key
    long long post_off = -1;
};

// Per-thread scratch of the parallel elimination passes.
struct Scratch {
    std::vector<size_t> rv_off;
    std::vector<double> rv_sq, bw;
    std::vector<unsigned char> rv_nz;
    std::vector<std::vector<int>> sel;
    std::vector<int> keyset, spos, best, cand;
    std::vector<PRow> rows;
};

// Allocator whose value-initialisation is default-initialisation: vectors that
// receive device downloads are resized without zero-filling them first.
template <class T>
struct NoInitAlloc : std::allocator<T> {
    template <class U>
    struct rebind {
        using other = NoInitAlloc<U>;
    };
    NoInitAlloc() = default;
    template <class U>
    NoInitAlloc(const NoInitAlloc<U>&) {}
    template <class U>
    void construct(U* p) noexcept {
        ::new (static_cast<void*>(p)) U;
    }
    template <class U, class... A>
    void construct(U* p, A&&... a) {
        ::new (static_cast<void*>(p)) U(std::forward<A>(a)...);
    }
};
template <class T>
using dl_vector = std::vector<T, NoInitAlloc<T>>;

// Growable array of trivially copyable elements whose growth does not
// value-initialise (the row maps are rewritten in parallel right after).
template <class T>
struct PodVec {
    std::unique_ptr<T[]> p;
    size_t n = 0, cap = 0;
    void reserve(size_t c) {
        if (c <= cap) return;
        const size_t nc = std::max(c, 2 * cap);
        std::unique_ptr<T[]> q(new T[nc]);
        if (n) std::memcpy(q.get(), p.get(), n * sizeof(T));
        p = std::move(q);
        cap = nc;
    }
    void resize_uninit(size_t m) {
        reserve(m);
        n = m;
    }
    void resize(size_t m, const T& v) {
        reserve(m);
        for (size_t i = n; i < m; ++i) p[i] = v;
        n = m;
    }
    void shrink(size_t m) { n = std::min(n, m); }
    T& operator[](size_t i) { return p[i]; }
    const T* data() const { return p.get(); }
    size_t size() const { return n; }
    void clear() { n = 0; }
};

// Stage arenas and pinned staging buffers outlive one factorization: a new
// Engine takes them from this pool (per device) and returns them, so repeated
// factorizations in a process do not pay cudaMalloc / cudaMallocHost again.  The
// pool is never destroyed (no CUDA calls during process teardown).
struct HostBuilders;
struct ArenaPool {
    std::mutex mu;
    std::map<int, std::vector<std::unique_ptr<DeviceArena>>> dev;
    std::vector<std::unique_ptr<PinnedArena>> pin;
    std::vector<std::unique_ptr<HostBuilders>> host;
    static ArenaPool& get() {
        static ArenaPool* p = new ArenaPool;
        return *p;
    }
};

// Assemble job builder (generic gather, dev.h).
struct AsmBuilder {
    std::vector<AsmDst> dst;
    PodVec<int4> rowref;
    std::vector<int> segoff, kmap;
    std::vector<AsmSrc> src;
    long long elems = 0;
    // init_rows = false: the caller writes every row map entry itself
    int begin(double* p, int ld, int nrows, int ncols, int nsrc, int nseg, bool init_rows = true) {
        AsmDst d;
        d.p = p;
        d.ld = ld;
        d.nrows = nrows;
        d.ncols = ncols;
        d.nsrc = nsrc;
        d.nseg = std::max(nseg, 1);
        d.trans = 0;
        d.row_off = static_cast<long long>(rowref.size());
        d.seg_off = static_cast<long long>(segoff.size());
        d.kmap_off = static_cast<long long>(kmap.size());
        d.src_off = static_cast<long long>(src.size());
        d.elem_off = elems;
        elems += static_cast<long long>(nrows) * ncols;
        if (init_rows)
            rowref.resize(rowref.size() + nrows, int4{-1, 0, -1, 0});
        else
            rowref.resize_uninit(rowref.size() + nrows);
        segoff.resize(segoff.size() + d.nseg + 1, 0);
        segoff[d.seg_off + d.nseg] = ncols;
        kmap.resize(kmap.size() + static_cast<size_t>(d.nseg) * nsrc, -1);
        src.resize(src.size() + nsrc);
        dst.push_back(d);
        return static_cast<int>(dst.size()) - 1;
    }
    void seg(int di, int q, int start) { segoff[dst[di].seg_off + q] = start; }
    int& km(int di, int q, int s) { return kmap[dst[di].kmap_off + static_cast<long long>(q) * dst[di].nsrc + s]; }
    int4& row(int di, int i) { return rowref[dst[di].row_off + i]; }
    AsmSrc& source(int di, int s) { return src[dst[di].src_off + s]; }
    void drop_if_empty() {
        if (!dst.empty() && (dst.back().nrows == 0 || dst.back().ncols == 0)) {
            const AsmDst d = dst.back();
            elems = d.elem_off;
            rowref.shrink(d.row_off);
            segoff.resize(d.seg_off);
            kmap.resize(d.kmap_off);
            src.resize(d.src_off);
            dst.pop_back();
        }
    }
    void clear() {
        dst.clear();
        rowref.clear();
        segoff.clear();
        kmap.clear();
        src.clear();
        elems = 0;
    }
};

// materialize_pending's per-front plan (kept by the engine between calls)
struct MatPlan {
    int f = -1;
    bool same = false;
    Front nf;
    std::vector<int> bases, stacks, ord;
    int di = -1;
};

struct HostBuilders {
    AsmBuilder wcopy;    // W copies + materialised fronts
    AsmBuilder slot[6];  // one per gather call site
};

// key indices of a front in physical column order
inline void phys_order(const std::vector<KeyRef>& keys, std::vector<int>& ord) {
    ord.resize(keys.size());
    for (size_t i = 0; i < keys.size(); ++i) ord[i] = static_cast<int>(i);
    std::sort(ord.begin(), ord.end(), [&](int a, int b) { return keys[a].col < keys[b].col; });
}

// One persistent background thread frees the engines' host containers (hundreds of thousands
// of small vectors) off the caller's critical path; it drains its queue and is joined when the
// library is unloaded / the process exits.
class Reaper {
public:
    static Reaper& get() {
        static Reaper r;
        return r;
    }
    void post(std::function<void()> f) {
        {
            std::lock_guard<std::mutex> lk(mu_);
            q_.push_back(std::move(f));
        }
        cv_.notify_one();
    }
    ~Reaper() {
        {
            std::lock_guard<std::mutex> lk(mu_);
            stop_ = true;
        }
        cv_.notify_one();
        if (th_.joinable()) th_.join();
    }

private:
    Reaper() : th_([this] { run(); }) {}
    void run() {
        std::unique_lock<std::mutex> lk(mu_);
        for (;;) {
            cv_.wait(lk, [this] { return stop_ || !q_.empty(); });
            if (q_.empty() && stop_) return;
            auto f = std::move(q_.front());
            q_.pop_front();
            lk.unlock();
            f();
            lk.lock();
        }
    }
    std::mutex mu_;
    std::condition_variable cv_;
    std::deque<std::function<void()>> q_;
    bool stop_ = false;
    std::thread th_;
};

// The library's own stream-ordered pool per device for big fronts and stacks: it keeps freed
// memory cached across waves and factorizations (release threshold = max) without touching
// the device's default pool, which other allocators in the process (torch, the caller) use.
cudaMemPool_t engine_pool(int dev) {
    static std::mutex mu;
    static std::vector<cudaMemPool_t> pools;
    std::lock_guard<std::mutex> lk(mu);
    if (static_cast<int>(pools.size()) <= dev) pools.resize(dev + 1, nullptr);
    if (!pools[dev]) {
        cudaMemPoolProps props{};
        props.allocType = cudaMemAllocationTypePinned;
        props.location.type = cudaMemLocationTypeDevice;
        props.location.id = dev;
        CK(cudaMemPoolCreate(&pools[dev], &props));
        uint64_t thr = UINT64_MAX;
        CK(cudaMemPoolSetAttribute(pools[dev], cudaMemPoolAttrReleaseThreshold, &thr));
    }
    return pools[dev];
}

class Engine {
public:
    Engine(const Csc& A, const ClusterHierarchy& h, const std::vector<int>& owner, const FactorizeOptions& opt,
           cudaStream_t st, const FactorizeObserver* obs = nullptr)
        : A_(A), h_(h), opt_(opt), st_(st), L_(h.num_levels), obs_(obs) {
        out_.M = A.m;
        out_.N = A.n;
        out_.eps = opt.eps;
        out_.pivot_row.assign(A.n, -1);
        out_.warena = std::make_unique<DeviceArena>(size_t(128) << 20);
        out_.has_q = opt.store_q;
        if (opt.ranks > 1) {
            out_.rank.ranks = opt.ranks;
            out_.rank.owner = rank_owners(h, ata_graph(A), opt.ranks);
        }
        if (opt.dist && opt.dist->size > 1) {
            dist_ = opt.dist;
            dist_owner_ = rank_owners(h, ata_graph(A), dist_->size);
            // the split stages: from the leaves down to the first stage that sparsifies (its
            // eliminations still precede any scale_all) and above the top lg levels
            int lg = 0;
            while ((1 << lg) < dist_->size) ++lg;
            const int ksp = (opt.eps > 0.0 && L_ + 1 - opt.skip_levels >= 2) ? L_ + 1 - opt.skip_levels : 0;
            dist_kend_ = std::max(lg + 1, ksp);
            dist_top_.assign(h.clusters.size(), 0);  // pieces of the top lg separators: every rank keeps them
            for (size_t c = 0; c < h.clusters.size(); ++c) dist_top_[c] = h.tree->nodes[h.clusters[c].tree_node].level <= lg;
            // merges stay inside one subtree (or among the top pieces): a parent cluster has its
            // children's tree node, so the partitioned state is closed under merge_level
            for (size_t c = 0; c < h.clusters.size(); ++c) {
                const int P = h.clusters[c].parent;
                if (P >= 0 && (dist_top_[P] != dist_top_[c] || (!dist_top_[c] && dist_owner_[P] != dist_owner_[c])))
                    throw std::logic_error("distributed factorization: a merge crosses subtrees (cluster " + std::to_string(c) + ")");
            }
            if (opt.store_q) throw std::invalid_argument("a distributed factorization does not record Q");
        }
        if (opt.store_q) out_.qarena = std::make_unique<DeviceArena>(size_t(64) << 20);
        const size_t nc = h.clusters.size();
        fr_.resize(nc);
        cols_.resize(nc);
        gone_.assign(nc, 0);
        alive_.assign(nc, 0);
        holders_.resize(nc);
        pend_id_.assign(nc, -1);
        mark_.assign(nc, 0);
        colmask_.assign(nc, 0);
        stage_of_.assign(nc, 0);
        for (size_t c = 0; c < nc; ++c) stage_of_[c] = (h.clusters[c].level == h.clusters[c].stage) ? h.clusters[c].stage : 0;
        stage_list_.resize(L_ + 2);
        for (size_t c = 0; c < nc; ++c) {
            const auto& C = h.clusters[c];
            if (C.level == C.stage && C.stage >= 1 && C.stage <= L_ + 1) stage_list_[C.stage].push_back(static_cast<int>(c));
        }
        tree_clusters_.resize(h.tree->nodes.size());
        for (size_t c = 0; c < nc; ++c) tree_clusters_[h.clusters[c].tree_node].push_back(static_cast<int>(c));
        {
            int dev = 0;
            CK(cudaGetDevice(&dev));
            dev_ = dev;
            pool_ = engine_pool(dev);
        }
        CK(cudaEventCreate(&ev0_));
        CK(cudaEventCreate(&ev1_));
        {  // stage arenas and pinned staging come from the process-wide pool (kept across factorizations)
            ArenaPool& P = ArenaPool::get();
            std::lock_guard<std::mutex> lk(P.mu);
            auto& dv = P.dev[dev_];
            for (auto& a : arena_) {
                if (!dv.empty()) {
                    a = std::move(dv.back());
                    dv.pop_back();
                } else {
                    a = std::make_unique<DeviceArena>();
                }
            }
            if (!P.pin.empty()) {
                pin_ = std::move(P.pin.back());
                P.pin.pop_back();
            } else {
                pin_ = std::make_unique<PinnedArena>();
            }
            if (!P.host.empty()) {
                hp_ = std::move(P.host.back());
                P.host.pop_back();
            } else {
                hp_ = std::make_unique<HostBuilders>();
            }
            hp_->wcopy.clear();
        }
        init_fronts(owner);
    }
    ~Engine() {
        if (dist_vbuf_) cudaFree(dist_vbuf_);  // an exchange that failed before rank 0's ack
        {  // the per-cluster host containers (hundreds of thousands of small vectors) are
           // freed on a background thread instead of on the caller's critical path
            struct Trash {
                std::vector<Front> fr;
                std::vector<std::vector<int>> cols, sl, tc, sb;
                std::vector<HolderSet> holders;
                std::deque<PFront> pend;
                std::vector<Elim> el;
                std::vector<MatPlan> plans;
            };
            auto* t = new Trash{std::move(fr_),      std::move(cols_),    std::move(stage_list_), std::move(tree_clusters_),
                                std::move(sb_bases_), std::move(holders_), std::move(pend_),      std::move(el_),
                                std::move(mplans_)};
            Reaper::get().post([t] { delete t; });
        }
        cudaStreamSynchronize(st_);  // nothing may still use the arenas when they go back to the pool
        cudaEventDestroy(ev0_);
        cudaEventDestroy(ev1_);
        ArenaPool& P = ArenaPool::get();
        std::lock_guard<std::mutex> lk(P.mu);
        for (auto& a : arena_)
            if (a) {
                a->reset();
                P.dev[dev_].push_back(std::move(a));
            }
        if (pin_) {
            pin_->reset();
            P.pin.push_back(std::move(pin_));
        }
        if (hp_) P.host.push_back(std::move(hp_));
    }

    DeviceFactorization run();

private:
    const Csc& A_;
    const ClusterHierarchy& h_;
    FactorizeOptions opt_;
    cudaStream_t st_;
    int L_;
    const FactorizeObserver* obs_ = nullptr;
    int cur_stage_ = 0;
    // SPQR_DUMP_G=<stage>:<cluster>:<path> writes that interface's sparsify_cols input G
    // (cs x nG, column-major, int32 dims first) before each of its CPQRs (parity diagnostics)
    struct GDump {
        int stage = -1, cluster = -1;
        std::string path;
        GDump() {
            if (const char* e = std::getenv("SPQR_DUMP_G")) {
                const std::string v(e);
                const size_t a = v.find(':'), b = v.find(':', a + 1);
                if (a != std::string::npos && b != std::string::npos) {
                    stage = std::atoi(v.substr(0, a).c_str());
                    cluster = std::atoi(v.substr(a + 1, b - a - 1).c_str());
                    path = v.substr(b + 1);
                }
            }
        }
    } gdump_;
    void dump_g(const double* dG, int cs, int nG) {
        CK(cudaStreamSynchronize(st_));
        std::vector<double> h(static_cast<size_t>(cs) * nG);
        if (!h.empty()) CK(cudaMemcpy(h.data(), dG, sizeof(double) * h.size(), cudaMemcpyDeviceToHost));
        if (std::FILE* f = std::fopen(gdump_.path.c_str(), "wb")) {
            const int dims[2] = {cs, nG};
            std::fwrite(dims, 4, 2, f);
            std::fwrite(h.data(), 8, h.size(), f);
            std::fclose(f);
        }
    }
    // SPQR_DIGEST=<path> (parity diagnostics, tools/phase_digest.py): after every stage-level
    // phase, one record per live front: cluster, #rows, #keys, a polynomial hash of its row ids,
    // of its (key, width) list and — with SPQR_DIGEST_VALUES=1 — of its significance pattern
    // (row-key blocks whose squared norm exceeds 1e-20 x the front's largest).  The oracle writes
    // the same records (ORC_DIGEST, oracle/orc_capi.cpp), so the first diverging phase and front
    // can be found without moving whole states.
    void digest(int phase_id) {
        static const char* path = std::getenv("SPQR_DIGEST");
        if (!path) return;
        static const bool values = std::getenv("SPQR_DIGEST_VALUES") != nullptr;
        CK(cudaStreamSynchronize(st_));
        auto mix = [](uint64_t h, uint64_t x) { return h * 1000003ull + x + 1; };
        std::vector<int> rec;
        std::vector<uint64_t> hs;
        std::vector<double> buf;
        for (size_t c = 0; c < fr_.size(); ++c) {
            if (!alive_[c] || !fr_[c].live) continue;
            const Front& F = fr_[c];
            uint64_t hr = 0, hk = 0, hv = 0;
            for (int r : F.rows) hr = mix(hr, static_cast<uint64_t>(r));
            for (const KeyRef& k : F.keys) hk = mix(mix(hk, static_cast<uint64_t>(k.key)), static_cast<uint64_t>(k.width));
            if (values && F.nrows() > 0 && F.ncols > 0 && F.mat) {
                buf.resize(static_cast<size_t>(F.ld) * F.ncols);
                CK(cudaMemcpy(buf.data(), F.mat, sizeof(double) * buf.size(), cudaMemcpyDeviceToHost));
                std::vector<double> nq(static_cast<size_t>(F.nrows()) * F.keys.size(), 0.0);
                double mx = 0;
                for (int r = 0; r < F.nrows(); ++r)
                    for (size_t q = 0; q < F.keys.size(); ++q) {
                        double s = 0;
                        for (int j = 0; j < F.keys[q].width; ++j) {
                            const double x = buf[static_cast<size_t>(F.keys[q].col + j) * F.ld + r];
                            s += x * x;
                        }
                        nq[r * F.keys.size() + q] = s;
                        mx = std::max(mx, s);
                    }
                for (double s : nq) hv = mix(hv, s > 1e-20 * mx ? 1u : 0u);
            }
            rec.push_back(static_cast<int>(c));
            rec.push_back(F.nrows());
            rec.push_back(static_cast<int>(F.keys.size()));
            hs.push_back(hr);
            hs.push_back(hk);
            hs.push_back(hv);
        }
        // SPQR_DUMP_FRONTS=<c1,c2,...>: those fronts in full (rows, keys, per-row per-key squared
        // norms) as text (<path>.fronts.txt), the same lines the oracle writes
        static std::vector<int> dumpc = [] {
            std::vector<int> v;
            if (const char* e = std::getenv("SPQR_DUMP_FRONTS"))
                for (const char* q = e; *q;) {
                    v.push_back(std::atoi(q));
                    while (*q && *q != ',') ++q;
                    if (*q == ',') ++q;
                }
            return v;
        }();
        if (!dumpc.empty())
            if (std::FILE* fp = std::fopen((std::string(path) + ".fronts.txt").c_str(), "a")) {
                for (int c : dumpc) {
                    if (c < 0 || static_cast<size_t>(c) >= fr_.size() || !alive_[c] || !fr_[c].live) continue;
                    const Front& F = fr_[c];
                    std::fprintf(fp, "phase %d stage %d front %d rows %zu keys", phase_id, cur_stage_, c, F.rows.size());
                    for (const KeyRef& k : F.keys) std::fprintf(fp, " %d:%d", k.key, k.width);
                    std::fprintf(fp, "\n");
                    buf.assign(static_cast<size_t>(F.ld) * std::max(F.ncols, 0), 0.0);
                    if (!buf.empty() && F.mat)
                        CK(cudaMemcpy(buf.data(), F.mat, sizeof(double) * buf.size(), cudaMemcpyDeviceToHost));
                    for (int r = 0; r < F.nrows(); ++r) {
                        std::fprintf(fp, "  row %d", F.rows[r]);
                        for (const KeyRef& k : F.keys) {
                            double s = 0;
                            for (int j = 0; j < k.width; ++j) {
                                const double x = buf[static_cast<size_t>(k.col + j) * F.ld + r];
                                s += x * x;
                            }
                            std::fprintf(fp, " %.6e", s);
                        }
                        std::fprintf(fp, "\n");
                    }
                }
                std::fclose(fp);
            }
        static bool first = true;
        if (std::FILE* f = std::fopen(path, first ? "wb" : "ab")) {
            const int head[3] = {phase_id, cur_stage_, static_cast<int>(hs.size() / 3)};
            std::fwrite(head, 4, 3, f);
            std::fwrite(rec.data(), 4, rec.size(), f);
            std::fwrite(hs.data(), 8, hs.size(), f);
            std::fclose(f);
        }
        first = false;
    }
    // factorize.cpp:86-95: the state after a phase, downloaded for the observer (tests only)
    void notify(const char* phase, int detail, const std::vector<int>* wave = nullptr) {
        if (phase[0] != 'e' || wave == nullptr) {
            static const char* names[5] = {"eliminate", "scale", "sparsify_rows", "sparsify_cols", "merge"};
            for (int i = 1; i < 5; ++i)
                if (std::string(phase) == names[i]) digest(i);
        }
        if (!obs_ || !*obs_) return;
        CK(cudaStreamSynchronize(st_));
        static const bool structure_only = std::getenv("SPQR_OBSERVE_STRUCTURE_ONLY") != nullptr;
        EngineView v;
        std::vector<double> buf;
        for (size_t c = 0; c < fr_.size(); ++c) {
            if (!alive_[c] || !fr_[c].live) continue;
            const Front& F = fr_[c];
            v.front_cluster.push_back(static_cast<int>(c));
            v.rows.insert(v.rows.end(), F.rows.begin(), F.rows.end());
            v.rows_ptr.push_back(static_cast<int>(v.rows.size()));
            const int nr = F.nrows();
            if (!structure_only) {
                buf.assign(static_cast<size_t>(F.ld) * std::max(F.ncols, 0), 0.0);
                if (!buf.empty() && F.mat)
                    CK(cudaMemcpy(buf.data(), F.mat, sizeof(double) * buf.size(), cudaMemcpyDeviceToHost));
            }
            for (const KeyRef& k : F.keys) {  // ascending keys
                v.keys.push_back(k.key);
                v.key_width.push_back(k.width);
                v.block_off.push_back(static_cast<long long>(v.values.size()));
                if (structure_only) continue;  // SPQR_OBSERVE_STRUCTURE_ONLY: rows, keys and widths only
                for (int j = 0; j < k.width; ++j)
                    for (int r = 0; r < nr; ++r) v.values.push_back(buf[static_cast<size_t>(k.col + j) * F.ld + r]);
            }
            v.keys_ptr.push_back(static_cast<int>(v.keys.size()));
        }
        for (const auto& cl : cols_) {
            v.cols.insert(v.cols.end(), cl.begin(), cl.end());
            v.cols_ptr.push_back(static_cast<int>(v.cols.size()));
        }
        if (wave) v.wave = *wave;
        v.pivots = npiv_;
        v.dropped = static_cast<long long>(out_.dropped_rows.size());
        v.trailing = static_cast<long long>(out_.trailing_rows.size());
        (*obs_)(phase, cur_stage_, detail, v);
    }
    std::vector<Front> fr_;
    std::vector<std::vector<int>> cols_;
    std::vector<char> gone_;
    std::vector<char> alive_;  // mirror of fr_[c].live, scanned instead of the Front objects
    std::vector<HolderSet> holders_;
    std::vector<std::vector<int>> stage_list_, tree_clusters_;
    // distributed stages (opt.dist): owner rank per cluster; the stages L+1 ..
    // dist_kend_ split their eliminations by subtree
    const DistTransport* dist_ = nullptr;
    std::vector<int> dist_owner_;
    int dist_kend_ = 0;
    bool dist_stage(int k) const { return dist_ && k >= dist_kend_; }
    std::vector<std::vector<int>> start_rows_;      // every front's rows at the start of the stage
    std::vector<char> dist_ghost_;                  // other subtrees' clusters alive on their ranks (columns tracked here)
    std::vector<int> dist_touched_;                 // fronts this rank's eliminations touched
    std::vector<std::pair<int, int>> dist_tr_;      // (front, row) rows they transformed in place
    std::vector<char> dist_top_;                    // 1: a top-separator piece (kept by every rank)
    struct SnapE {
        int c, cs;
        double asp;
    };
    std::map<int, std::vector<SnapE>> dist_snap_;  // split stage -> its snapshot entries by cluster
    std::vector<std::pair<int, size_t>> dist_tseg_; // (stage, end) of this rank's trailing rows per split stage
    bool dist_mine(int c) const { return !dist_top_[c] && dist_owner_[c] == dist_->rank; }
    void dist_partition_state();
    std::vector<char> dist_export(int k, bool final_to_root);
    void dist_apply(const std::vector<std::vector<char>>& msgs, bool final_to_root);
    double* dist_vbuf_ = nullptr;  // exported values (CUDA IPC) until every peer acknowledges
    void dist_exchange(int k, int err_cluster, const std::string& err_reason);
    void rebuild_holders() {
        for (auto& hs : holders_) hs.clear();
        for (size_t c = 0; c < fr_.size(); ++c)
            if (alive_[c] && fr_[c].live)
                for (const KeyRef& kr : fr_[c].keys) holders_[kr.key].add(static_cast<int>(c));
    }
    DeviceFactorization out_;
    std::unique_ptr<DeviceArena> arena_[2];
    int cur_ = 0, dev_ = 0;
    cudaMemPool_t pool_ = nullptr;
    std::unique_ptr<PinnedArena> pin_;
    Index npiv_ = 0;
    int batch_ = 0;
    cudaEvent_t ev0_, ev1_;
    KTimer kt_;
    HostProf prof_;
    NamedProf nprof_;
    std::vector<int> waves_per_stage_;
    struct StageProf {
        int stage = 0, waves = 0, scol_waves = 0;
        long long s_elems = 0, s_max_rows = 0, s_max_cols = 0, mat_fronts = 0, mat_rows = 0, mat_elems = 0, elims = 0;
        long long max_front_rows = 0, max_front_cols = 0;
        double t[HostProf::N] = {0};
    };
    std::vector<StageProf> sprof_;
    int spec_depth_ = std::getenv("SPQR_SPEC_DEPTH") ? std::atoi(std::getenv("SPQR_SPEC_DEPTH")) : 3;
    // eliminate-batch state
    std::deque<PFront> pend_;  // deque: references stay valid while new fronts become pending
    size_t npend_ = 0;
    std::vector<int> pend_id_, pend_list_;
    std::vector<Elim> el_;
    std::vector<std::vector<int>> sb_bases_;  // per-elimination source fronts (pool)
    std::vector<char> mark_;
    std::vector<int> stage_of_;
    std::vector<std::pair<int, int>> dep_;
    std::unique_ptr<HostBuilders> hp_;  // assemble builders, pooled across factorizations
    std::vector<MatPlan> mplans_;       // materialize_pending plans, reused between waves
    AsmBuilder& asm_slot(int i) {  // one per call site: vectors keep their capacity
        hp_->slot[i].clear();
        return hp_->slot[i];
    }
    dl_vector<double> pre_sq_, post_sq_;
    dl_vector<unsigned char> pre_nz_, post_nz_;
    // first error in reference order
    int err_cluster_ = -1;
    std::string err_reason_;

    DeviceArena& arena() { return *arena_[cur_]; }
    // Large matrices (3D fronts, big stacks) are allocated stream-ordered and
    // released as soon as the launch that consumes them is enqueued, so a
    // stage's peak footprint is its live data, not everything it rebuilt.
    static constexpr size_t kBig = size_t(4) << 20;
    double* dalloc(DeviceArena& ar, size_t n, bool& big) {
        const size_t bytes = sizeof(double) * std::max<size_t>(n, 1);
        big = bytes >= kBig;
        if (!big) return ar.alloc_n<double>(std::max<size_t>(n, 1));
        void* p = nullptr;
        CK(cudaMallocFromPoolAsync(&p, bytes, pool_, st_));
        return static_cast<double*>(p);
    }
    void dfree(double* p, bool big) {
        if (big && p) CK(cudaFreeAsync(p, st_));
    }
    Uploader up() { return Uploader{&arena(), pin_.get(), st_}; }
    int width(int key) const { return static_cast<int>(cols_[key].size()); }

    void sync() {
        {
            ProfScope ps(prof_, HostProf::SYNC);
            CK(cudaStreamSynchronize(st_));
        }
        CK(cudaGetLastError());  // a failed launch must not pass silently
        pin_->reset();
        kt_.resolve(out_.ctr);
        out_.ctr.syncs++;
    }
    // batched device->host copies with a single stream sync
    struct Pending {
        void* host;
        void* pin;
        size_t bytes;
    };
    std::vector<Pending> dl_;
    template <class T, class A>
    void enqueue(std::vector<T, A>& h, const T* d, size_t n) {
        if (h.capacity() < n) {  // grow without copying the stale contents
            h.clear();
            h.reserve(n);
        }
        h.resize(n);
        if (n == 0) return;
        void* p = pin_->alloc(sizeof(T) * n);
        CK(cudaMemcpyAsync(p, d, sizeof(T) * n, cudaMemcpyDeviceToHost, st_));
        dl_.push_back({h.data(), p, sizeof(T) * n});
        out_.ctr.d2h_bytes += sizeof(T) * n;
    }
    void fetch() {
        ProfScope ps(prof_, HostProf::FETCH);
        {
            ProfScope pw(prof_, HostProf::SYNC);
            CK(cudaStreamSynchronize(st_));
        }
        CK(cudaGetLastError());  // a failed launch must not pass silently
        for (auto& q : dl_) par_memcpy(q.host, q.pin, q.bytes);
        dl_.clear();
        pin_->reset();
        kt_.resolve(out_.ctr);
        out_.ctr.syncs++;
    }
    template <class T, class A>
    void download(std::vector<T, A>& h, const T* d, size_t n) {
        if (h.capacity() < n) {
            h.clear();
            h.reserve(n);
        }
        h.resize(n);
        if (n == 0) return;
        T* p = static_cast<T*>(pin_->alloc(sizeof(T) * n));
        CK(cudaMemcpyAsync(p, d, sizeof(T) * n, cudaMemcpyDeviceToHost, st_));
        sync();
        par_memcpy(h.data(), p, sizeof(T) * n);
        out_.ctr.d2h_bytes += sizeof(T) * n;
    }
    void flush_assemble(AsmBuilder& b) {
        if (b.dst.empty() || b.elems == 0) {
            b.clear();
            return;
        }
        ProfScope ps(prof_, HostProf::UPLOAD);
        Uploader u = up();
        const AsmDst* d = u.put(b.dst);
        const int4* rr = u.put(b.rowref.data(), b.rowref.size());
        const int* so = u.put(b.segoff);
        const int* km = u.put(b.kmap);
        const AsmSrc* s = u.put(b.src);
        out_.ctr.h2d_bytes += u.bytes_h2d;
        cudaEvent_t e0 = kt_.begin(st_);
        launch_assemble(d, static_cast<int>(b.dst.size()), b.elems, rr, so, km, s, st_);
        kt_.end(K_ASSEMBLE, e0, st_, 16.0 * b.elems);
        out_.ctr.launches++;
        b.clear();
    }
    void record_error(int cluster, const std::string& why) {
        if (err_cluster_ < 0) {
            err_cluster_ = cluster;
            err_reason_ = why;
        }
    }
    void raise_if_error() {
        if (err_cluster_ >= 0) throw SingularFrontError(err_cluster_, err_reason_);
    }

    // column layout: own key first, then ascending keys
    void layout(int self, std::vector<KeyRef>& keys, int& ncols) const {
        int o = 0;
        for (auto& k : keys)
            if (k.key == self) {
                k.col = 0;
                o = k.width;
            }
        for (auto& k : keys)
            if (k.key != self) {
                k.col = o;
                o += k.width;
            }
        ncols = o;
    }

    void init_fronts(const std::vector<int>& owner);
    // size-split batched launches (shared-memory staged when the block fits)
    void run_qr(const std::vector<QrDesc>& qd, const QrDesc* dq, Uploader& u) {
        std::vector<int> small, large, huge;
        size_t smem = 0;
        // column-tiled path (qr_tile.cu) for every front whose panel fits in shared memory
        std::vector<int> cls(qd.size(), -1);
        size_t tsmem[5] = {0, 0, 0, 0, 0};
        int tcount[5] = {0, 0, 0, 0, 0};
        int* qcount = nullptr;
        static const bool no_tile = std::getenv("SPQR_QR_PATH") && std::string(std::getenv("SPQR_QR_PATH")) != "tile";
        for (size_t i = 0; i < qd.size(); ++i) {
            cls[i] = no_tile ? -1 : qr_tile_class(qd[i].m, qd[i].n);
            if (cls[i] < 0) continue;
            tsmem[cls[i]] = std::max<size_t>(tsmem[cls[i]], qr_tile_smem(cls[i], qd[i].n));
            ++tcount[cls[i]];
        }
        for (int c = 0; c < 5; ++c) {
            if (!tcount[c]) continue;
            std::vector<int> ids;
            for (size_t i = 0; i < qd.size(); ++i)
                if (cls[i] == c) ids.push_back(static_cast<int>(i));
            const std::vector<int4> wk = qr_tile_plan(qd.data(), ids.data(), static_cast<int>(ids.size()), sm_count());
            const int4* dw = u.put(wk);
            double qb = 0;
            for (size_t i = 0; i < qd.size(); ++i)
                if (cls[i] == c) qb += 16.0 * qd[i].m * qd[i].ntot;
            cudaEvent_t e0 = kt_.begin(st_);
            if (!qcount) {
                qcount = arena().alloc_n<int>(qd.size());
                cudaMemsetAsync(qcount, 0, sizeof(int) * qd.size(), st_);
            }
            static const bool check = std::getenv("SPQR_QR_CHECK") != nullptr;
            std::vector<std::vector<double>> before;
            if (check) {
                cudaStreamSynchronize(st_);
                for (int i : ids) {
                    const QrDesc& q = qd[i];
                    before.emplace_back(static_cast<size_t>(q.m) * q.ntot);
                    cudaMemcpy2D(before.back().data(), 8 * q.m, q.a, 8 * q.ld, 8 * q.m, q.ntot, cudaMemcpyDeviceToHost);
                }
            }
            launch_qr_tile(c, dq, dw, static_cast<int>(wk.size()), tsmem[c], qcount, st_);
            kt_.end(K_QR, e0, st_, qb);
            if (check) {
                cudaStreamSynchronize(st_);
                const cudaError_t le = cudaGetLastError();
                if (le != cudaSuccess) std::fprintf(stderr, "[qr check] cls %d launch error %s (smem %zu)\n", c, cudaGetErrorString(le), tsmem[c]);
                int* didx = nullptr;
                cudaMalloc(&didx, sizeof(int));
                for (size_t t = 0; t < ids.size(); ++t) {
                    const QrDesc& q = qd[ids[t]];
                    std::vector<double> tile(static_cast<size_t>(q.m) * q.ntot), old(tile.size());
                    cudaMemcpy2D(tile.data(), 8 * q.m, q.a, 8 * q.ld, 8 * q.m, q.ntot, cudaMemcpyDeviceToHost);
                    cudaMemcpy2D(q.a, 8 * q.ld, before[t].data(), 8 * q.m, 8 * q.m, q.ntot, cudaMemcpyHostToDevice);
                    cudaMemcpy(didx, &ids[t], sizeof(int), cudaMemcpyHostToDevice);
                    launch_qr_split(dq, nullptr, 0, 0, didx, 1, st_);
                    cudaStreamSynchronize(st_);
                    cudaMemcpy2D(old.data(), 8 * q.m, q.a, 8 * q.ld, 8 * q.m, q.ntot, cudaMemcpyDeviceToHost);
                    double md = 0, mx = 0;
                    long long arg = -1;
                    for (size_t z = 0; z < old.size(); ++z) {
                        mx = std::max(mx, std::fabs(old[z]));
                        if (std::fabs(old[z] - tile[z]) > md) {
                            md = std::fabs(old[z] - tile[z]);
                            arg = static_cast<long long>(z);
                        }
                    }
                    if (md > 1e-9 * (1 + mx))
                        std::fprintf(stderr, "[qr check] cls %d desc %d m %d n %d ntot %d ld %d set_id %d zl %d rout %d: max diff %.3e at (%lld,%lld) of %.3e\n",
                                     c, ids[t], q.m, q.n, q.ntot, q.ld, q.set_identity, q.zero_lower, q.rout != nullptr, md,
                                     arg % q.m, arg / q.m, mx);
                    if (md > 1e-9 * (1 + mx))
                        std::fprintf(stderr, "    before %.6e tile %.6e old %.6e\n", before[t][arg], tile[arg], old[arg]);
                }
                cudaFree(didx);
            }
        }
        for (size_t i = 0; i < qd.size(); ++i) {
            if (cls[i] >= 0) continue;
            const size_t b = qr_smem_bytes(qd[i].m, qd[i].n, qd[i].ntot);
            if (b <= kSmemBudget && qd[i].n <= 1024) {
                small.push_back(static_cast<int>(i));
                smem = std::max(smem, b);
            } else if (b > kBlockedQrBytes && qd[i].n >= 16) {
                huge.push_back(static_cast<int>(i));
            } else {
                large.push_back(static_cast<int>(i));
            }
        }
        // big fronts: panel factorisation + compact-WY trailing updates on DMMA (mbqr.cu)
        for (int i : huge) {
            const QrDesc& q = qd[i];
            cudaEvent_t e0 = kt_.begin(st_);
            double* scratch = arena().alloc_n<double>(2 * static_cast<size_t>(q.n) + 32 * 32);
            blocked_qr_apply(1, q.m, q.n, q.ntot, q.a, q.tau ? q.tau : scratch, q.sign ? q.sign : scratch + q.n, q.flag,
                             scratch + 2 * q.n, st_, q.ld);
            blocked_qr_post(q.a, q.ld, q.m, q.n, q.rout, q.set_identity, q.zero_lower, st_);
            kt_.end(K_QR, e0, st_, 16.0 * q.m * q.ntot);
        }
        if (small.empty() && large.empty()) return;
        const int* ds = u.put(small);
        const int* dl = u.put(large);
        double qb = 0;
        for (int i : small) qb += 16.0 * qd[i].m * qd[i].ntot;
        for (int i : large) qb += 16.0 * qd[i].m * qd[i].ntot;
        cudaEvent_t e0 = kt_.begin(st_);
        static const bool qrlog = std::getenv("SPQR_QRLOG") != nullptr;
        cudaEvent_t b0 = nullptr, b1 = nullptr;
        if (qrlog) {
            cudaEventCreate(&b0);
            cudaEventCreate(&b1);
            cudaEventRecord(b0, st_);
        }
        launch_qr_split(dq, ds, static_cast<int>(small.size()), smem, dl, static_cast<int>(large.size()), st_);
        if (qrlog) {
            cudaEventRecord(b1, st_);
            cudaEventSynchronize(b1);
            float ms = 0;
            cudaEventElapsedTime(&ms, b0, b1);
            int sm_m = 0, sm_n = 0, sm_t = 0, lg_m = 0, lg_n = 0, lg_t = 0;
            double sbytes = 0, lbytes = 0;
            for (int i : small) {
                sm_m = std::max(sm_m, qd[i].m);
                sm_n = std::max(sm_n, qd[i].n);
                sm_t = std::max(sm_t, qd[i].ntot);
                sbytes += 16.0 * qd[i].m * qd[i].ntot;
            }
            for (int i : large) {
                lg_m = std::max(lg_m, qd[i].m);
                lg_n = std::max(lg_n, qd[i].n);
                lg_t = std::max(lg_t, qd[i].ntot);
                lbytes += 16.0 * qd[i].m * qd[i].ntot;
            }
            std::fprintf(stderr, "[spqr qr batch] small %zu (max %dx%d/%d, %.1f MB) large %zu (max %dx%d/%d, %.1f MB) huge %zu  %.3f ms\n",
                         small.size(), sm_m, sm_n, sm_t, sbytes / 1e6, large.size(), lg_m, lg_n, lg_t, lbytes / 1e6,
                         huge.size(), ms);
            cudaEventDestroy(b0);
            cudaEventDestroy(b1);
        }
        kt_.end(K_QR, e0, st_, qb);
    }
    void run_cpqr(const std::vector<CpqrDesc>& cd, const CpqrDesc* dc, Uploader& u) {
        std::vector<int> small, large;
        size_t smem = 0;
        int maxm = 1;
        // Problems too big for one CTA's shared memory either run one CTA each
        // (k_cpqr, in parallel) or one at a time on the whole GPU (cpqr_big.cu).
        // Cost model (measured): one CTA streams ~20 GB/s; the cooperative
        // kernel costs ~8 us per pivot plus the trailing traffic at ~6 TB/s.
        // Move the largest problems to the cooperative kernel while that lowers
        // the estimated batch time.
        std::vector<int> glob, clus;
        size_t csmem = 0;
        std::vector<int> tall[2];
        std::vector<std::vector<int>> narrow(12);
        std::vector<char> coop(cd.size(), 0), nar(cd.size(), 0);
        static const bool no_narrow = std::getenv("SPQR_NO_NARROW") != nullptr;
        size_t nsmem[12] = {0, 0, 0, 0, 0, 0, 0, 0, 0, 0, 0, 0};
        size_t nnar = 0;
        // Narrow blocks too large for one CTA's shared memory (the in-place classes, m <= 128 by up
        // to 2048 columns: the widest sparsify_cols G at C2) go to the thread-block clusters, whose
        // CTAs each stage a column range: per pivot a cluster barrier instead of one CTA walking
        // the whole block in L2 (C2: CPQR 105 -> 77 ms).  SPQR_NARROW_IN_PLACE=1 keeps them narrow.
        static const bool glb_clus =
            std::getenv("SPQR_NARROW_IN_PLACE") == nullptr && std::getenv("SPQR_NO_CPQR_CLUSTER") == nullptr;
        for (size_t i = 0; i < cd.size(); ++i) {
            int nc = no_narrow ? -1 : cpqr_narrow_class(cd[i].m, cd[i].n);
            if (glb_clus && nc >= 0 && nc % 6 >= 3 && cd[i].n >= 16 && cpqr_clus_smem_bytes(cd[i].m, cd[i].n) <= 200 * 1024)
                nc = -1;
            if (nc >= 0) {
                narrow[nc].push_back(static_cast<int>(i));
                nar[i] = 1;
                ++nnar;
                if (nc % 6 < 3) nsmem[nc] = std::max(nsmem[nc], cpqr_narrow_smem(cd[i].m, cd[i].n));
            } else if (cpqr_smem_bytes(cd[i].m, cd[i].n) > kSmemBudget) {
                glob.push_back(static_cast<int>(i));
            }
        }
        for (int c = 0; c < 12; ++c) {
            if (narrow[c].empty()) continue;
            const int* dn = u.put(narrow[c]);
            double nb = 0;
            for (int i : narrow[c]) nb += 8.0 * cd[i].m * cd[i].n;
            // SPQR_CPQR_LOG=<path>: per narrow launch, its device time and problem shapes
            // (diagnostics; synchronises after the launch)
            static const char* clog = std::getenv("SPQR_CPQR_LOG");
            cudaEvent_t la = nullptr, lb = nullptr;
            if (clog) {
                CK(cudaEventCreate(&la));
                CK(cudaEventCreate(&lb));
                CK(cudaEventRecord(la, st_));
            }
            cudaEvent_t e0 = kt_.begin(st_);
            launch_cpqr_narrow(c, dc, dn, static_cast<int>(narrow[c].size()), nsmem[c], st_);
            kt_.end(K_CPQR, e0, st_, nb, 0, static_cast<double>(narrow[c].size()));
            if (clog) {
                CK(cudaEventRecord(lb, st_));
                CK(cudaEventSynchronize(lb));
                float ms = 0;
                CK(cudaEventElapsedTime(&ms, la, lb));
                cudaEventDestroy(la);
                cudaEventDestroy(lb);
                if (std::FILE* f = std::fopen(clog, "a")) {
                    std::fprintf(f, "L %d %d %.4f %d", cur_stage_, c, ms, static_cast<int>(narrow[c].size()));
                    for (int i : narrow[c]) std::fprintf(f, " %dx%d", cd[i].m, cd[i].n);
                    std::fprintf(f, "\n");
                    std::fclose(f);
                }
            }
        }
        if (nnar == cd.size()) return;
        // Problems too big for one CTA's shared memory run on a thread-block cluster of
        // cpqr_clus_ctas() CTAs each (k_cpqr_clus, concurrently), or — the largest — one at a
        // time on the whole GPU (k_cpqr_big).  SPQR_NO_CPQR_CLUSTER=1: one CTA each in global
        // memory instead of the clusters (the previous route, for comparison).
        static const bool use_clus = std::getenv("SPQR_NO_CPQR_CLUSTER") == nullptr;
        auto clus_ok = [&](int i) {
            return use_clus && cd[i].n >= 16 && cpqr_clus_smem_bytes(cd[i].m, cd[i].n) <= 200 * 1024;
        };
        if (!glob.empty()) {
            // estimated time off the cooperative kernel: one CTA streams ~20 GB/s; a cluster
            // ~cpqr_clus_ctas() times that plus ~3 us of cluster barriers per pivot
            static const double clus_bw =  // per-CTA streaming rate assumed for the clusters (GB/s)
                std::getenv("SPQR_CLUS_BW") ? std::atof(std::getenv("SPQR_CLUS_BW")) : 20.0;
            auto single = [&](int i) {
                const double mn = std::min(cd[i].m, cd[i].n), bytes = 16.0 * double(cd[i].m) * cd[i].n;
                return clus_ok(i) ? mn * (3e-6 + bytes / (cpqr_clus_ctas() * clus_bw * 1e9)) : mn * bytes / 20e9;
            };
            auto cost = [&](int i) {
                return std::min(cd[i].m, cd[i].n) * (8e-6 + 16.0 * double(cd[i].m) * cd[i].n / 6e12);
            };
            std::sort(glob.begin(), glob.end(), [&](int a, int b) { return single(a) > single(b); });
            const double lanes = use_clus ? std::max(1.0, double(sm_count()) / cpqr_clus_ctas()) : 2.0 * sm_count();
            std::vector<double> suf(glob.size() + 1, 0.0);
            for (size_t j = glob.size(); j-- > 0;) suf[j] = suf[j + 1] + single(glob[j]);
            double best = 1e300, ccum = 0.0;
            size_t bj = 0;
            for (size_t j = 0; j <= glob.size(); ++j) {
                const double rest = j < glob.size() ? std::max(single(glob[j]), suf[j] / lanes) : 0.0;
                if (ccum + rest < best) {
                    best = ccum + rest;
                    bj = j;
                }
                if (j < glob.size()) {
                    const int i = glob[j];
                    if (cpqr_big_smem_bytes(cd[i].m, cd[i].n) > 200 * 1024 || cd[i].m < 32) break;
                    ccum += cost(i);
                }
            }
            for (size_t j = 0; j < bj; ++j) coop[glob[j]] = 1;
        }
        for (size_t i = 0; i < cd.size(); ++i) {
            if (nar[i]) continue;
            const size_t b = cpqr_smem_bytes(cd[i].m, cd[i].n);
            if (coop[i]) {
                CpqrDesc d = cd[i];
                d.work = arena().alloc_n<double>(cpqr_big_work_doubles(d.n));
                cudaEvent_t e0 = kt_.begin(st_);
                launch_cpqr_big(d, st_);
                kt_.end(K_CPQR, e0, st_, 8.0 * d.m * d.n, 1, 1.0);
                continue;
            }
            static const bool no_tall = std::getenv("SPQR_NO_TALL") != nullptr;
            const int tc = no_tall ? -1 : cpqr_tall_class(cd[i].m, cd[i].n);
            if (b <= kSmemBudget) {
                small.push_back(static_cast<int>(i));
                smem = std::max(smem, b);
            } else if (tc >= 0) {  // 128 < m <= 512: warp-per-column kernel, in place
                tall[tc].push_back(static_cast<int>(i));
            } else if (clus_ok(static_cast<int>(i))) {
                clus.push_back(static_cast<int>(i));
                csmem = std::max(csmem, cpqr_clus_smem_bytes(cd[i].m, cd[i].n));
            } else {
                large.push_back(static_cast<int>(i));
                maxm = std::max(maxm, cd[i].m);
            }
        }
        if (!clus.empty()) {
            const int* dcl = u.put(clus);
            double cbb = 0;
            for (int i : clus) cbb += 8.0 * cd[i].m * cd[i].n;
            cudaEvent_t e0 = kt_.begin(st_);
            launch_cpqr_clus(dc, dcl, static_cast<int>(clus.size()), csmem, st_);
            kt_.end(K_CPQR, e0, st_, cbb, 4, static_cast<double>(clus.size()));
        }
        for (int c = 0; c < 2; ++c) {
            if (tall[c].empty()) continue;
            const int* dt = u.put(tall[c]);
            double tb = 0;
            for (int i : tall[c]) tb += 8.0 * cd[i].m * cd[i].n;
            cudaEvent_t e0 = kt_.begin(st_);
            launch_cpqr_tall(c, dc, dt, static_cast<int>(tall[c].size()), st_);
            kt_.end(K_CPQR, e0, st_, tb, 2, static_cast<double>(tall[c].size()));
        }
        if (small.empty() && large.empty()) return;
        const int* ds = u.put(small);
        const int* dl = u.put(large);
        double cb = 0;
        for (int i : small) cb += 8.0 * cd[i].m * cd[i].n;
        for (int i : large) cb += 8.0 * cd[i].m * cd[i].n;
        cudaEvent_t e0 = kt_.begin(st_);
        launch_cpqr_split(dc, ds, static_cast<int>(small.size()), smem, dl, static_cast<int>(large.size()), maxm, st_);
        kt_.end(K_CPQR, e0, st_, cb, 3, static_cast<double>(small.size() + large.size()));
    }
    void eliminate_stage(int k);
    void eliminate_wave(const std::vector<int>& list);
    void compute_stats(const std::vector<int>& P);
    std::vector<int> stage_fronts(const std::vector<int>& list);
    void elim_pass1(Elim& e, Scratch& S);
    void elim_prep2(Elim& e, Scratch& S);
    void elim_commit2(Elim& e);
    void flush_holder_removals();
    std::vector<std::pair<int, int>> hrem_;  // (key, eliminated cluster) removals pending for the wave
    std::vector<Scratch> tscr_;
    std::vector<uint64_t> colmask_;
    void materialize_pending();
    void scale_all();
    void sparsify_rows_all();
    void sparsify_cols_all();
    void merge_level();
    void snapshot(StageStats& st);
    int ancestor_target(int c) const;

    PFront& pend(int f) {
        if (pend_id_[f] < 0) {
            if (npend_ == pend_.size()) pend_.emplace_back();
            pend_id_[f] = static_cast<int>(npend_);
            pend_list_.push_back(f);
            PFront& P = pend_[npend_++];
            const Front& F = fr_[f];
            P.rows.resize(F.rows.size());
            for (size_t i = 0; i < F.rows.size(); ++i)
                P.rows[i] = PRow{F.rows[i], f, static_cast<int>(i), -1, 0, F.tag.empty() ? -1 : F.tag[i]};
            P.keys.resize(F.keys.size());
            for (size_t i = 0; i < F.keys.size(); ++i) P.keys[i] = KW{F.keys[i].key, F.keys[i].width};
        }
        return pend_[pend_id_[f]];
    }
    // squared norm / nonzero of a symbolic row on one key
    void rowval(const PRow& r, int key, double& sq, bool& nz, bool post_ok) const;
    // rowval for every row of a pending front, with a fast path for rows still
    // in their own front's old matrix
    void row_vals(const PFront& P, int self, int key, double* sq, unsigned char* nz, bool post_ok) const {
        const Front& B = fr_[self];
        const int qi = B.find(key);
        const long long off = (qi >= 0 && !B.soff.empty()) ? B.soff[qi] : -1;
        for (size_t q = 0; q < P.rows.size(); ++q) {
            const PRow& r = P.rows[q];
            if (r.base == self && r.sidx < 0) {
                if (off < 0) {
                    sq[q] = 0.0;
                    nz[q] = 0;
                } else {
                    sq[q] = pre_sq_[off + r.brow];
                    nz[q] = pre_nz_[off + r.brow];
                }
            } else {
                bool b;
                rowval(r, key, sq[q], b, post_ok);
                nz[q] = b;
            }
        }
    }
    std::vector<size_t> rv_off_;
    std::vector<double> rv_sq_;
    std::vector<unsigned char> rv_nz_;
    std::vector<std::vector<int>> sel_;
    std::vector<int> scr_cand_, scr_best_, scr_keyset_, scr_spos_;
    std::vector<int> qrows_scratch_;
    std::vector<double> scr_bw_;
    std::vector<std::pair<int, int>> scr_dest_;
    std::vector<PRow> scr_rows_;
    DevWFactor& new_factor(int kind, int cluster, int c, int k, const std::vector<int>& cols, const std::vector<int>* coupled) {
        DevWFactor f;
        f.kind = kind;
        f.batch = batch_;
        f.cluster = cluster;
        f.c = c;
        f.k = k;
        f.scale_only = kind == 0 && coupled == nullptr;
        f.cols_off = static_cast<long long>(out_.idx.size());
        out_.idx.insert(out_.idx.end(), cols.begin(), cols.end());
        f.coupled_off = static_cast<long long>(out_.idx.size());
        if (coupled) out_.idx.insert(out_.idx.end(), coupled->begin(), coupled->end());
        out_.W.push_back(f);
        return out_.W.back();
    }
    // store_q: one RowReflect (transforms.h:34-37) on `rows` with k reflectors; storage for V
    // (rows x k), tau and sign from the Q arena unless the caller shares a W rotation's
    DevWFactor& new_qfactor(int cluster, const int* rows, int nrows, int k, bool alloc = true) {
        DevWFactor f;
        f.kind = 1;
        f.cluster = cluster;
        f.c = nrows;
        f.k = k;
        f.cols_off = static_cast<long long>(out_.qidx.size());
        out_.qidx.insert(out_.qidx.end(), rows, rows + nrows);
        f.coupled_off = static_cast<long long>(out_.qidx.size());
        if (alloc) {
            f.a = out_.qarena->alloc_n<double>(std::max<size_t>(static_cast<size_t>(nrows) * k, 1));
            f.tau = out_.qarena->alloc_n<double>(std::max(k, 1));
            f.sign = out_.qarena->alloc_n<double>(std::max(k, 1));
        }
        out_.Q.push_back(f);
        return out_.Q.back();
    }
    // subtree-split accounting (opt.ranks > 1)
    bool ranked() const { return out_.rank.ranks > 1; }
    int own(int c) const { return out_.rank.owner[c]; }
    void rank_flops(int c, double f) {
        auto& v = out_.rank.flops;
        const size_t s = out_.stages.size();
        if (v.size() <= s) v.resize(s + 1, std::vector<double>(out_.rank.ranks, 0.0));
        v[s][own(c)] += f;
    }
    void rank_cross(int phase, double bytes) {
        auto& v = out_.rank.cross;
        const size_t s = out_.stages.size();
        if (v.size() <= s) v.resize(s + 1, std::vector<double>(4, 0.0));
        v[s][phase] += bytes;
    }
};

// factorize.cpp:32-82 — finest fronts, rows ascending into owners, one block
// per (owner(row), finest(col)) pair seen in A, values scattered on device.
void Engine::init_fronts(const std::vector<int>& owner) {
    ProfScope ps_(prof_, HostProf::INIT);
    const int Lf = L_ + 1;
    for (size_t c = 0; c < h_.clusters.size(); ++c)
        if (h_.clusters[c].level == Lf) {
            cols_[c] = h_.clusters[c].cols;
            fr_[c].live = true;
            alive_[c] = 1;
        }
    std::vector<int> local(A_.m);
    {  // rows (ascending) and a key-count bound per front, counted first so every list grows once
        std::vector<int> nr(fr_.size(), 0);
        std::vector<long long> nk(fr_.size(), 0);
        for (Index r = 0; r < A_.m; ++r) ++nr[owner[r]];
        for (Index k = 0; k < A_.nnz(); ++k) ++nk[owner[A_.i[k]]];
#pragma omp parallel for schedule(dynamic, 1024)
        for (long long c = 0; c < static_cast<long long>(fr_.size()); ++c) {
            if (nr[c]) fr_[c].rows.reserve(nr[c]);
            if (nk[c]) fr_[c].keys.reserve(std::min<long long>(nk[c], 64));
        }
    }
    for (Index r = 0; r < A_.m; ++r) {
        Front& f = fr_[owner[r]];
        local[r] = f.nrows();
        f.rows.push_back(r);
    }
    std::vector<int> colpos(A_.n);
    for (size_t c = 0; c < h_.clusters.size(); ++c)
        if (h_.clusters[c].level == Lf)
            for (size_t i = 0; i < h_.clusters[c].cols.size(); ++i) colpos[h_.clusters[c].cols[i]] = static_cast<int>(i);
    // key sets
    for (Index j = 0; j < A_.n; ++j) {
        const int q = h_.finest_of_col[j];
        for (Index k = A_.p[j]; k < A_.p[j + 1]; ++k) {
            Front& f = fr_[owner[A_.i[k]]];
            if (f.keys.empty() || f.keys.back().key != q) {  // cheap dedupe; full dedupe below
                f.keys.push_back(KeyRef{q, width(q), 0});
            }
        }
    }
#pragma omp parallel for schedule(dynamic, 256)
    for (long long c = 0; c < static_cast<long long>(fr_.size()); ++c) {
        Front& f = fr_[c];
        if (!f.live) continue;
        std::sort(f.keys.begin(), f.keys.end(), [](const KeyRef& a, const KeyRef& b) { return a.key < b.key; });
        f.keys.erase(std::unique(f.keys.begin(), f.keys.end(), [](const KeyRef& a, const KeyRef& b) { return a.key == b.key; }),
                     f.keys.end());
        layout(static_cast<int>(c), f.keys, f.ncols);
        f.ld = std::max(1, f.nrows());
    }
    size_t total = 0;
    for (size_t c = 0; c < fr_.size(); ++c) {
        Front& f = fr_[c];
        if (!f.live) continue;
        for (auto& k : f.keys) holders_[k.key].add(static_cast<int>(c));
        total += static_cast<size_t>(f.ld) * f.ncols;
    }
    // one zeroed slab for all initial fronts + scatter of A's values
    double* slab = arena().alloc_n<double>(std::max<size_t>(total, 1));
    CK(cudaMemsetAsync(slab, 0, sizeof(double) * std::max<size_t>(total, 1), st_));
    size_t o = 0;
    for (size_t c = 0; c < fr_.size(); ++c) {
        Front& f = fr_[c];
        if (!f.live) continue;
        f.mat = slab + o;
        o += static_cast<size_t>(f.ld) * f.ncols;
    }
    // scatter: per nnz destination offset (host-computed), values from A
    std::vector<long long> dsto(A_.nnz());
#pragma omp parallel for schedule(dynamic, 1024)
    for (Index j = 0; j < A_.n; ++j) {
        const int q = h_.finest_of_col[j];
        for (Index k = A_.p[j]; k < A_.p[j + 1]; ++k) {
            const int r = A_.i[k];
            const Front& f = fr_[owner[r]];
            const int qi = f.find(q);
            dsto[k] = (f.mat - slab) + local[r] + static_cast<long long>(f.keys[qi].col + colpos[j]) * f.ld;
        }
    }
    Uploader u = up();
    const long long* d_off = u.put(dsto);
    const double* d_val = u.put(A_.x);
    out_.ctr.h2d_bytes += u.bytes_h2d;
    cudaEvent_t e0 = kt_.begin(st_);
    launch_scatter_values(d_off, d_val, A_.nnz(), slab, st_);
    kt_.end(K_SCATTER, e0, st_, 24.0 * A_.nnz());
    out_.ctr.launches++;
}

int Engine::ancestor_target(int c) const {  // factorize.cpp:98-107
    int node = h_.tree->nodes[h_.clusters[c].tree_node].parent;
    while (node != -1) {
        for (int id : tree_clusters_[node])  // ascending ids; live front, not eliminated
            if (fr_[id].live && !gone_[id]) return id;
        node = h_.tree->nodes[node].parent;
    }
    return -1;
}

void Engine::rowval(const PRow& r, int key, double& sq, bool& nz, bool post_ok) const {
    if (r.sidx >= 0) {
        const Elim& e = el_[r.sidx];
        auto it = std::lower_bound(e.keys.begin() + 1, e.keys.end(), key);
        if (it != e.keys.end() && *it == key) {
            if (!post_ok || e.post_off < 0 || r.srow < e.cs || r.srow >= e.nsel_c)
                throw std::logic_error("spaqr engine: a row stacked twice within one stage (invariant violated)");
            const int ki = static_cast<int>(it - e.keys.begin());
            // post layout per elim: [blockmax all][blockmax key 1..nk][key 1..nk x own non-pivot rows]
            const long long nk = static_cast<long long>(e.keys.size()) - 1;
            const long long nown = e.nsel_c - e.cs;
            const long long o = e.post_off + 1 + nk + static_cast<long long>(ki - 1) * nown + (r.srow - e.cs);
            sq = post_sq_[o];
            nz = post_nz_[o];
            return;
        }
    }
    const Front& b = fr_[r.base];
    const int qi = b.find(key);
    if (qi < 0) {
        sq = 0.0;
        nz = false;
        return;
    }
    const long long o = b.soff[qi] + r.brow;
    sq = pre_sq_[o];
    nz = pre_nz_[o];
}

// factorize.cpp:176-271 (selection, keyset, stack layout) and :286-418's
// structural half (pivots, scatter bookkeeping) — values come later.  Runs in
// parallel over eliminations that share no participant front; effects on
// shared state (holders, npiv) are deferred to the caller.
void Engine::elim_pass1(Elim& e, Scratch& S) {
    const int c = e.c;
    const int cs = e.cs;
    const double eps = opt_.eps;
    const size_t np = e.parts.size();
    S.rv_off.assign(np + 1, 0);
    for (size_t pi = 0; pi < np; ++pi) S.rv_off[pi + 1] = S.rv_off[pi] + pend_[pend_id_[e.parts[pi]]].rows.size();
    S.rv_sq.resize(S.rv_off[np]);
    S.rv_nz.resize(S.rv_off[np]);
    double mx = 0.0;
    for (size_t pi = 0; pi < np; ++pi) {
        const PFront& P = pend_[pend_id_[e.parts[pi]]];
        row_vals(P, e.parts[pi], c, S.rv_sq.data() + S.rv_off[pi], S.rv_nz.data() + S.rv_off[pi], false);
        for (size_t q = S.rv_off[pi]; q < S.rv_off[pi + 1]; ++q) mx = std::max(mx, S.rv_sq[q]);
    }
    const double tau2 = eps > 0.0 ? mx * eps * eps * 1e-4 : 0.0;
    e.cmax2 = mx;
    if (S.sel.size() < np) S.sel.resize(np);
    auto& sel = S.sel;
    int total = 0;
    auto select = [&](double floor2) {
        total = 0;
        for (size_t pi = 0; pi < np; ++pi) {
            sel[pi].clear();
            const size_t o = S.rv_off[pi], n = S.rv_off[pi + 1] - o;
            for (size_t q = 0; q < n; ++q)
                if (floor2 > 0.0 ? S.rv_sq[o + q] > floor2 : S.rv_nz[o + q]) sel[pi].push_back(static_cast<int>(q));
            total += static_cast<int>(sel[pi].size());
        }
    };
    select(tau2);
    if (total < cs && tau2 > 0.0) select(0.0);
    if (total < cs) {
        e.err = "only " + std::to_string(total) + " rows couple " + std::to_string(cs) + " columns";
        e.cs = -1;  // marks the failing elimination
        return;
    }
    auto& keyset = S.keyset;
    keyset.clear();
    for (size_t pi = 0; pi < np; ++pi) {
        if (sel[pi].empty()) continue;
        const PFront& P = pend_[pend_id_[e.parts[pi]]];
        for (const KW& kw : P.keys) {
            const int key = kw.key;
            if (key == c || width(key) == 0 || std::binary_search(keyset.begin(), keyset.end(), key)) continue;
            for (int q : sel[pi]) {
                double sq;
                bool nz;
                rowval(P.rows[q], key, sq, nz, false);
                if (tau2 > 0.0 ? sq > tau2 : nz) {
                    sorted_insert(keyset, key);
                    break;
                }
            }
        }
    }
    e.keys.assign(1, c);
    e.keys.insert(e.keys.end(), keyset.begin(), keyset.end());
    e.off.assign(e.keys.size() + 1, 0);
    for (size_t i = 0; i < e.keys.size(); ++i) e.off[i + 1] = e.off[i] + width(e.keys[i]);
    e.tcols = e.off.back();
    e.total_rows = total;
    e.srows.clear();
    for (size_t pi = 0; pi < np; ++pi)
        for (int q : sel[pi]) e.srows.push_back(pend_[pend_id_[e.parts[pi]]].rows[q]);
    e.nsel_c = (np > 0 && e.parts[0] == c) ? static_cast<int>(sel[0].size()) : 0;
    for (const PRow& r : e.srows)
        if (r.sidx >= 0) throw std::logic_error("spaqr engine: row selected by two eliminations of one stage");
    // :332-344 pivots (disjoint columns per elimination)
    for (int pos = 0; pos < cs; ++pos) out_.pivot_row[cols_[c][pos]] = e.srows[pos].gid;
    // :346-418 scatter bookkeeping (participants are exclusive within a colour)
    const int eidx = static_cast<int>(&e - el_.data());
    int roff = 0;
    for (size_t pi = 0; pi < np; ++pi) {
        const int m = e.parts[pi];
        PFront& P = pend_[pend_id_[m]];
        const auto& s = sel[pi];
        if (s.empty()) {
            P.erase(c);
            continue;
        }
        if (roff >= cs) {
            for (size_t i = 0; i < s.size(); ++i) {
                P.rows[s[i]].sidx = eidx;
                P.rows[s[i]].srow = roff + static_cast<int>(i);
            }
        } else {
            auto& spos = S.spos;
            spos.assign(P.rows.size(), -1);
            for (size_t i = 0; i < s.size(); ++i) spos[s[i]] = roff + static_cast<int>(i);
            auto& nr = S.rows;
            nr.clear();
            for (size_t q = 0; q < P.rows.size(); ++q) {
                if (spos[q] >= 0 && spos[q] < cs) continue;
                PRow r = P.rows[q];
                if (spos[q] >= 0) {
                    r.sidx = eidx;
                    r.srow = spos[q];
                }
                nr.push_back(r);
            }
            P.rows.swap(nr);
        }
        for (int key : keyset) {
            P.add(key, width(key));
            e.hadd.emplace_back(key, m);
        }
        P.erase(c);
        fr_[m].scaled_ok = false;
        roff += static_cast<int>(s.size());
    }
}

// :286-323 coupling pruning and :138-174 move_extras decisions (parallel,
// read-only on shared state).
void Engine::elim_prep2(Elim& e, Scratch& S) {
    const int c = e.c;
    const int cs = e.cs;
    if (cs > 0) {
        const long long nk = static_cast<long long>(e.keys.size()) - 1;
        double floor_ = 0.0;
        if (opt_.eps > 0.0 && e.tcols > cs) floor_ = post_sq_[e.post_off] * opt_.eps * 1e-2;
        for (long long ki = 1; ki <= nk; ++ki) {
            const double mx = post_sq_[e.post_off + ki];
            const bool nz = post_nz_[e.post_off + ki];
            if (floor_ > 0.0 ? mx > floor_ : nz) {
                e.keepk.push_back(static_cast<int>(ki));
                e.kept += width(e.keys[ki]);
                e.coupled.insert(e.coupled.end(), cols_[e.keys[ki]].begin(), cols_[e.keys[ki]].end());
            }
        }
    }
    const PFront& fc = pend_[pend_id_[c]];
    if (fc.rows.empty()) return;
    auto& cand = S.cand;
    cand.clear();
    for (int m : e.parts)
        if (m != c && !gone_[m] && fr_[m].live && width(m) > 0 && fc.find(m) >= 0) cand.push_back(m);
    const size_t nr = fc.rows.size();
    S.bw.assign(nr, -1.0);
    S.best.assign(nr, -1);
    S.rv_sq.resize(nr);
    S.rv_nz.resize(nr);
    // roundoff rule shared with the oracle (spqr.h kMoveNoise2): candidate norms at the noise
    // floor of the elimination count as exact zeros
    const double noise2 = kMoveNoise2 * e.cmax2;
    for (int m : cand) {  // strict > in candidate order == the reference's per-row loop
        row_vals(fc, c, m, S.rv_sq.data(), S.rv_nz.data(), true);
        for (size_t q = 0; q < nr; ++q) {
            const double w = S.rv_sq[q] <= noise2 ? 0.0 : S.rv_sq[q];
            if (w > S.bw[q]) {
                S.bw[q] = w;
                S.best[q] = m;
            }
        }
    }
    int anc = -2;
    for (size_t q = 0; q < nr; ++q) {
        int b = S.best[q];
        if (b < 0) {
            if (anc == -2) anc = ancestor_target(c);
            b = anc;
        }
        if (b < 0)
            e.trail.push_back(static_cast<int>(q));
        else
            e.dest.emplace_back(b, static_cast<int>(q));
    }
    std::stable_sort(e.dest.begin(), e.dest.end(), [](const auto& x, const auto& y) { return x.first < y.first; });
}

// W factor + appends, in ascending cluster order (sequential).
void Engine::elim_commit2(Elim& e) {
    const int c = e.c;
    const int cs = e.cs;
    if (cs > 0) {
        const int kept = e.kept;
        DevWFactor& f = new_factor(0, c, cs, kept, cols_[c], &e.coupled);
        f.a = out_.warena->alloc_n<double>(static_cast<size_t>(cs) * (cs + kept));
        const int di = hp_->wcopy.begin(f.a, cs, cs, cs + kept, 1, 1 + static_cast<int>(e.keepk.size()));
        hp_->wcopy.source(di, 0) = AsmSrc{e.S, 1, e.total_rows};
        for (int i = 0; i < cs; ++i) hp_->wcopy.row(di, i) = int4{-1, 0, 0, i};
        hp_->wcopy.seg(di, 0, 0);
        hp_->wcopy.km(di, 0, 0) = 0;
        int o = cs;
        for (size_t q = 0; q < e.keepk.size(); ++q) {
            hp_->wcopy.seg(di, static_cast<int>(q) + 1, o);
            hp_->wcopy.km(di, static_cast<int>(q) + 1, 0) = e.off[e.keepk[q]];
            o += width(e.keys[e.keepk[q]]);
        }
    }
    PFront& fc = pend_[pend_id_[c]];
    for (int q : e.trail) out_.trailing_rows.push_back(fc.rows[q].gid);
    for (size_t a = 0; a < e.dest.size();) {  // append_rows, factorize.cpp:112-133 (ascending targets)
        size_t b = a;
        while (b < e.dest.size() && e.dest[b].first == e.dest[a].first) ++b;
        const int tgt = e.dest[a].first;
        PFront& T = pend(tgt);
        for (const KW& kw : fc.keys) {
            if (width(kw.key) == 0 || T.find(kw.key) >= 0) continue;
            T.add(kw.key, width(kw.key));
            holders_[kw.key].add(tgt);
        }
        // sequential order appends in ascending c: keep groups sorted by their source cluster
        auto pos = std::upper_bound(T.rows.begin(), T.rows.end(), c, [](int cc, const PRow& r) { return cc < r.tag; });
        const size_t at = static_cast<size_t>(pos - T.rows.begin());
        T.rows.insert(pos, b - a, PRow{});
        for (size_t t = a; t < b; ++t) {
            PRow r = fc.rows[e.dest[t].second];
            r.tag = c;
            T.rows[at + (t - a)] = r;
        }
        fr_[tgt].scaled_ok = false;
        a = b;
    }
    for (const KW& kw : fc.keys) hrem_.emplace_back(kw.key, c);  // removed in one pass per key after the wave
    gone_[c] = 1;
    fr_[c].live = false;
    alive_[c] = 0;
}

// the commits of one wave only add holders, so the eliminated clusters' removals
// are batched: each touched set is normalised once and filtered in one pass
void Engine::flush_holder_removals() {
    if (hrem_.empty()) return;
    std::sort(hrem_.begin(), hrem_.end());
    std::vector<size_t> gs;
    for (size_t i = 0; i < hrem_.size(); ++i)
        if (i == 0 || hrem_[i].first != hrem_[i - 1].first) gs.push_back(i);
    gs.push_back(hrem_.size());
    const long long ng = static_cast<long long>(gs.size()) - 1;
#pragma omp parallel for schedule(dynamic, 64) if (ng > 256)
    for (long long g = 0; g < ng; ++g) {
        HolderSet& h = holders_[hrem_[gs[g]].first];
        h.norm();
        size_t w = 0, q = gs[g];
        const size_t qe = gs[g + 1];
        for (size_t i = 0; i < h.v.size(); ++i) {
            while (q < qe && hrem_[q].second < h.v[i]) ++q;
            if (q < qe && hrem_[q].second == h.v[i]) continue;
            h.v[w++] = h.v[i];
        }
        h.v.resize(w);
    }
    hrem_.clear();
}

// Materialise every pending (touched, still live) front with one gather.
void Engine::materialize_pending() {
    ProfScope ps_(prof_, HostProf::MATER);
    std::unique_ptr<NScope> mt1 = std::make_unique<NScope>(nprof_, "mat.descriptors");
    AsmBuilder& b = hp_->wcopy;  // W copies already queued; fronts go in the same launch
    // plans persist across calls: a plan's new front is swapped into fr_, so the
    // superseded front's vectors come back here and are reused next time (no
    // malloc / free per front and wave)
    using Plan = MatPlan;
    const size_t nplan = pend_list_.size();
    if (mplans_.size() < nplan) mplans_.resize(nplan);
    std::vector<Plan>& plans = mplans_;
    // phase A (parallel): new row / key lists, layout, sources
#pragma omp parallel for schedule(dynamic, 32)
    for (long long t = 0; t < static_cast<long long>(nplan); ++t) {
        const int f = pend_list_[t];
        Plan& pl = plans[t];
        pl.f = -1;
        pl.same = false;
        pl.di = -1;
        pl.bases.clear();
        pl.stacks.clear();
        pl.ord.clear();
        if (!fr_[f].live) continue;
        pl.f = f;
        const PFront& P = pend_[pend_id_[f]];
        Front& nf = pl.nf;
        nf.mat = nullptr;
        nf.big = false;
        nf.soff.clear();
        nf.tag.clear();
        nf.live = true;
        nf.scaled_ok = fr_[f].scaled_ok;
        nf.rows.resize(P.rows.size());
        bool tagged = false;
        for (size_t i = 0; i < P.rows.size(); ++i) {
            nf.rows[i] = P.rows[i].gid;
            tagged |= P.rows[i].tag >= 0;
        }
        if (tagged) {
            nf.tag.resize(P.rows.size());
            for (size_t i = 0; i < P.rows.size(); ++i) nf.tag[i] = P.rows[i].tag;
        }
        nf.keys.resize(P.keys.size());
        for (size_t i = 0; i < P.keys.size(); ++i) nf.keys[i] = KeyRef{P.keys[i].key, P.keys[i].width, 0};
        layout(f, nf.keys, nf.ncols);
        nf.ld = std::max(1, nf.nrows());
        bool same = nf.keys.size() == fr_[f].keys.size() && P.rows.size() == fr_[f].rows.size();
        for (size_t i = 0; same && i < nf.keys.size(); ++i)
            same = nf.keys[i].key == fr_[f].keys[i].key && nf.keys[i].width == fr_[f].keys[i].width;
        for (size_t i = 0; same && i < P.rows.size(); ++i)
            same = P.rows[i].base == f && P.rows[i].brow == static_cast<int>(i) && P.rows[i].sidx < 0;
        pl.same = same;
        if (same) continue;
        for (const PRow& r : P.rows) {
            if (std::find(pl.bases.begin(), pl.bases.end(), r.base) == pl.bases.end()) pl.bases.push_back(r.base);
            if (r.sidx >= 0 && std::find(pl.stacks.begin(), pl.stacks.end(), r.sidx) == pl.stacks.end())
                pl.stacks.push_back(r.sidx);
        }
        phys_order(nf.keys, pl.ord);
    }
    // phase B (sequential): allocation and descriptor reservation
    for (size_t t = 0; t < nplan; ++t) {
        Plan& pl = plans[t];
        if (pl.f < 0 || pl.same) continue;
        Front& nf = pl.nf;
        nf.mat = dalloc(arena(), static_cast<size_t>(nf.ld) * std::max(nf.ncols, 1), nf.big);
        if (!sprof_.empty()) {
            auto& sp = sprof_.back();
            sp.mat_fronts++;
            sp.mat_rows += nf.nrows();
            sp.mat_elems += static_cast<long long>(nf.nrows()) * nf.ncols;
            sp.max_front_rows = std::max<long long>(sp.max_front_rows, nf.nrows());
            sp.max_front_cols = std::max<long long>(sp.max_front_cols, nf.ncols);
        }
        if (nf.nrows() == 0 || nf.ncols == 0) continue;
        const int nsrc = static_cast<int>(pl.bases.size() + pl.stacks.size());
        // every row map entry is written in phase C (one per pending row)
        pl.di = b.begin(nf.mat, nf.ld, nf.nrows(), nf.ncols, std::max(nsrc, 1), static_cast<int>(pl.ord.size()), false);
    }
    // phase C (parallel): fill
#pragma omp parallel for schedule(dynamic, 32)
    for (long long t = 0; t < static_cast<long long>(nplan); ++t) {
        Plan& pl = plans[t];
        if (pl.di < 0) continue;
        const int di = pl.di;
        const PFront& P = pend_[pend_id_[pl.f]];
        const Front& nf = pl.nf;
        const int nb = static_cast<int>(pl.bases.size());
        for (int s = 0; s < nb; ++s) {
            const Front& B = fr_[pl.bases[s]];
            b.source(di, s) = AsmSrc{B.mat, 1, B.ld};
        }
        for (size_t s = 0; s < pl.stacks.size(); ++s) {
            const Elim& E = el_[pl.stacks[s]];
            b.source(di, nb + static_cast<int>(s)) = AsmSrc{E.S, 1, E.total_rows};
        }
        int lastb = -1, lastslot = 0;
        for (size_t i = 0; i < P.rows.size(); ++i) {
            const PRow& r = P.rows[i];
            if (r.base != lastb) {
                lastb = r.base;
                lastslot = static_cast<int>(std::find(pl.bases.begin(), pl.bases.end(), r.base) - pl.bases.begin());
            }
            int s1 = -1;
            if (r.sidx >= 0)
                s1 = nb + static_cast<int>(std::find(pl.stacks.begin(), pl.stacks.end(), r.sidx) - pl.stacks.begin());
            b.row(di, static_cast<int>(i)) = int4{s1, r.srow, lastslot, r.brow};
        }
        for (size_t q = 0; q < pl.ord.size(); ++q) {
            const KeyRef& k = nf.keys[pl.ord[q]];
            b.seg(di, static_cast<int>(q), k.col);
            for (int s = 0; s < nb; ++s) {
                const Front& B = fr_[pl.bases[s]];
                const int qi = B.find(k.key);
                if (qi >= 0) b.km(di, static_cast<int>(q), s) = B.keys[qi].col;
            }
            for (size_t s = 0; s < pl.stacks.size(); ++s) {
                const Elim& E = el_[pl.stacks[s]];
                auto it = std::lower_bound(E.keys.begin() + 1, E.keys.end(), k.key);
                if (it == E.keys.end() || *it != k.key) continue;
                b.km(di, static_cast<int>(q), nb + static_cast<int>(s)) = E.off[it - E.keys.begin()];
            }
        }
    }
    mt1.reset();
    std::unique_ptr<NScope> mt2 = std::make_unique<NScope>(nprof_, "mat.flush");
    flush_assemble(b);
    mt2.reset();
    NScope mt3(nprof_, "mat.swap");
    for (size_t t = 0; t < nplan; ++t) {
        Plan& pl = plans[t];
        if (pl.f >= 0 && !pl.same) dfree(fr_[pl.f].mat, fr_[pl.f].big);  // the gather reading it is already enqueued
    }
#pragma omp parallel for schedule(dynamic, 64) if (nplan > 256)
    for (long long t = 0; t < static_cast<long long>(nplan); ++t) {
        Plan& pl = plans[t];
        if (pl.f >= 0 && !pl.same) std::swap(fr_[pl.f], pl.nf);  // old front's storage is recycled
    }
    // eliminated fronts and this wave's stacks are no longer referenced
    for (int f : pend_list_)
        if (!fr_[f].live && fr_[f].big) {
            dfree(fr_[f].mat, true);
            fr_[f].mat = nullptr;
            fr_[f].big = false;
        }
    for (size_t t = 0; t < el_.size(); ++t)
        if (el_[t].sbig) {
            dfree(el_[t].S, true);
            el_[t].S = nullptr;
            el_[t].sbig = false;
        }
    for (int f : pend_list_) pend_id_[f] = -1;
    pend_list_.clear();
    npend_ = 0;
}

// pre-stage row statistics (sum of squares, any-nonzero) of every block of the fronts in P
void Engine::compute_stats(const std::vector<int>& P) {
    ProfScope ps_(prof_, HostProf::STATS);
    // two-phase (count, parallel fill) descriptor build
    const size_t nP = P.size();
    std::vector<long long> dcount(nP + 1, 0), wcount(nP + 1, 0);
    for (size_t t = 0; t < nP; ++t) {
        const Front& F = fr_[P[t]];
        const int nk = F.nrows() > 0 ? static_cast<int>(F.keys.size()) : 0;
        dcount[t + 1] = dcount[t] + nk;
        wcount[t + 1] = wcount[t] + static_cast<long long>(nk) * F.nrows();
    }
    const long long work = wcount[nP];
    dl_vector<StatDesc> sd(dcount[nP]);  // every entry is written by the fill below
#pragma omp parallel for schedule(dynamic, 256)
    for (long long t = 0; t < static_cast<long long>(nP); ++t) {
        Front& F = fr_[P[t]];
        F.soff.assign(F.keys.size(), -1);
        long long w = wcount[t];
        long long dd = dcount[t];
        for (size_t qi = 0; qi < F.keys.size(); ++qi) {
            F.soff[qi] = w;
            if (F.nrows() == 0) continue;
            sd[dd++] = StatDesc{F.mat, F.ld, 0, F.nrows(), F.keys[qi].col, F.keys[qi].width, 0, w, w};
            w += F.nrows();
        }
    }
    double* d_sq = arena().alloc_n<double>(std::max<long long>(work, 1));
    unsigned char* d_nz = arena().alloc_n<unsigned char>(std::max<long long>(work, 1));
    if (!sd.empty()) {
        Uploader u = up();
        const StatDesc* dd = u.put(sd.data(), sd.size());
        out_.ctr.h2d_bytes += u.bytes_h2d;
        double sb = 0;
        for (auto& q : sd) sb += 8.0 * q.nrows * q.ncols + 9.0 * q.nrows;
        cudaEvent_t e0 = kt_.begin(st_);
        launch_stats(dd, static_cast<int>(sd.size()), work, d_sq, d_nz, st_);
        kt_.end(K_STATS, e0, st_, sb);
        out_.ctr.launches++;
    }
    enqueue(pre_sq_, d_sq, work);
    enqueue(pre_nz_, d_nz, work);
    fetch();
}

std::vector<int> Engine::stage_fronts(const std::vector<int>& list) {
    std::vector<int> P;
    for (int c : list) {
        if (fr_[c].live && !mark_[c]) {
            mark_[c] = 1;
            P.push_back(c);
        }
        if (width(c) > 0)
            for (int m : holders_[c].get())
                if (fr_[m].live && !mark_[m]) {
                    mark_[m] = 1;
                    P.push_back(m);
                }
    }
    for (int f : P) mark_[f] = 0;
    return P;
}

// Eliminations of one stage touch disjoint rows in exact mode, but once
// scale_all has mixed a shared front's rows, two clusters of the same stage
// can couple to the same row: the later one must see the earlier one's
// transformed values (the reference runs them in ascending id order).  The
// stage is split into dependency waves (edge c1 -> c2, c1 < c2, when some row
// is nonzero in both blocks); each wave is one batched round.
void Engine::eliminate_stage(int k) {
    std::vector<int> mine;
    if (dist_stage(k)) {  // a split stage: this rank's subtree only (ranks.cpp owners)
        for (int c : stage_list_[k])
            if (dist_mine(c)) mine.push_back(c);
    }
    const auto& list = dist_stage(k) ? mine : stage_list_[k];
    if (list.empty()) return;
    for (size_t f = 0; f < fr_.size(); ++f)
        if (alive_[f]) fr_[f].tag.clear();
    std::vector<int> P = stage_fronts(list);
    compute_stats(P);
    std::vector<int> lvl(fr_.size(), -1);
    for (int c : list) lvl[c] = 0;
    {
        ProfScope ps(prof_, HostProf::DEPS);
        std::vector<int> last;
        for (int f : P) {
            const Front& F = fr_[f];
            last.assign(F.nrows(), -1);
            for (size_t qi = 0; qi < F.keys.size(); ++qi) {  // ascending keys
                const int c = F.keys[qi].key;
                if (lvl[c] < 0 || stage_of_[c] != k) continue;
                for (int r = 0; r < F.nrows(); ++r)
                    if (pre_nz_[F.soff[qi] + r]) {
                        if (last[r] >= 0) dep_.emplace_back(last[r], c);
                        last[r] = c;
                    }
            }
        }
        std::sort(dep_.begin(), dep_.end(), [](const auto& a, const auto& b) { return a.second < b.second; });
        size_t q = 0;
        for (int c : list) {  // ascending: every edge points to a larger id
            for (; q < dep_.size() && dep_[q].second == c; ++q) lvl[c] = std::max(lvl[c], lvl[dep_[q].first] + 1);
        }
        dep_.clear();
    }
    int nw = 0;
    for (int c : list) nw = std::max(nw, lvl[c] + 1);
    std::vector<std::vector<int>> waves(nw);
    for (int c : list) waves[lvl[c]].push_back(c);
    out_.ctr.elim_waves += nw;
    waves_per_stage_.push_back(nw);
    sprof_.back().waves = nw;
    const size_t w0 = out_.W.size(), q0 = out_.Q.size();
    for (int w = 0; w < nw; ++w) {
        if (w > 0) compute_stats(stage_fronts(waves[w]));
        batch_ = out_.nbatches++;  // a wave's factors touch independent column sets
        eliminate_wave(waves[w]);
        notify("eliminate", waves[w].front(), &waves[w]);
    }
    // W in the reference's chronological order (ascending cluster); the solve
    // plan regroups by batch, which only reorders independent factors
    std::stable_sort(out_.W.begin() + w0, out_.W.end(),
                     [](const DevWFactor& a, const DevWFactor& b) { return a.cluster < b.cluster; });
    std::stable_sort(out_.Q.begin() + q0, out_.Q.end(),
                     [](const DevWFactor& a, const DevWFactor& b) { return a.cluster < b.cluster; });
}

void Engine::eliminate_wave(const std::vector<int>& list) {
    const size_t n = list.size();
    if (el_.size() < n) el_.resize(n);  // pool: Elim objects keep their capacity
    int nth = 1;
#ifdef _OPENMP
    nth = omp_get_max_threads();
#endif
    if (static_cast<int>(tscr_.size()) < nth) tscr_.resize(nth);
    // prepass (sequential): participants, pending fronts, conflict colouring
    // (eliminations of one colour share no participant front)
    std::vector<std::vector<int>> colour_lists;
    {
        ProfScope ps(prof_, HostProf::PASS1);
        for (size_t t = 0; t < n; ++t) {
            const int c = list[t];
            Elim& e = el_[t];
            e.reset(c, width(c));
            pend(c);
            if (e.cs <= 0) continue;
            for (int m : holders_[c].get())
                if (m != c) e.parts.push_back(m);
            if (pend(c).find(c) >= 0) e.parts.insert(e.parts.begin(), c);
            for (int m : e.parts) pend(m);
            uint64_t used = 0;
            for (int m : e.parts) used |= colmask_[m];
            int col = 0;
            while (col < 63 && ((used >> col) & 1)) ++col;
            e.color = col;  // colour 63 collects overflow; it is run sequentially
            for (int m : e.parts) colmask_[m] |= (uint64_t(1) << col);
            if (static_cast<int>(colour_lists.size()) <= col) colour_lists.resize(col + 1);
            colour_lists[col].push_back(static_cast<int>(t));
        }
        for (size_t t = 0; t < n; ++t)
            for (int m : el_[t].parts) colmask_[m] = 0;
        // pass 1, colour by colour
        for (size_t col = 0; col < colour_lists.size(); ++col) {
            const auto& cl = colour_lists[col];
            const bool par = col < 63 && cl.size() > 16;
#pragma omp parallel for schedule(dynamic, 8) if (par)
            for (long long q = 0; q < static_cast<long long>(cl.size()); ++q) {
                Elim& e = el_[cl[q]];
                if (e.cs <= 0) continue;
                int tid = 0;
#ifdef _OPENMP
                tid = omp_get_thread_num();
#endif
                try {
                    elim_pass1(e, tscr_[tid]);
                } catch (const std::exception& x) {
                    e.logic = true;
                    e.err = x.what();
                }
            }
        }
    }
    for (size_t t = 0; t < n; ++t)
        if (el_[t].logic) throw std::logic_error(el_[t].err);
    // the first failing elimination in ascending order stops the sequence
    int nvalid = 0;
    for (size_t t = 0; t < n; ++t) {
        if (el_[t].cs < 0) {
            record_error(el_[t].c, el_[t].err);
            break;
        }
        ++nvalid;
    }
    for (int t = 0; t < nvalid; ++t) {
        Elim& e = el_[t];
        for (auto& hk : e.hadd) holders_[hk.first].add(hk.second);
        if (e.cs > 0) {
            npiv_ += e.cs;
            holders_[e.c].clear();
        }
    }
    // gather stacks, QR + apply, post statistics
    ProfScope ps_sb(prof_, HostProf::SBUILD);
    std::unique_ptr<NScope> sb_desc = std::make_unique<NScope>(nprof_, "sb.descriptors");
    AsmBuilder& sb = asm_slot(0);  // keeps its capacity across calls
    std::vector<QrDesc> qd;
    std::vector<StatDesc> pd;
    std::vector<VCopyDesc> vq;  // store_q
    long long pwork = 0, postlen = 0;
    std::vector<int> flags_init;
    // stack descriptors in three phases: source fronts per elimination
    // (parallel), allocation + descriptor reservation (sequential, cheap),
    // row / segment maps (parallel, disjoint ranges of the builder)
    if (sb_bases_.size() < static_cast<size_t>(nvalid)) sb_bases_.resize(nvalid);
    std::vector<int> edi(nvalid, -1);
#pragma omp parallel for schedule(dynamic, 16) if (nvalid > 64)
    for (int ei = 0; ei < nvalid; ++ei) {
        std::vector<int>& bases = sb_bases_[ei];
        bases.clear();
        if (el_[ei].cs <= 0) continue;
        for (const PRow& r : el_[ei].srows)
            if (std::find(bases.begin(), bases.end(), r.base) == bases.end()) bases.push_back(r.base);
    }
    {
        size_t npd = 0;
        for (int ei = 0; ei < nvalid; ++ei)
            if (el_[ei].cs > 0) npd += 1 + 2 * el_[ei].keys.size();
        pd.reserve(npd);
        qd.reserve(nvalid);
        flags_init.reserve(nvalid);
    }
    for (int ei = 0; ei < nvalid; ++ei) {
        Elim& e = el_[ei];
        if (e.cs <= 0) continue;
        e.S = dalloc(arena(), static_cast<size_t>(e.total_rows) * e.tcols, e.sbig);
        if (!sprof_.empty()) {
            auto& sp = sprof_.back();
            sp.s_elems += static_cast<long long>(e.total_rows) * e.tcols;
            sp.s_max_rows = std::max<long long>(sp.s_max_rows, e.total_rows);
            sp.s_max_cols = std::max<long long>(sp.s_max_cols, e.tcols);
            sp.elims++;
        }
        const int nsrc = static_cast<int>(sb_bases_[ei].size());
        edi[ei] = sb.begin(e.S, e.total_rows, e.total_rows, e.tcols, nsrc, static_cast<int>(e.keys.size()), false);
        flags_init.push_back(INT_MAX);
        QrDesc q{e.S, e.total_rows, e.total_rows, e.cs, e.tcols, nullptr, nullptr, nullptr, nullptr, 0, 1};
        if (opt_.store_q) {  // factorize.cpp:324-330: H of the stack on its rows, parts order
            std::vector<int>& rws = qrows_scratch_;
            rws.resize(e.total_rows);
            for (int i = 0; i < e.total_rows; ++i) rws[i] = e.srows[i].gid;
            DevWFactor& qf = new_qfactor(e.c, rws.data(), e.total_rows, e.cs);
            q.tau = qf.tau;
            q.sign = qf.sign;
            q.zero_lower = 0;
            vq.push_back(VCopyDesc{e.S, e.total_rows, e.total_rows, e.cs, VCOPY_ZERO_LOWER, qf.a});
        }
        qd.push_back(q);
        out_.ctr.qr_flops += 2.0 * e.total_rows * double(e.cs) * e.cs - 2.0 / 3.0 * double(e.cs) * e.cs * e.cs +
                             (4.0 * e.total_rows * e.cs - 2.0 * e.cs * double(e.cs)) * (e.tcols - e.cs);
        out_.ctr.qr_bytes += 16.0 * e.total_rows * e.tcols;
        if (ranked()) {  // rows gathered from (and written back to) fronts of other ranks
            rank_flops(e.c, 2.0 * e.total_rows * double(e.cs) * e.cs - 2.0 / 3.0 * double(e.cs) * e.cs * e.cs +
                                (4.0 * e.total_rows * e.cs - 2.0 * e.cs * double(e.cs)) * (e.tcols - e.cs));
            long long remote = 0;
            for (int i = 0; i < e.total_rows; ++i) remote += own(e.srows[i].base) != own(e.c);
            rank_cross(0, 16.0 * remote * e.tcols);
        }
        // post stats: [max over all neighbour cols][max per key][own non-pivot rows x keys]
        const long long nk = static_cast<long long>(e.keys.size()) - 1;
        e.post_off = postlen;
        if (e.tcols > e.cs) {
            pd.push_back(StatDesc{e.S, e.total_rows, 0, e.cs, e.cs, e.tcols - e.cs, 1, postlen, pwork});
            pwork += 1;
        }
        postlen += 1;
        for (long long ki = 1; ki <= nk; ++ki) {
            pd.push_back(StatDesc{e.S, e.total_rows, 0, e.cs, e.off[ki], width(e.keys[ki]), 1, postlen, pwork});
            pwork += 1;
            postlen += 1;
        }
        const int nown = std::max(0, e.nsel_c - e.cs);
        if (nown > 0)
            for (long long ki = 1; ki <= nk; ++ki) {  // own non-pivot rows, one descriptor per key
                pd.push_back(StatDesc{e.S, e.total_rows, e.cs, nown, e.off[ki], width(e.keys[ki]), 0, postlen, pwork});
                pwork += nown;
                postlen += nown;
            }
    }
#pragma omp parallel for schedule(dynamic, 16) if (nvalid > 64)
    for (int ei = 0; ei < nvalid; ++ei) {
        const Elim& e = el_[ei];
        const int di = edi[ei];
        if (di < 0) continue;
        const std::vector<int>& bases = sb_bases_[ei];
        const int nsrc = static_cast<int>(bases.size());
        for (int s = 0; s < nsrc; ++s) sb.source(di, s) = AsmSrc{fr_[bases[s]].mat, 1, fr_[bases[s]].ld};
        for (int i = 0; i < e.total_rows; ++i) {
            const PRow& r = e.srows[i];
            const int s = static_cast<int>(std::find(bases.begin(), bases.end(), r.base) - bases.begin());
            sb.row(di, i) = int4{-1, 0, s, r.brow};
        }
        for (size_t ki = 0; ki < e.keys.size(); ++ki) {
            sb.seg(di, static_cast<int>(ki), e.off[ki]);
            for (int s = 0; s < nsrc; ++s) {
                const Front& B = fr_[bases[s]];
                const int qi = B.find(e.keys[ki]);
                if (qi >= 0) sb.km(di, static_cast<int>(ki), s) = B.keys[qi].col;
            }
        }
    }
    hp_->wcopy.clear();
    double *d_psq = nullptr;
    unsigned char* d_pnz = nullptr;
    if (!qd.empty()) {
        sb_desc.reset();
        NScope sx(nprof_, "sb.upload+launch+fetch");
        flush_assemble(sb);
        Uploader u = up();
        int* d_flags = u.put(flags_init);
        for (size_t i = 0, qi = 0; i < static_cast<size_t>(nvalid); ++i)
            if (el_[i].cs > 0) {
                el_[i].flag = d_flags + qi;
                qd[qi].flag = d_flags + qi;
                ++qi;
            }
        const QrDesc* dq = u.put(qd);
        d_psq = arena().alloc_n<double>(std::max<long long>(postlen, 1));
        d_pnz = arena().alloc_n<unsigned char>(std::max<long long>(postlen, 1));
        pwork = layout_stats(pd.data(), pd.size());
        const StatDesc* dp = u.put(pd);
        out_.ctr.h2d_bytes += u.bytes_h2d;
        int maxm = 0;
        for (auto& q : qd) maxm = std::max(maxm, q.m);
        run_qr(qd, dq, u);
        out_.ctr.launches++;
        out_.ctr.qr_launches++;
        if (!vq.empty()) launch_vcopy(u.put(vq), static_cast<int>(vq.size()), st_);
        double sb = 0;
        for (auto& q : pd) sb += 8.0 * q.nrows * q.ncols + 9.0;
        cudaEvent_t e0 = kt_.begin(st_);
        launch_stats(dp, static_cast<int>(pd.size()), pwork, d_psq, d_pnz, st_);
        kt_.end(K_STATS, e0, st_, sb);
        out_.ctr.launches++;
        std::vector<int> flags;
        enqueue(flags, d_flags, flags_init.size());
        enqueue(post_sq_, d_psq, postlen);
        enqueue(post_nz_, d_pnz, postlen);
        fetch();
        // first error in ascending order (singular pivot precedes a later "rows couple")
        for (size_t i = 0, qi = 0; i < static_cast<size_t>(nvalid); ++i)
            if (el_[i].cs > 0) {
                if (flags[qi] != INT_MAX) {
                    err_cluster_ = -1;
                    record_error(el_[i].c, "pivot " + std::to_string(flags[qi]) + " is zero or denormal");
                    break;
                }
                ++qi;
            }
    }
    raise_if_error();
    {
        ProfScope ps(prof_, HostProf::PASS2);
#pragma omp parallel for schedule(dynamic, 8) if (nvalid > 32)
        for (int t = 0; t < nvalid; ++t) {
            int tid = 0;
#ifdef _OPENMP
            tid = omp_get_thread_num();
#endif
            try {
                elim_prep2(el_[t], tscr_[tid]);
            } catch (const std::exception& x) {
                el_[t].logic = true;
                el_[t].err = x.what();
            }
        }
        for (int t = 0; t < nvalid; ++t)
            if (el_[t].logic) throw std::logic_error(el_[t].err);
        if (dist_stage(cur_stage_))  // split stage: what the other ranks must merge
            for (int t = 0; t < nvalid; ++t) {
                const Elim& e = el_[t];
                for (int m : e.parts) dist_touched_.push_back(m);
                for (const auto& d : e.dest) dist_touched_.push_back(d.first);
                for (int i = std::max(e.cs, 0); i < e.total_rows; ++i) dist_tr_.emplace_back(e.srows[i].base, e.srows[i].gid);
            }
        for (int t = 0; t < nvalid; ++t) elim_commit2(el_[t]);
        flush_holder_removals();
    }
    materialize_pending();
}

// factorize.cpp:425-486
void Engine::scale_all() {
    ProfScope ps_(prof_, HostProf::SCALE);
    std::vector<int> cand;
    std::vector<StatDesc> sd;
    for (size_t p = 0; p < fr_.size(); ++p) {
        if (!alive_[p]) continue;
        Front& f = fr_[p];
        if (!f.live) continue;
        f.scaled_ok = false;
        const int cs = width(static_cast<int>(p));
        if (cs == 0) continue;
        const int r = f.nrows();
        if (r < cs) continue;
        const int qi = f.find(static_cast<int>(p));
        if (qi < 0) {  // a zero diagonal block: QR of zeros fails at pivot 0
            record_error(static_cast<int>(p), "pivot 0 is zero or denormal");
            continue;
        }
        sd.push_back(StatDesc{f.mat, f.ld, 0, r, f.keys[qi].col, cs, 2, static_cast<long long>(cand.size()),
                              static_cast<long long>(cand.size())});
        cand.push_back(static_cast<int>(p));
    }
    if (cand.empty()) {
        raise_if_error();
        return;
    }
    double* d_sq = arena().alloc_n<double>(cand.size());
    unsigned char* d_nz = arena().alloc_n<unsigned char>(cand.size());
    {
        Uploader u = up();
        const long long swork = layout_stats(sd.data(), sd.size());
        const StatDesc* dd = u.put(sd);
        out_.ctr.h2d_bytes += u.bytes_h2d;
        double sb = 0;
        for (auto& q : sd) sb += 8.0 * q.nrows * q.ncols;
        cudaEvent_t e0 = kt_.begin(st_);
        launch_stats(dd, static_cast<int>(sd.size()), swork, d_sq, d_nz, st_);
        kt_.end(K_STATS, e0, st_, sb);
        out_.ctr.launches++;
    }
    std::vector<unsigned char> ident;
    download(ident, d_nz, cand.size());
    std::vector<QrDesc> qd;
    std::vector<TrsmDesc> td;
    std::vector<VCopyDesc> vq;  // store_q
    std::vector<int> qp;
    long long trows = 0;
    for (size_t i = 0; i < cand.size(); ++i) {
        const int p = cand[i];
        Front& f = fr_[p];
        if (ident[i]) {
            f.scaled_ok = true;
            continue;
        }
        const int cs = width(p);
        DevWFactor& w = new_factor(0, p, cs, 0, cols_[p], nullptr);
        w.a = out_.warena->alloc_n<double>(static_cast<size_t>(cs) * cs);
        qd.push_back(QrDesc{f.mat, f.ld, f.nrows(), cs, f.ncols, nullptr, nullptr, w.a, nullptr, 1, 0});
        if (opt_.store_q) {  // factorize.cpp:483: U on all of p's rows
            DevWFactor& qf = new_qfactor(p, f.rows.data(), f.nrows(), cs);
            qd.back().tau = qf.tau;
            qd.back().sign = qf.sign;
            qd.back().set_identity = 0;
            vq.push_back(VCopyDesc{f.mat, f.ld, f.nrows(), cs, VCOPY_SET_IDENTITY, qf.a});
        }
        qp.push_back(p);
        out_.ctr.qr_flops += 2.0 * f.nrows() * double(cs) * cs - 2.0 / 3.0 * double(cs) * cs * cs +
                             (4.0 * f.nrows() * cs - 2.0 * cs * double(cs)) * (f.ncols - cs);
        out_.ctr.qr_bytes += 16.0 * f.nrows() * f.ncols;
        if (ranked())
            rank_flops(p, 2.0 * f.nrows() * double(cs) * cs - 2.0 / 3.0 * double(cs) * cs * cs +
                              (4.0 * f.nrows() * cs - 2.0 * cs * double(cs)) * (f.ncols - cs));
        for (int m : holders_[p].get()) {
            if (m == p) continue;
            const Front& fm = fr_[m];
            const int mq = fm.find(p);
            if (fm.nrows() == 0) continue;
            td.push_back(TrsmDesc{fm.mat + static_cast<long long>(fm.keys[mq].col) * fm.ld, fm.ld, fm.nrows(), cs, w.a, cs, trows});
            if (ranked() && own(m) != own(p)) rank_cross(1, 8.0 * cs * cs);
            trows += fm.nrows();
        }
        f.scaled_ok = true;
    }
    if (!qd.empty()) {
        std::vector<int> flags_init(qd.size(), INT_MAX);
        Uploader u = up();
        int* d_flags = u.put(flags_init);
        for (size_t i = 0; i < qd.size(); ++i) qd[i].flag = d_flags + i;
        const QrDesc* dq = u.put(qd);
        const TrsmDesc* dt = u.put(td);
        out_.ctr.h2d_bytes += u.bytes_h2d;
        int maxm = 0;
        for (auto& q : qd) maxm = std::max(maxm, q.m);
        double tb = 0;
        for (auto& t : td) tb += 16.0 * t.nrows * t.n;
        run_qr(qd, dq, u);
        out_.ctr.launches++;
        out_.ctr.qr_launches++;
        if (!vq.empty()) launch_vcopy(u.put(vq), static_cast<int>(vq.size()), st_);
        cudaEvent_t e0 = kt_.begin(st_);
        launch_trsm(dt, static_cast<int>(td.size()), trows, st_);
        kt_.end(K_TRSM, e0, st_, tb);
        out_.ctr.launches++;
        std::vector<int> flags;
        download(flags, d_flags, flags_init.size());
        for (size_t i = 0; i < flags.size(); ++i)
            if (flags[i] != INT_MAX) {
                if (err_cluster_ < 0 || qp[i] < err_cluster_) {
                    err_cluster_ = qp[i];
                    err_reason_ = "pivot " + std::to_string(flags[i]) + " is zero or denormal";
                }
                break;
            }
    }
    raise_if_error();
}

// factorize.cpp:488-537 — CPQR of every front's extra rows against its neighbours.
void Engine::sparsify_rows_all() {
    ProfScope ps_(prof_, HostProf::SROWS);
    struct Job {
        int p, cs, p2, nw, c0;
        double* B;
        bool big;
    };
    std::vector<Job> jobs;
    AsmBuilder& gb = asm_slot(1);  // keeps its capacity across calls
    std::vector<CpqrDesc> cd;
    int maxm = 0;
    for (size_t pp = 0; pp < fr_.size(); ++pp) {
        const int p = static_cast<int>(pp);
        if (!alive_[p]) continue;
        Front& f = fr_[p];
        if (!f.live) continue;
        const int cs = width(p);
        if (cs > 0 && !f.scaled_ok) continue;
        const int r = f.nrows();
        const int p2 = r - cs;
        if (p2 <= 0) continue;
        const int qi = f.find(p);
        const int c0 = (qi >= 0) ? f.keys[qi].width : 0;
        int nw = 0, nseg = 0;
        for (const KeyRef& k : f.keys)
            if (k.key != p && k.width > 0) {
                nw += k.width;
                ++nseg;
            }
        if (nw == 0) {  // keep = 0: every extra row is dropped
            for (int i = cs; i < r; ++i) out_.dropped_rows.push_back(f.rows[i]);
            f.rows.resize(cs);
            continue;
        }
        bool bbig = false;
        Job j{p, cs, p2, nw, c0, dalloc(arena(), static_cast<size_t>(p2) * nw, bbig), bbig};
        // B = extra rows x live neighbour columns, ascending keys (physical order)
        const int di = gb.begin(j.B, p2, p2, nw, 1, nseg);
        gb.source(di, 0) = AsmSrc{f.mat + cs, 1, f.ld};
        for (int i = 0; i < p2; ++i) gb.row(di, i) = int4{-1, 0, 0, i};
        {
            std::vector<int> ord;
            phys_order(f.keys, ord);
            int sg = 0, bo = 0;
            for (int q : ord) {
                const KeyRef& k = f.keys[q];
                if (k.key == p || k.width == 0) continue;
                gb.seg(di, sg, bo);
                gb.km(di, sg, 0) = k.col;
                bo += k.width;
                ++sg;
            }
        }
        jobs.push_back(j);
        maxm = std::max(maxm, p2);
        out_.ctr.cpqr_bytes += 8.0 * p2 * nw;
    }
    if (jobs.empty()) return;
    flush_assemble(gb);
    const size_t nj = jobs.size();
    int* d_rank = arena().alloc_n<int>(nj);
    double* d_r11 = arena().alloc_n<double>(nj);
    std::vector<double*> qv(opt_.store_q ? nj * 3 : 0);  // store_q: T.H of every job (V, tau, sign)
    for (size_t i = 0; i < nj; ++i) {
        const Job& j = jobs[i];
        double* work = arena().alloc_n<double>(3 * static_cast<size_t>(j.nw));
        cd.push_back(CpqrDesc{j.B, j.p2, j.p2, j.nw, opt_.eps, d_rank + i, d_r11 + i, nullptr, 0, nullptr, nullptr,
                              nullptr, work});
        if (opt_.store_q) {
            const int kmax = std::max(1, std::min(j.p2, j.nw));
            qv[3 * i] = cd.back().V = out_.qarena->alloc_n<double>(static_cast<size_t>(j.p2) * kmax);
            cd.back().ldv = j.p2;
            qv[3 * i + 1] = cd.back().tau = out_.qarena->alloc_n<double>(kmax);
            qv[3 * i + 2] = cd.back().sign = out_.qarena->alloc_n<double>(kmax);
        }
    }
    {
        Uploader u = up();
        const CpqrDesc* dc = u.put(cd);
        out_.ctr.h2d_bytes += u.bytes_h2d;
        run_cpqr(cd, dc, u);
        out_.ctr.launches++;
    }
    std::vector<int> rank;
    download(rank, d_rank, nj);
    AsmBuilder& wb = asm_slot(2);  // keeps its capacity across calls
    for (size_t i = 0; i < nj; ++i) {
        const Job& j = jobs[i];
        const int keep = rank[i];
        out_.ctr.cpqr_flops += 4.0 * j.p2 * double(j.nw) * keep + 2.0 * j.p2 * j.nw;
        if (ranked()) rank_flops(j.p, 4.0 * j.p2 * double(j.nw) * keep + 2.0 * j.p2 * j.nw);
        out_.ctr.cpqr_bytes += 8.0 * keep * j.nw;  // R out (8mn + 8rn)
        out_.ctr.k_bytes[K_CPQR] += 8.0 * keep * j.nw;
        if (keep >= j.p2) continue;
        Front& f = fr_[j.p];
        if (opt_.store_q) {  // factorize.cpp:514-519: T.H on the extra rows
            DevWFactor& qf = new_qfactor(j.p, f.rows.data() + j.cs, j.p2, keep, false);
            qf.a = qv[3 * i];
            qf.tau = qv[3 * i + 1];
            qf.sign = qv[3 * i + 2];
        }
        for (int r = j.cs + keep; r < j.cs + j.p2; ++r) out_.dropped_rows.push_back(f.rows[r]);
        f.rows.resize(j.cs + keep);
        if (keep == 0) continue;
        // write R back into the live neighbour columns (dead gaps get zeros)
        std::vector<int> ord;
        phys_order(f.keys, ord);
        std::vector<std::pair<int, int>> segs{{0, -1}};  // (dst col relative to c0, B col or -1)
        int bo = 0;
        for (size_t t = 0; t < ord.size(); ++t) {
            const KeyRef& k = f.keys[ord[t]];
            if (k.key == j.p || k.width == 0) continue;
            segs.emplace_back(k.col - j.c0, bo);
            segs.emplace_back(k.col + k.width - j.c0, -1);
            bo += k.width;
        }
        const int dcols = f.ncols - j.c0;
        const int di = wb.begin(f.mat + j.cs + static_cast<long long>(j.c0) * f.ld, f.ld, keep, dcols, 1,
                                static_cast<int>(segs.size()));
        wb.source(di, 0) = AsmSrc{j.B, 1, j.p2};
        for (int r = 0; r < keep; ++r) wb.row(di, r) = int4{-1, 0, 0, r};
        for (size_t s = 0; s < segs.size(); ++s) {
            wb.seg(di, static_cast<int>(s), std::min(segs[s].first, dcols));
            wb.km(di, static_cast<int>(s), 0) = segs[s].second;
        }
    }
    flush_assemble(wb);
    for (const Job& j : jobs) dfree(j.B, j.big);
}

// factorize.cpp:539-633 — Gauss-Seidel over interfaces, run as waves of a
// DAG whose edges join fronts that hold each other's key (the only way one
// interface's step reads what another writes).
void Engine::sparsify_cols_all() {
    ProfScope ps_(prof_, HostProf::SCOLS);
    std::vector<int> elig;
    for (size_t p = 0; p < fr_.size(); ++p)
        if (alive_[p] && fr_[p].live && width(static_cast<int>(p)) > 0 && fr_[p].scaled_ok) elig.push_back(static_cast<int>(p));
    if (elig.empty()) return;
    // Speculative rounds: every pending interface is factored from the
    // current data; in ascending order a result is accepted unless a lower
    // neighbour (an interface holding its key or whose key it holds) was
    // rejected or changed (rank < width) in the same round.  Accepted
    // results are exactly those of the reference's sequential sweep, since an
    // unchanged neighbour leaves every input untouched.
    std::vector<std::vector<int>> lower(elig.size());
    std::vector<int> eidx(fr_.size(), -1);
    for (size_t i = 0; i < elig.size(); ++i) eidx[elig[i]] = static_cast<int>(i);
    for (size_t i = 0; i < elig.size(); ++i) {
        const int p = elig[i];
        for (int m : holders_[p].get())
            if (m < p && eidx[m] >= 0) lower[i].push_back(m);
        for (const KeyRef& k : fr_[p].keys)
            if (k.key < p && eidx[k.key] >= 0) lower[i].push_back(k.key);
    }
    std::vector<char> bad(fr_.size(), 0), changed(fr_.size(), 0);
    std::vector<int> pending = elig;
    int rounds = 0;
    const int rot_batch = batch_;
    const size_t w0 = out_.W.size(), q0 = out_.Q.size();
    std::vector<int> depth(fr_.size(), -1);  // speculation depth of interfaces included in this round
    std::vector<char> done(fr_.size(), 0);
    const int kmax_depth = spec_depth_;
    while (!pending.empty()) {
        ++rounds;
        // include p when every lower neighbour is done or included, at a
        // bounded speculation depth
        std::vector<int> wave, later;
        for (int p : pending) {
            int dp = 0;
            bool ok = true;
            for (int q : lower[eidx[p]]) {
                if (done[q]) continue;
                if (depth[q] < 0) {
                    ok = false;
                    break;
                }
                dp = std::max(dp, depth[q] + 1);
            }
            if (ok && dp <= kmax_depth) {
                depth[p] = dp;
                wave.push_back(p);
            } else {
                later.push_back(p);
            }
        }
        struct Job {
            int p, cs, nG, wrows, kmax;
            std::vector<int> rparts, seg;  // seg offsets of holders in G
            std::vector<std::pair<int, int>> kg;  // (neighbour key, its first column in G's own part)
            bool gbig = false;
            int di = -1;
            double* G;
            double *V, *tau, *sign;
        };
        std::vector<Job> jobs;
        std::unique_ptr<NScope> sc1 = std::make_unique<NScope>(nprof_, "scols.G_descriptors");
        AsmBuilder& gb = asm_slot(3);  // keeps its capacity across calls
        std::vector<CpqrDesc> cd;
        int maxm = 0;
        // per-job shapes in parallel (holder sets normalised first: get() sorts lazily),
        // then allocation and descriptor reservation in wave order
        for (int p : wave) holders_[p].norm();
        jobs.resize(wave.size());
#pragma omp parallel for schedule(dynamic, 8) if (wave.size() > 64)
        for (long long wi = 0; wi < static_cast<long long>(wave.size()); ++wi) {
            const int p = wave[wi];
            const Front& f = fr_[p];
            Job& j = jobs[wi];
            j.p = p;
            j.cs = width(p);
            for (int m : holders_[p].v)
                if (m != p && fr_[m].live) j.rparts.push_back(m);
            int wrows = 0;
            for (int m : j.rparts) {
                j.seg.push_back(wrows);
                wrows += fr_[m].nrows();
            }
            int wcols = 0;
            for (const KeyRef& k : f.keys)  // ascending keys = physical order of the neighbour blocks
                if (k.key != p && k.width > 0) {
                    j.kg.emplace_back(k.key, wcols);
                    wcols += k.width;
                }
            j.wrows = wrows;
            j.nG = wrows + wcols;
            j.kmax = std::min(j.cs, j.nG);
        }
        if (ranked())
            for (const Job& j : jobs) {
                rank_flops(j.p, 4.0 * j.cs * double(j.nG) * j.kmax + 2.0 * j.cs * j.nG);  // upper bound (rank <= kmax)
                for (int m : j.rparts)
                    if (own(m) != own(j.p)) rank_cross(2, 16.0 * fr_[m].nrows() * j.cs);
            }
        for (Job& j : jobs) {
            j.G = dalloc(arena(), static_cast<size_t>(j.cs) * std::max(j.nG, 1), j.gbig);
            // G (cs x nG) built transposed: G column g <- a row of holder m or a column of own block;
            // logical G^T (nG x cs) gathered row by row, stored transposed as G (ld = cs).  The
            // row maps are filled in parallel below.
            const int nsrc = static_cast<int>(j.rparts.size()) + 1;
            j.di = -1;
            if (j.nG > 0) {
                j.di = gb.begin(j.G, j.cs, j.nG, j.cs, nsrc, 1, false);
                gb.dst[j.di].trans = 1;
            }
            j.V = out_.warena->alloc_n<double>(static_cast<size_t>(j.cs) * std::max(j.kmax, 1));
            j.tau = out_.warena->alloc_n<double>(std::max(j.kmax, 1));
            j.sign = out_.warena->alloc_n<double>(std::max(j.kmax, 1));
            maxm = std::max(maxm, j.cs);
            out_.ctr.cpqr_bytes += 8.0 * j.cs * j.nG;
        }
        sc1.reset();
        sc1 = std::make_unique<NScope>(nprof_, "scols.G_fill");
#pragma omp parallel for schedule(dynamic, 4) if (jobs.size() > 16)
        for (long long ji = 0; ji < static_cast<long long>(jobs.size()); ++ji) {
            const Job& j = jobs[ji];
            if (j.di < 0) continue;
            const int di = j.di, p = j.p;
            const Front& f = fr_[p];
            for (size_t s = 0; s < j.rparts.size(); ++s) {
                const Front& fm = fr_[j.rparts[s]];
                const int mq = fm.find(p);
                gb.source(di, static_cast<int>(s)) = AsmSrc{fm.mat + static_cast<long long>(fm.keys[mq].col) * fm.ld, 1, fm.ld};
                for (int q = 0; q < fm.nrows(); ++q) gb.row(di, j.seg[s] + q) = int4{-1, 0, static_cast<int>(s), q};
                gb.km(di, 0, static_cast<int>(s)) = 0;
            }
            const int so = static_cast<int>(j.rparts.size());
            gb.source(di, so) = AsmSrc{f.mat, f.ld, 1};  // transposed view of p's own rows
            for (const auto& kg : j.kg) {
                const KeyRef& k = f.keys[f.find(kg.first)];
                for (int o = 0; o < k.width; ++o) gb.row(di, j.wrows + kg.second + o) = int4{-1, 0, so, k.col + o};
            }
            gb.km(di, 0, so) = 0;
        }
        sc1.reset();
        std::unique_ptr<NScope> sc2 = std::make_unique<NScope>(nprof_, "scols.upload+cpqr+fetch");
        flush_assemble(gb);
        const size_t nj = jobs.size();
        if (gdump_.cluster >= 0)  // diagnostics (SPQR_DUMP_G): one interface's G before its CPQR
            for (const Job& j : jobs)
                if (j.p == gdump_.cluster && cur_stage_ == gdump_.stage) dump_g(j.G, j.cs, j.nG);
        int* d_rank = arena().alloc_n<int>(nj);
        double* d_r11 = arena().alloc_n<double>(nj);
        for (size_t i = 0; i < nj; ++i) {
            Job& j = jobs[i];
            double* work = arena().alloc_n<double>(3 * static_cast<size_t>(std::max(j.nG, 1)));
            cd.push_back(CpqrDesc{j.G, j.cs, j.cs, j.nG, opt_.eps, d_rank + i, d_r11 + i, j.V, j.cs, j.tau, j.sign,
                                  nullptr, work});
        }
        {
            Uploader u = up();
            const CpqrDesc* dc = u.put(cd);
            out_.ctr.h2d_bytes += u.bytes_h2d;
        run_cpqr(cd, dc, u);
            out_.ctr.launches++;
        }
        std::vector<int> rank;
        download(rank, d_rank, nj);
        sc2.reset();
        std::unique_ptr<NScope> sc3 = std::make_unique<NScope>(nprof_, "scols.apply+rebuild_descr");
        // acceptance (ascending p), then structural updates of accepted changes
        std::map<int, std::vector<std::pair<int, int>>> hed;  // holder m -> (job, holder slot)
        std::vector<int> changed_p;
        std::vector<int> rejected;
        for (size_t i = 0; i < nj; ++i) {
            Job& j = jobs[i];
            const int r2 = rank[i];
            const double jf = 4.0 * j.cs * double(j.nG) * r2 + 2.0 * j.cs * j.nG;
            bool ok = true;
            for (int q : lower[eidx[j.p]])
                if (bad[q] || changed[q]) {
                    ok = false;
                    break;
                }
            if (ok) {
                out_.ctr.cpqr_flops += jf;
                out_.ctr.cpqr_bytes += 8.0 * r2 * j.nG;  // R out (8mn + 8rn)
                out_.ctr.k_bytes[K_CPQR] += 8.0 * r2 * j.nG;
            } else {  // speculative result discarded: redundant, not algorithmic, work
                out_.ctr.cpqr_bytes -= 8.0 * j.cs * j.nG;
                out_.ctr.k_bytes[K_CPQR] -= 8.0 * j.cs * j.nG;
                out_.ctr.cpqr_redundant_bytes += 8.0 * j.cs * j.nG + 8.0 * r2 * j.nG;
                out_.ctr.cpqr_redundant_flops += jf;
            }
            if (!ok) {
                bad[j.p] = 1;
                rejected.push_back(j.p);
                continue;
            }
            done[j.p] = 1;
            if (r2 >= j.cs) continue;
            changed[j.p] = 1;
            const int p = j.p;
            Front& f = fr_[p];
            if (r2 > 0) {
                batch_ = rot_batch;
                DevWFactor& w = new_factor(1, p, j.cs, r2, cols_[p], nullptr);
                w.a = j.V;
                w.tau = j.tau;
                w.sign = j.sign;
                if (opt_.store_q) {  // factorize.cpp:583-588: the same T.H on p's first cs rows
                    DevWFactor& qf = new_qfactor(p, f.rows.data(), j.cs, r2, false);
                    qf.a = j.V;
                    qf.tau = j.tau;
                    qf.sign = j.sign;
                }
            }
            for (size_t s = 0; s < j.rparts.size(); ++s) {
                const int m = j.rparts[s];
                if (r2 > 0)
                    hed[m].emplace_back(static_cast<int>(i), static_cast<int>(s));
                else {
                    hed[m].emplace_back(static_cast<int>(i), -1 - static_cast<int>(s));  // drop key p
                    holders_[p].remove(m);
                }
            }
            for (int q = r2; q < j.cs; ++q) {
                out_.pivot_row[cols_[p][q]] = f.rows[q];
                ++npiv_;
            }
            changed_p.push_back(static_cast<int>(i));
        }
        // materialise p fronts and their holders
        AsmBuilder& mb = asm_slot(4);  // keeps its capacity across calls
        std::vector<std::pair<int, Front>> updates;
        for (int ji : changed_p) {
            Job& j = jobs[ji];
            const int p = j.p, cs = j.cs, r2 = rank[ji];
            const Front& f = fr_[p];
            const int p2 = f.nrows() - cs;
            Front nf;
            nf.live = true;
            nf.rows.assign(f.rows.begin(), f.rows.begin() + r2);
            nf.rows.insert(nf.rows.end(), f.rows.begin() + cs, f.rows.end());
            for (const KeyRef& k : f.keys) {
                if (k.key == p) {
                    if (r2 > 0) nf.keys.push_back(KeyRef{p, r2, 0});
                } else {
                    nf.keys.push_back(KeyRef{k.key, k.width, 0});
                }
            }
            nf.scaled_ok = r2 > 0;
            layout(p, nf.keys, nf.ncols);
            nf.ld = std::max(1, nf.nrows());
            nf.mat = dalloc(arena(), static_cast<size_t>(nf.ld) * std::max(nf.ncols, 1), nf.big);
            std::vector<int> ord;
            phys_order(nf.keys, ord);
            const int di = mb.begin(nf.mat, nf.ld, nf.nrows(), nf.ncols, 2, static_cast<int>(ord.size()));
            mb.source(di, 0) = AsmSrc{j.G, 1, cs};      // R rows (top r2)
            mb.source(di, 1) = AsmSrc{f.mat, 1, f.ld};  // old extra rows
            for (int q = 0; q < r2; ++q) mb.row(di, q) = int4{0, q, -1, 0};
            for (int q = 0; q < p2; ++q) mb.row(di, r2 + q) = int4{1, cs + q, -1, 0};
            for (size_t q = 0; q < ord.size(); ++q) {
                const KeyRef& k = nf.keys[ord[q]];
                mb.seg(di, static_cast<int>(q), k.col);
                if (k.key == p) {  // D = [I; 0]
                    mb.km(di, static_cast<int>(q), 0) = -2;
                    mb.km(di, static_cast<int>(q), 1) = -2;
                    continue;
                }
                const KeyRef& ok = f.keys[f.find(k.key)];
                int gofs = -1;
                for (const auto& kg : j.kg)
                    if (kg.first == k.key) gofs = kg.second;
                if (gofs >= 0) mb.km(di, static_cast<int>(q), 0) = j.wrows + gofs;
                mb.km(di, static_cast<int>(q), 1) = ok.col;
            }
            mb.drop_if_empty();
            cols_[p].resize(r2);
            if (r2 == 0) holders_[p].clear();
            updates.emplace_back(p, std::move(nf));
        }
        // holders: B_m = (R seg_m)^T written in place into the first r2 columns of
        // m's p block (the rest of the block becomes dead columns), or the key is
        // dropped when r2 == 0 — no rebuild of m
        for (auto& [m, edits] : hed) {
            Front& fm = fr_[m];
            for (auto& [ji, s] : edits) {
                const Job& j = jobs[ji];
                const int mq = fm.find(j.p);
                if (s < 0) {
                    fm.keys.erase(fm.keys.begin() + mq);
                    continue;
                }
                const int r2 = rank[ji];
                if (fm.nrows() > 0) {
                    const int di = mb.begin(fm.mat + static_cast<long long>(fm.keys[mq].col) * fm.ld, fm.ld, fm.nrows(), r2,
                                            1, 1, false);
                    mb.source(di, 0) = AsmSrc{j.G + static_cast<long long>(j.seg[s]) * j.cs, j.cs, 1};
                    for (int q = 0; q < fm.nrows(); ++q) mb.row(di, q) = int4{-1, 0, 0, q};
                    mb.km(di, 0, 0) = 0;
                }
                fm.keys[mq].width = r2;
            }
        }
        sc3.reset();
        {
            NScope sc4(nprof_, "scols.rebuild_flush");
            flush_assemble(mb);
        }
        for (auto& [f, nf] : updates) {
            dfree(fr_[f].mat, fr_[f].big);
            fr_[f] = std::move(nf);
        }
        for (const Job& j : jobs) dfree(j.G, j.gbig);
        for (const Job& j : jobs) {
            bad[j.p] = 0;
            changed[j.p] = 0;
            depth[j.p] = -1;
        }
        pending.clear();
        std::merge(rejected.begin(), rejected.end(), later.begin(), later.end(), std::back_inserter(pending));
    }
    if (!sprof_.empty()) sprof_.back().scol_waves = rounds;
    std::stable_sort(out_.W.begin() + w0, out_.W.end(),
                     [](const DevWFactor& a, const DevWFactor& b) { return a.cluster < b.cluster; });
    std::stable_sort(out_.Q.begin() + q0, out_.Q.end(),
                     [](const DevWFactor& a, const DevWFactor& b) { return a.cluster < b.cluster; });
}

// factorize.cpp:635-729 — children concatenate into parents; every live front
// is rebuilt into the other arena (pivot rows of all children first).
void Engine::merge_level() {
    ProfScope ps_(prof_, HostProf::MERGE);
    // groups of live fronts by parent cluster (ascending parents, ascending kids)
    std::vector<int> gp;       // parent per group
    std::vector<int> gstart;   // kids of group g: gkids[gstart[g] .. gstart[g+1])
    std::vector<int> gkids;
    std::vector<int> group_of(fr_.size(), -1);
    {
        std::vector<std::pair<int, int>> pk;  // (parent, kid)
        for (size_t c = 0; c < fr_.size(); ++c)
            if (alive_[c] && fr_[c].live) pk.emplace_back(h_.clusters[c].parent, static_cast<int>(c));
        std::sort(pk.begin(), pk.end());
        for (size_t i = 0; i < pk.size(); ++i) {
            if (pk[i].first < 0)
                throw std::logic_error("spaqr engine: live front without a parent cluster at merge (cluster " +
                                       std::to_string(pk[i].second) + ", level " +
                                       std::to_string(h_.clusters[pk[i].second].level) + ", stage " +
                                       std::to_string(cur_stage_) + ", rows " + std::to_string(fr_[pk[i].second].nrows()) +
                                       ", width " + std::to_string(width(pk[i].second)) + ")");
            if (i == 0 || pk[i].first != pk[i - 1].first) {
                gp.push_back(pk[i].first);
                gstart.push_back(static_cast<int>(gkids.size()));
                group_of[pk[i].first] = static_cast<int>(gp.size()) - 1;
            }
            gkids.push_back(pk[i].second);
        }
        gstart.push_back(static_cast<int>(gkids.size()));
    }
    const int ng = static_cast<int>(gp.size());
    if (ranked())
        for (int g = 0; g < ng; ++g)
            for (int t = gstart[g]; t < gstart[g + 1]; ++t) {
                const Front& F = fr_[gkids[t]];
                if (own(gkids[t]) != own(gp[g])) rank_cross(3, 8.0 * F.nrows() * F.ncols);
            }
    std::vector<int> child_off(fr_.size(), -1);
    for (int g = 0; g < ng; ++g) {
        const int P = gp[g];
        cols_[P].clear();
        int o = 0;
        for (int t = gstart[g]; t < gstart[g + 1]; ++t) {
            const int c = gkids[t];
            cols_[P].insert(cols_[P].end(), cols_[c].begin(), cols_[c].end());
            child_off[c] = o;
            o += width(c);
        }
    }
    if (!dist_ghost_.empty()) {
        // the other subtrees' merges, columns only (their ranks merge the fronts): groups ng..
        // hold them, so a top-separator front's keys on those clusters split like any other
        std::vector<std::pair<int, int>> gk;
        for (size_t c = 0; c < dist_ghost_.size(); ++c)
            if (dist_ghost_[c]) gk.emplace_back(h_.clusters[c].parent, static_cast<int>(c));
        std::sort(gk.begin(), gk.end());
        int o = 0;
        for (size_t i = 0; i < gk.size(); ++i) {
            const int P = gk[i].first, c = gk[i].second;
            if (P < 0) throw std::logic_error("distributed factorization: subtree cluster without a parent");
            if (i == 0 || P != gk[i - 1].first) {
                if (i > 0) gstart.push_back(static_cast<int>(gkids.size()));
                gp.push_back(P);
                group_of[P] = static_cast<int>(gp.size()) - 1;
                cols_[P].clear();
                o = 0;
            }
            gkids.push_back(c);
            child_off[c] = o;
            o += width(c);
            cols_[P].insert(cols_[P].end(), cols_[c].begin(), cols_[c].end());
            dist_ghost_[c] = 0;
        }
        if (!gk.empty()) gstart.push_back(static_cast<int>(gkids.size()));
        for (const auto& pc : gk) dist_ghost_[pc.first] = 1;
    }
    DeviceArena& next = *arena_[cur_ ^ 1];
    std::unique_ptr<NScope> m1 = std::make_unique<NScope>(nprof_, "merge.descriptors");
    AsmBuilder& mb = asm_slot(5);  // keeps its capacity across calls
    struct Plan {
        Front nf;
        std::vector<int2> rowsrc;  // (kid slot, row)
        std::vector<int> ord;
        int nseg = 0, di = -1;
    };
    std::vector<Plan> plans(ng);
#pragma omp parallel for schedule(dynamic, 64)
    for (int g = 0; g < ng; ++g) {
        const int P = gp[g];
        const int k0 = gstart[g], k1 = gstart[g + 1];
        Plan& pl = plans[g];
        Front& nf = pl.nf;
        nf.live = true;
        bool movable = false;
        if (k1 - k0 == 1) {
            movable = true;
            for (const KeyRef& k : fr_[gkids[k0]].keys)
                if (width(k.key) != 0 && width(h_.clusters[k.key].parent) != width(k.key)) {
                    movable = false;
                    break;
                }
        }
        nf.scaled_ok = movable ? fr_[gkids[k0]].scaled_ok : false;
        size_t nr = 0;
        for (int t = k0; t < k1; ++t) nr += fr_[gkids[t]].rows.size();
        nf.rows.reserve(nr);
        pl.rowsrc.reserve(nr);
        for (int pass = 0; pass < 2; ++pass)  // pivot rows of all children first, then remainders
            for (int t = k0; t < k1; ++t) {
                const Front& fc = fr_[gkids[t]];
                const int take = std::min(width(gkids[t]), fc.nrows());
                const int i0 = pass == 0 ? 0 : take, i1 = pass == 0 ? take : fc.nrows();
                for (int i = i0; i < i1; ++i) {
                    nf.rows.push_back(fc.rows[i]);
                    pl.rowsrc.push_back(int2{t - k0, i});
                }
            }
        std::vector<int> pkeys;
        for (int t = k0; t < k1; ++t)
            for (const KeyRef& k : fr_[gkids[t]].keys)
                if (width(k.key) != 0) pkeys.push_back(h_.clusters[k.key].parent);
        std::sort(pkeys.begin(), pkeys.end());
        pkeys.erase(std::unique(pkeys.begin(), pkeys.end()), pkeys.end());
        nf.keys.reserve(pkeys.size());
        for (int K : pkeys) nf.keys.push_back(KeyRef{K, width(K), 0});
        layout(P, nf.keys, nf.ncols);
        nf.ld = std::max(1, nf.nrows());
        phys_order(nf.keys, pl.ord);
        for (int q : pl.ord) {
            const int gk = group_of[nf.keys[q].key];
            pl.nseg += gstart[gk + 1] - gstart[gk];
        }
    }
    for (int g = 0; g < ng; ++g) {
        Plan& pl = plans[g];
        Front& nf = pl.nf;
        nf.mat = dalloc(next, static_cast<size_t>(nf.ld) * std::max(nf.ncols, 1), nf.big);
        if (nf.nrows() == 0 || nf.ncols == 0) continue;
        pl.di = mb.begin(nf.mat, nf.ld, nf.nrows(), nf.ncols, gstart[g + 1] - gstart[g], pl.nseg);
    }
#pragma omp parallel for schedule(dynamic, 64)
    for (int g = 0; g < ng; ++g) {
        Plan& pl = plans[g];
        if (pl.di < 0) continue;
        const int di = pl.di, k0 = gstart[g], nsrc = gstart[g + 1] - k0;
        for (int s = 0; s < nsrc; ++s) mb.source(di, s) = AsmSrc{fr_[gkids[k0 + s]].mat, 1, fr_[gkids[k0 + s]].ld};
        for (size_t i = 0; i < pl.rowsrc.size(); ++i) mb.row(di, static_cast<int>(i)) = int4{-1, 0, pl.rowsrc[i].x, pl.rowsrc[i].y};
        int sg = 0;
        for (int q : pl.ord) {  // each parent key splits into its children's column ranges
            const KeyRef& dk = pl.nf.keys[q];
            const int gk = group_of[dk.key];
            for (int t = gstart[gk]; t < gstart[gk + 1]; ++t) {
                const int ck = gkids[t];
                mb.seg(di, sg, dk.col + child_off[ck]);
                for (int s = 0; s < nsrc; ++s) {
                    const Front& fc = fr_[gkids[k0 + s]];
                    const int ci = fc.find(ck);
                    if (ci >= 0) mb.km(di, sg, s) = fc.keys[ci].col;
                }
                ++sg;
            }
        }
    }
    m1.reset();
    std::unique_ptr<NScope> m2 = std::make_unique<NScope>(nprof_, "merge.flush+rebuild_host");
    flush_assemble(mb);
    for (size_t c = 0; c < fr_.size(); ++c)
        if (alive_[c] && fr_[c].live && fr_[c].big) dfree(fr_[c].mat, true);
#pragma omp parallel for schedule(dynamic, 512)
    for (long long c = 0; c < static_cast<long long>(fr_.size()); ++c)
        if (alive_[c] && fr_[c].live) {
            fr_[c].retire();
            alive_[c] = 0;
        }
#pragma omp parallel for schedule(dynamic, 512)
    for (long long c = 0; c < static_cast<long long>(holders_.size()); ++c) holders_[c].clear();
    for (int g = 0; g < ng; ++g) {
        fr_[gp[g]] = std::move(plans[g].nf);
        alive_[gp[g]] = 1;
    }
    {  // holder sets: counted first, so each set grows once (ascending P: already sorted)
        std::vector<int> cnt(holders_.size(), 0);
        for (int g = 0; g < ng; ++g)
            for (const KeyRef& k : fr_[gp[g]].keys) ++cnt[k.key];
#pragma omp parallel for schedule(dynamic, 512)
        for (long long c = 0; c < static_cast<long long>(holders_.size()); ++c)
            if (cnt[c]) holders_[c].v.reserve(cnt[c]);
        for (int g = 0; g < ng; ++g) {
            const int P = gp[g];
            for (const KeyRef& k : fr_[P].keys) holders_[k.key].add(P);
        }
    }
    // everything of this stage lived in arena cur_; the next stage starts clean
    sync();
    arena_[cur_]->reset();
    cur_ ^= 1;
}

void Engine::snapshot(StageStats& st) {  // factorize.cpp:731-743
    // ascending cluster order (the reference iterates its std::map); blocks of clusters
    // are scanned in parallel and concatenated in order
    const long long nc = static_cast<long long>(fr_.size());
    constexpr long long kBlk = 4096;
    const long long nb = (nc + kBlk - 1) / kBlk;
    std::vector<std::vector<std::pair<int, double>>> part(nb);
    std::vector<long long> trows(nb, 0), tcols(nb, 0);
#pragma omp parallel for schedule(static)
    for (long long q = 0; q < nb; ++q)
        for (long long c = q * kBlk; c < std::min(nc, (q + 1) * kBlk); ++c) {
            if (!alive_[c]) continue;
            const Front& f = fr_[c];
            if (!f.live) continue;
            const int cs = width(static_cast<int>(c));
            if (cs > 0) part[q].emplace_back(cs, static_cast<double>(f.nrows()) / cs);
            if (h_.clusters[c].tree_node == h_.tree->root) {
                trows[q] += f.nrows();
                tcols[q] += cs;
            }
        }
    for (long long q = 0; q < nb; ++q) {
        for (const auto& pc : part[q]) {
            st.front_cols.push_back(pc.first);
            st.front_aspect.push_back(pc.second);
        }
        st.top_rows += trows[q];
        st.top_cols += tcols[q];
    }
    if (dist_stage(cur_stage_)) {  // split stage: the entries by cluster, merged on rank 0 at the end
        auto& v = dist_snap_[cur_stage_];
        v.clear();
        for (long long c = 0; c < nc; ++c)
            if (alive_[c] && fr_[c].live && width(static_cast<int>(c)) > 0 && (dist_->rank == 0 || !dist_top_[c]))
                v.push_back(SnapE{static_cast<int>(c), width(static_cast<int>(c)),
                                  static_cast<double>(fr_[c].nrows()) / width(static_cast<int>(c))});
    }
}


// ---------------------------------------------------------------------------------------
// Distributed split stages (opt.dist).  Every rank builds the same engine; in
// the stages L+1 .. dist_kend_ (before any scale_all: rows are still pure) each eliminates only
// its own subtree's clusters (ranks.cpp owners).  No row of A couples two subtrees' interiors,
// so the ranks' eliminations commute; the only fronts two ranks touch are pieces of the top
// separators, each rank transforming its own side's rows.  After each split stage the ranks
// exchange their effects on those fronts and re-merge them exactly as the sequential engine
// leaves them (rows at the start of the stage in order minus every rank's pivots, then appended
// rows in ascending source-cluster order = rank order); after the last one ranks > 0 hand their
// subtree to rank 0, which runs the remaining stages.
namespace {
struct DistWriter {
    std::vector<char> b;
    template <class T>
    void put(const T* p, size_t n) {
        const char* c = reinterpret_cast<const char*>(p);
        b.insert(b.end(), c, c + sizeof(T) * n);
    }
    void i64(long long v) { put(&v, 1); }
    void ivec(const std::vector<int>& v) {
        i64(static_cast<long long>(v.size()));
        put(v.data(), v.size());
    }
};
struct DistReader {
    const char* p;
    size_t n, o = 0;
    template <class T>
    void get(T* d, size_t cnt) {
        const size_t bytes = sizeof(T) * cnt;
        if (o + bytes > n) throw std::runtime_error("distributed factorization: truncated message");
        std::memcpy(d, p + o, bytes);
        o += bytes;
    }
    long long i64() {
        long long v;
        get(&v, 1);
        return v;
    }
    std::vector<int> ivec() {
        const long long k = i64();
        if (k < 0 || static_cast<size_t>(k) > n) throw std::runtime_error("distributed factorization: bad length");
        std::vector<int> v(k);
        get(v.data(), v.size());
        return v;
    }
};
}  // namespace

// Partitioned state of a distributed factorization: each rank keeps the fronts of its own
// subtree and the pieces of the top separators (every rank, kept identical stage by stage); the
// other subtrees' fronts are released here and reach rank 0 at the end of the split stages.
void Engine::dist_partition_state() {
    dist_ghost_.assign(fr_.size(), 0);
    for (size_t c = 0; c < fr_.size(); ++c)
        if (!dist_top_[c] && dist_owner_[c] != dist_->rank && fr_[c].live) {
            dfree(fr_[c].mat, fr_[c].big);
            fr_[c].retire();
            alive_[c] = 0;
            dist_ghost_[c] = 1;
        }
    rebuild_holders();
}

// Values travel device to device: each rank gathers the values it sends into one cudaMalloc'ed
// buffer and sends its CUDA IPC handle with the metadata; the receivers open it (peer memory
// over NVLink on a multi-GPU node, the same memory when the ranks share a GPU) and their gather
// kernels read the values in place; acknowledgements release the buffer.  SPQR_DIST_HOST=1 sends
// the values inline through the host transport instead.
//
// Per split stage (all ranks to all): the clusters this rank eliminated and the top-separator
// fronts it touched (rows, keys, values, rows transformed in place).  At the last split stage
// (ranks > 0 to rank 0) also: every front of its subtree, their clusters' columns, all its W
// factors, pivot rows, trailing rows per stage and snapshot entries per stage.
std::vector<char> Engine::dist_export(int k, bool final_to_root) {
    static const bool host_mode = std::getenv("SPQR_DIST_HOST") != nullptr;
    DistWriter w;
    w.i64(0x53505144);  // "SPQD"
    w.i64(host_mode ? 0 : 1);
    std::vector<int> el, all_el;
    for (int c : stage_list_[k])
        if (dist_mine(c) && gone_[c]) el.push_back(c);
    std::sort(dist_touched_.begin(), dist_touched_.end());
    dist_touched_.erase(std::unique(dist_touched_.begin(), dist_touched_.end()), dist_touched_.end());
    std::vector<int> T, S;  // touched top fronts; (final) this subtree's live fronts
    for (int f : dist_touched_)
        if (dist_top_[f] && !gone_[f] && fr_[f].live) T.push_back(f);
    if (final_to_root)
        for (size_t c = 0; c < fr_.size(); ++c) {
            if (dist_top_[c] || dist_owner_[c] != dist_->rank) continue;
            if (gone_[c])
                all_el.push_back(static_cast<int>(c));
            else if (alive_[c] && fr_[c].live)
                S.push_back(static_cast<int>(c));
        }
    std::sort(dist_tr_.begin(), dist_tr_.end());
    // value space: T's blocks, then S's (ascending keys, ld = rows), then (final) W's [R | C]
    std::vector<int> TS(T);
    TS.insert(TS.end(), S.begin(), S.end());
    std::vector<long long> voff(TS.size() + 1, 0);
    for (size_t t = 0; t < TS.size(); ++t) voff[t + 1] = voff[t] + static_cast<long long>(fr_[TS[t]].nrows()) * fr_[TS[t]].ncols;
    const size_t nw = final_to_root ? out_.W.size() : 0;
    std::vector<long long> woff(nw + 1, voff.back());
    for (size_t q = 0; q < nw; ++q) {
        const DevWFactor& f = out_.W[q];
        if (f.kind != 0) throw std::logic_error("distributed factorization: rotation factor in a split stage");
        woff[q + 1] = woff[q] + static_cast<long long>(f.c) * (f.c + f.k);
    }
    const long long total = woff.back();
    double* dv = nullptr;
    CK(cudaMalloc(&dv, sizeof(double) * std::max<long long>(total, 1)));
    dist_vbuf_ = dv;
    AsmBuilder& gb = asm_slot(0);
    for (size_t t = 0; t < TS.size(); ++t) {
        const Front& F = fr_[TS[t]];
        if (F.nrows() == 0 || F.ncols == 0) continue;
        const int di = gb.begin(dv + voff[t], F.nrows(), F.nrows(), F.ncols, 1, static_cast<int>(F.keys.size()));
        gb.source(di, 0) = AsmSrc{F.mat, 1, F.ld};
        for (int i = 0; i < F.nrows(); ++i) gb.row(di, i) = int4{0, i, -1, 0};
        int o = 0;
        for (size_t q = 0; q < F.keys.size(); ++q) {
            gb.seg(di, static_cast<int>(q), o);
            gb.km(di, static_cast<int>(q), 0) = F.keys[q].col;
            o += F.keys[q].width;
        }
    }
    for (size_t q = 0; q < nw; ++q) {
        const DevWFactor& f = out_.W[q];
        if (f.c == 0) continue;
        const int di = gb.begin(dv + woff[q], f.c, f.c, f.c + f.k, 1, 1);
        gb.source(di, 0) = AsmSrc{f.a, 1, f.c};
        for (int i = 0; i < f.c; ++i) gb.row(di, i) = int4{0, i, -1, 0};
        gb.seg(di, 0, 0);
        gb.km(di, 0, 0) = 0;
    }
    flush_assemble(gb);
    sync();
    if (!host_mode) {
        cudaIpcMemHandle_t hnd;
        CK(cudaIpcGetMemHandle(&hnd, dv));
        w.put(reinterpret_cast<const char*>(&hnd), sizeof hnd);
        w.i64(total);
    }
    w.ivec(el);
    auto put_front = [&](size_t t, bool with_tr) {
        const Front& F = fr_[TS[t]];
        w.i64(TS[t]);
        w.ivec(F.rows);
        std::vector<int> kw;
        for (const KeyRef& kr : F.keys) {
            kw.push_back(kr.key);
            kw.push_back(kr.width);
        }
        w.ivec(kw);
        if (with_tr) {
            std::vector<int> tr;
            auto it = std::lower_bound(dist_tr_.begin(), dist_tr_.end(), std::make_pair(TS[t], INT_MIN));
            for (; it != dist_tr_.end() && it->first == TS[t]; ++it) tr.push_back(it->second);
            w.ivec(tr);
        }
        w.i64(voff[t]);
    };
    w.i64(static_cast<long long>(T.size()));
    for (size_t t = 0; t < T.size(); ++t) put_front(t, true);
    if (final_to_root) {
        w.i64(static_cast<long long>(S.size()));
        for (size_t t = T.size(); t < TS.size(); ++t) put_front(t, false);
        for (int c : S) w.ivec(cols_[c]);
        w.ivec(all_el);
        w.i64(static_cast<long long>(nw));
        for (size_t q = 0; q < nw; ++q) {
            const DevWFactor& f = out_.W[q];
            const int meta[5] = {f.cluster, f.c, f.k, f.scale_only ? 1 : 0, f.batch};
            w.put(meta, 5);
            w.put(out_.idx.data() + f.cols_off, f.c);
            w.put(out_.idx.data() + f.coupled_off, f.k);
            w.i64(woff[q]);
        }
        std::vector<int> piv;
        for (int c : all_el)
            for (int j : cols_[c]) {
                piv.push_back(j);
                piv.push_back(static_cast<int>(out_.pivot_row[j]));
            }
        w.ivec(piv);
        w.i64(npiv_);
        w.i64(static_cast<long long>(dist_tseg_.size()));
        size_t t0 = 0;
        for (const auto& sg : dist_tseg_) {
            w.i64(sg.first);
            w.ivec(std::vector<int>(out_.trailing_rows.begin() + t0, out_.trailing_rows.begin() + sg.second));
            t0 = sg.second;
        }
        w.i64(static_cast<long long>(dist_snap_.size()));
        for (const auto& [st, v] : dist_snap_) {
            w.i64(st);
            w.i64(static_cast<long long>(v.size()));
            w.put(v.data(), v.size());
        }
    }
    if (host_mode) {  // the values inline
        std::vector<double> hv(total);
        if (total > 0) CK(cudaMemcpy(hv.data(), dv, sizeof(double) * total, cudaMemcpyDeviceToHost));
        w.i64(total);
        w.put(hv.data(), hv.size());
        CK(cudaFree(dv));
        dist_vbuf_ = nullptr;
    }
    return std::move(w.b);
}

// Apply the other ranks' messages (msgs[rank]; this rank's own entry is empty, its effects are
// in place).  Each touched top-separator front becomes what the sequential engine would hold
// after the stage: its rows at the start of the stage in order, minus every rank's pivots, then
// the rows each rank appended in rank order (= ascending source cluster); a row's values come
// from the rank that transformed or appended it, else from this rank's copy; its keys are the
// union minus the eliminated clusters.  The final messages (on rank 0) add the other subtrees'
// fronts, columns, W factors, pivot and trailing rows and snapshot entries.
void Engine::dist_apply(const std::vector<std::vector<char>>& msgs, bool final_to_root) {
    const int G = dist_->size, me = dist_->rank;
    struct WIn {
        int cl, c, k, so, batch;
        std::vector<int> cols, cp;
        long long off;
    };
    struct FIn {
        int f;
        std::vector<int> rows, kw, tr, cols;
        long long off;
    };
    struct Msg {
        bool present = false;
        std::vector<int> el, all_el, piv;
        long long npiv = 0;
        std::vector<WIn> ws;
        std::vector<FIn> fs, sub;
        std::vector<std::pair<int, std::vector<int>>> tsegs;
        std::vector<std::pair<int, std::vector<SnapE>>> snaps;
        const double* vp = nullptr;
        double* peer = nullptr;
        std::vector<double> inline_vals;
    };
    std::vector<Msg> M(G);
    struct PeerClose {
        std::vector<Msg>& m;
        ~PeerClose() {
            for (auto& x : m)
                if (x.peer) cudaIpcCloseMemHandle(x.peer);
        }
    } closer{M};
    for (int r = 0; r < G; ++r) {
        if (r == me || msgs[r].empty()) continue;
        DistReader rd{msgs[r].data(), msgs[r].size()};
        if (rd.i64() != 0x53505144) throw std::runtime_error("distributed factorization: bad message");
        const bool ipc = rd.i64() == 1;
        Msg& m = M[r];
        m.present = true;
        if (ipc) {
            cudaIpcMemHandle_t hnd;
            rd.get(reinterpret_cast<char*>(&hnd), sizeof hnd);
            out_.dist_bytes += 8 * rd.i64();  // the values, read over peer memory
            void* p = nullptr;
            CK(cudaIpcOpenMemHandle(&p, hnd, cudaIpcMemLazyEnablePeerAccess));
            m.peer = static_cast<double*>(p);
            m.vp = m.peer;
        }
        m.el = rd.ivec();
        auto get_front = [&](FIn& x, bool with_tr) {
            x.f = static_cast<int>(rd.i64());
            if (x.f < 0 || static_cast<size_t>(x.f) >= fr_.size()) throw std::runtime_error("distributed factorization: bad front");
            x.rows = rd.ivec();
            x.kw = rd.ivec();
            if (with_tr) x.tr = rd.ivec();
            x.off = rd.i64();
        };
        m.fs.resize(rd.i64());
        for (auto& x : m.fs) get_front(x, true);
        if (final_to_root) {
            m.sub.resize(rd.i64());
            for (auto& x : m.sub) get_front(x, false);
            for (auto& x : m.sub) x.cols = rd.ivec();
            m.all_el = rd.ivec();
            m.ws.resize(rd.i64());
            for (auto& f : m.ws) {
                int meta[5];
                rd.get(meta, 5);
                f.cl = meta[0], f.c = meta[1], f.k = meta[2], f.so = meta[3], f.batch = meta[4];
                f.cols.resize(f.c);
                f.cp.resize(f.k);
                rd.get(f.cols.data(), f.c);
                rd.get(f.cp.data(), f.k);
                f.off = rd.i64();
            }
            m.piv = rd.ivec();
            m.npiv = rd.i64();
            m.tsegs.resize(rd.i64());
            for (auto& sg : m.tsegs) {
                sg.first = static_cast<int>(rd.i64());
                sg.second = rd.ivec();
            }
            m.snaps.resize(rd.i64());
            for (auto& sn : m.snaps) {
                sn.first = static_cast<int>(rd.i64());
                sn.second.resize(rd.i64());
                rd.get(sn.second.data(), sn.second.size());
            }
        }
        if (!ipc) {
            const long long total = rd.i64();
            m.inline_vals.resize(static_cast<size_t>(std::max<long long>(total, 0)));
            rd.get(m.inline_vals.data(), m.inline_vals.size());
            double* d = arena().alloc_n<double>(std::max<long long>(total, 1));
            if (total > 0) CK(cudaMemcpyAsync(d, m.inline_vals.data(), sizeof(double) * total, cudaMemcpyHostToDevice, st_));
            m.vp = d;
        }
    }
    // clusters the other ranks eliminated (their fronts are not held here)
    for (int r = 0; r < G; ++r)
        for (const std::vector<int>* v : {&M[r].el, &M[r].all_el})
            for (int c : *v) {
                if (c < 0 || static_cast<size_t>(c) >= fr_.size()) throw std::runtime_error("distributed factorization: bad cluster");
                holders_[c].clear();
                gone_[c] = 1;
                dist_ghost_[c] = 0;
            }
    AsmBuilder& mb = asm_slot(0);
    auto in = [](const std::vector<int>& v, int a) { return std::binary_search(v.begin(), v.end(), a); };
    // touched top-separator fronts: versions by front
    std::map<int, std::vector<std::pair<int, const FIn*>>> byf;
    for (int r = 0; r < G; ++r)
        for (const auto& x : M[r].fs) byf[x.f].emplace_back(r, &x);
    std::vector<std::pair<int, Front>> repl;
    for (const auto& [f, vers] : byf) {
        if (gone_[f] || !fr_[f].live) throw std::runtime_error("distributed factorization: touched front not live");
        const Front& C = fr_[f];
        const std::vector<int>& start = start_rows_[f];
        std::vector<int> sstart(start), sc(C.rows);
        std::sort(sstart.begin(), sstart.end());
        std::sort(sc.begin(), sc.end());
        const int nv = static_cast<int>(vers.size());
        std::vector<std::vector<int>> sr(nv), str(nv);
        std::vector<std::vector<std::pair<int, int>>> pos(nv);
        for (int v = 0; v < nv; ++v) {
            const FIn& x = *vers[v].second;
            sr[v] = x.rows;
            std::sort(sr[v].begin(), sr[v].end());
            str[v] = x.tr;
            std::sort(str[v].begin(), str[v].end());
            for (size_t i = 0; i < x.rows.size(); ++i) pos[v].emplace_back(x.rows[i], static_cast<int>(i));
            std::sort(pos[v].begin(), pos[v].end());
        }
        std::vector<std::pair<int, int>> cpos;
        for (int i = 0; i < C.nrows(); ++i) cpos.emplace_back(C.rows[i], i);
        std::sort(cpos.begin(), cpos.end());
        auto find = [](const std::vector<std::pair<int, int>>& pv, int g) {
            auto it = std::lower_bound(pv.begin(), pv.end(), std::make_pair(g, INT_MIN));
            if (it == pv.end() || it->first != g) throw std::logic_error("distributed factorization: row missing");
            return it->second;
        };
        Front nf;
        nf.live = true;
        std::vector<int2> src;  // (source: 0 = this rank's front, 1 + v = version v; row)
        for (int g : start) {
            if (!in(sc, g)) continue;  // a pivot of this rank
            bool kept = true;
            for (int v = 0; v < nv && kept; ++v) kept = in(sr[v], g);
            if (!kept) continue;  // a pivot of another rank
            int s0 = 0, row = find(cpos, g);
            for (int v = 0; v < nv; ++v)
                if (in(str[v], g)) {
                    s0 = 1 + v;
                    row = find(pos[v], g);
                }
            nf.rows.push_back(g);
            src.push_back(int2{s0, row});
        }
        int vi = 0;
        for (int r = 0; r < G; ++r) {  // appended rows in rank order
            if (r == me) {
                for (int i = 0; i < C.nrows(); ++i)
                    if (!in(sstart, C.rows[i])) {
                        nf.rows.push_back(C.rows[i]);
                        src.push_back(int2{0, i});
                    }
                continue;
            }
            while (vi < nv && vers[vi].first < r) ++vi;
            if (vi < nv && vers[vi].first == r) {
                const FIn& x = *vers[vi].second;
                for (size_t i = 0; i < x.rows.size(); ++i)
                    if (!in(sstart, x.rows[i])) {
                        nf.rows.push_back(x.rows[i]);
                        src.push_back(int2{1 + vi, static_cast<int>(i)});
                    }
            }
        }
        std::vector<std::pair<int, int>> ks;
        for (const KeyRef& kr : C.keys)
            if (!gone_[kr.key]) ks.emplace_back(kr.key, kr.width);
        std::vector<std::vector<int>> roff(nv);
        for (int v = 0; v < nv; ++v) {
            const FIn& x = *vers[v].second;
            int o = 0;
            for (size_t q = 0; q + 1 < x.kw.size(); q += 2) {
                roff[v].push_back(o);
                o += x.kw[q + 1];
                if (!gone_[x.kw[q]]) ks.emplace_back(x.kw[q], x.kw[q + 1]);
            }
        }
        std::sort(ks.begin(), ks.end());
        ks.erase(std::unique(ks.begin(), ks.end(), [](const auto& a, const auto& b) { return a.first == b.first; }), ks.end());
        for (const auto& kk : ks) nf.keys.push_back(KeyRef{kk.first, kk.second, 0});
        layout(f, nf.keys, nf.ncols);
        nf.ld = std::max(1, nf.nrows());
        nf.mat = dalloc(arena(), static_cast<size_t>(nf.ld) * std::max(nf.ncols, 1), nf.big);
        std::vector<int> ord;
        phys_order(nf.keys, ord);
        const int di = mb.begin(nf.mat, nf.ld, nf.nrows(), nf.ncols, 1 + nv, static_cast<int>(ord.size()));
        mb.source(di, 0) = AsmSrc{C.mat, 1, C.ld};
        for (int v = 0; v < nv; ++v) {
            const FIn& x = *vers[v].second;
            mb.source(di, 1 + v) = AsmSrc{M[vers[v].first].vp + x.off, 1, static_cast<long long>(std::max<size_t>(x.rows.size(), 1))};
        }
        for (int i = 0; i < nf.nrows(); ++i) mb.row(di, i) = int4{src[i].x, src[i].y, -1, 0};
        for (size_t q = 0; q < ord.size(); ++q) {
            const KeyRef& kr = nf.keys[ord[q]];
            mb.seg(di, static_cast<int>(q), kr.col);
            const int ci = C.find(kr.key);
            mb.km(di, static_cast<int>(q), 0) = ci >= 0 ? C.keys[ci].col : -1;
            for (int v = 0; v < nv; ++v) {
                const FIn& x = *vers[v].second;
                int ri = -1;
                for (size_t t = 0; t + 1 < x.kw.size(); t += 2)
                    if (x.kw[t] == kr.key) ri = roff[v][t / 2];
                mb.km(di, static_cast<int>(q), 1 + v) = ri;
            }
            if (ci < 0) holders_[kr.key].add(f);
        }
        mb.drop_if_empty();
        repl.emplace_back(f, std::move(nf));
    }
    if (final_to_root) {
        // the other subtrees' fronts and columns
        for (int r = 0; r < G; ++r)
            for (const auto& x : M[r].sub) {
                cols_[x.f] = x.cols;
                Front nf;
                nf.live = true;
                nf.rows = x.rows;
                std::vector<int> roff;
                int o = 0;
                for (size_t q = 0; q + 1 < x.kw.size(); q += 2) {
                    roff.push_back(o);
                    o += x.kw[q + 1];
                    nf.keys.push_back(KeyRef{x.kw[q], x.kw[q + 1], 0});
                }
                layout(x.f, nf.keys, nf.ncols);
                nf.ld = std::max(1, nf.nrows());
                nf.mat = dalloc(arena(), static_cast<size_t>(nf.ld) * std::max(nf.ncols, 1), nf.big);
                std::vector<int> ord;
                phys_order(nf.keys, ord);
                const int di = mb.begin(nf.mat, nf.ld, nf.nrows(), nf.ncols, 1, static_cast<int>(ord.size()));
                mb.source(di, 0) = AsmSrc{M[r].vp + x.off, 1, static_cast<long long>(std::max<size_t>(x.rows.size(), 1))};
                for (int i = 0; i < nf.nrows(); ++i) mb.row(di, i) = int4{0, i, -1, 0};
                for (size_t q = 0; q < ord.size(); ++q) {
                    mb.seg(di, static_cast<int>(q), nf.keys[ord[q]].col);
                    mb.km(di, static_cast<int>(q), 0) = roff[ord[q]];
                }
                mb.drop_if_empty();
                if (!dist_ghost_[x.f]) throw std::runtime_error("distributed factorization: unexpected subtree front");
                dist_ghost_[x.f] = 0;
                alive_[x.f] = 1;
                repl.emplace_back(x.f, std::move(nf));
            }
        // W factors (values gathered into the W arena), pivot rows
        for (int r = 0; r < G; ++r) {
            const Msg& m = M[r];
            long long wtot = 0;
            for (const auto& f : m.ws) wtot += static_cast<long long>(f.c) * (f.c + f.k);
            double* dw = out_.warena->alloc_n<double>(std::max<long long>(wtot, 1));
            long long o = 0;
            int nb = 0;
            for (const auto& f : m.ws) {
                DevWFactor& d = new_factor(0, f.cl, f.c, f.k, f.cols, f.so ? nullptr : &f.cp);
                d.batch = out_.nbatches + f.batch;  // the sending rank's waves, after this rank's
                nb = std::max(nb, f.batch + 1);
                d.a = dw + o;
                if (f.c > 0) {
                    const int di = mb.begin(d.a, f.c, f.c, f.c + f.k, 1, 1);
                    mb.source(di, 0) = AsmSrc{m.vp + f.off, 1, f.c};
                    for (int i = 0; i < f.c; ++i) mb.row(di, i) = int4{0, i, -1, 0};
                    mb.seg(di, 0, 0);
                    mb.km(di, 0, 0) = 0;
                }
                o += static_cast<long long>(f.c) * (f.c + f.k);
            }
            out_.nbatches += nb;
            for (size_t i = 0; i + 1 < m.piv.size(); i += 2) out_.pivot_row[m.piv[i]] = m.piv[i + 1];
            npiv_ += m.npiv;
        }
    }
    flush_assemble(mb);
    sync();  // every read of the other ranks' values is done
    for (auto& pr : repl) {
        Front& F = fr_[pr.first];
        dfree(F.mat, F.big);
        F.rows = std::move(pr.second.rows);
        F.keys = std::move(pr.second.keys);
        F.mat = pr.second.mat;
        F.big = pr.second.big;
        F.ld = pr.second.ld;
        F.ncols = pr.second.ncols;
        F.live = true;
        F.scaled_ok = false;
        F.tag.clear();
        F.soff.clear();
    }
    if (!final_to_root) return;
    for (size_t c = 0; c < dist_ghost_.size(); ++c)
        if (dist_ghost_[c]) throw std::runtime_error("distributed factorization: subtree front " + std::to_string(c) + " not received");
    dist_ghost_.clear();
    // chronological order of the split stages' results: W by (stage, cluster), trailing rows by
    // (stage, rank), every split stage's snapshot by cluster, nnz(W) per stage
    auto stage_of = [&](int c) { return h_.clusters[c].stage; };
    std::stable_sort(out_.W.begin(), out_.W.end(), [&](const DevWFactor& a, const DevWFactor& b) {
        const int sa = stage_of(a.cluster), sb = stage_of(b.cluster);
        return sa != sb ? sa > sb : a.cluster < b.cluster;
    });
    std::map<int, std::vector<std::vector<int>>> tby;  // stage -> per rank
    {
        size_t t0 = 0;
        for (const auto& sg : dist_tseg_) {
            auto& v = tby[sg.first];
            v.resize(G);
            v[me].assign(out_.trailing_rows.begin() + t0, out_.trailing_rows.begin() + sg.second);
            t0 = sg.second;
        }
    }
    for (int r = 0; r < G; ++r)
        for (const auto& sg : M[r].tsegs) {
            auto& v = tby[sg.first];
            v.resize(G);
            v[r] = sg.second;
        }
    out_.trailing_rows.clear();
    for (auto it = tby.rbegin(); it != tby.rend(); ++it)  // stages descending
        for (const auto& v : it->second) out_.trailing_rows.insert(out_.trailing_rows.end(), v.begin(), v.end());
    for (int r = 0; r < G; ++r)
        for (const auto& sn : M[r].snaps) {
            auto& v = dist_snap_[sn.first];
            v.insert(v.end(), sn.second.begin(), sn.second.end());
        }
    for (auto& st : out_.stages) {
        auto it = dist_snap_.find(st.stage);
        if (it == dist_snap_.end()) continue;
        auto v = it->second;
        std::sort(v.begin(), v.end(), [](const SnapE& a, const SnapE& b) { return a.c < b.c; });
        st.front_cols.clear();
        st.front_aspect.clear();
        for (const auto& e : v) {
            st.front_cols.push_back(e.cs);
            st.front_aspect.push_back(e.asp);
        }
        long long nnz = 0;  // cumulative nnz(W) after the stage (transforms.cpp:25-38)
        for (const auto& f : out_.W) {
            if (stage_of(f.cluster) < st.stage) continue;
            const long long c = f.c, kk = f.k;
            nnz += f.kind == 0 ? c * (c + 1) / 2 + c * kk : kk * c - kk * (kk - 1) / 2 + kk;
        }
        st.nnz_w = nnz;
    }
    rebuild_holders();
}

// One split stage's exchange.  Before the last split stage every rank's message goes to every
// other rank (rank r sends while the others receive from r) and all apply them; at the last one
// ranks > 0 send to rank 0 only, which applies them and continues alone.  A rank whose
// elimination failed sends its first failing cluster instead; the first of all ranks is raised
// (the sequential engine's error), by every rank before the last split stage, by rank 0 at it.
void Engine::dist_exchange(int k, int err_cluster, const std::string& err_reason) {
    const double t0 = now_s();
    const int G = dist_->size, me = dist_->rank;
    const bool final_stage = k == dist_kend_;
    std::vector<char> own;
    if (err_cluster >= 0) {  // an error record: magic, -1, cluster, reason
        DistWriter w;
        w.i64(0x53505144);
        w.i64(-1);
        w.i64(err_cluster);
        w.ivec(std::vector<int>(err_reason.begin(), err_reason.end()));
        own = std::move(w.b);
    } else if (!(final_stage && me == 0)) {
        own = dist_export(k, final_stage);
    }
    auto fail = [] { throw std::runtime_error("distributed factorization: transport failed"); };
    std::vector<std::vector<char>> msgs(G);
    for (int r = 0; r < G; ++r) {
        if (final_stage && r == 0) continue;  // nothing goes out of rank 0 at the last split stage
        if (r == me) {
            const long long n = static_cast<long long>(own.size());
            for (int q = 0; q < G; ++q) {
                if (q == me || (final_stage && q != 0)) continue;
                if (dist_->send(dist_->user, q, &n, sizeof n) || dist_->send(dist_->user, q, own.data(), n)) fail();
                out_.dist_bytes += n;
            }
        } else if (!final_stage || me == 0) {
            long long n = 0;
            if (dist_->recv(dist_->user, r, &n, sizeof n)) fail();
            msgs[r].resize(static_cast<size_t>(std::max<long long>(n, 0)));
            if (n > 0 && dist_->recv(dist_->user, r, msgs[r].data(), n)) fail();
            out_.dist_bytes += n;
        }
    }
    auto mode = [](const std::vector<char>& b) {  // -1 error, 0 inline values, 1 IPC values
        if (b.size() < 16) return -2;
        DistReader rd{b.data(), b.size()};
        rd.i64();
        return static_cast<int>(rd.i64());
    };
    int ecl = err_cluster;
    std::string why = err_reason;
    for (int r = 0; r < G; ++r)
        if (r != me && mode(msgs[r]) == -1) {
            DistReader rd{msgs[r].data(), msgs[r].size()};
            rd.i64();
            rd.i64();
            const int cl = static_cast<int>(rd.i64());
            const std::vector<int> rv = rd.ivec();
            if (ecl < 0 || cl < ecl) {
                ecl = cl;
                why.assign(rv.begin(), rv.end());
            }
        }
    if (ecl < 0 && (!final_stage || me == 0)) dist_apply(msgs, final_stage);
    // acknowledgements: a rank's IPC buffer is released once its receivers have read it
    for (int r = 0; r < G; ++r) {
        const long long ack = 1;
        if (r == me) {
            if (dist_vbuf_) {
                for (int q = 0; q < G; ++q) {
                    if (q == me || (final_stage && q != 0)) continue;
                    long long a = 0;
                    if (dist_->recv(dist_->user, q, &a, sizeof a)) fail();
                }
                CK(cudaFree(dist_vbuf_));
                dist_vbuf_ = nullptr;
            }
        } else if (mode(msgs[r]) == 1) {
            if (dist_->send(dist_->user, r, &ack, sizeof ack)) fail();
        }
    }
    if (ecl >= 0) throw SingularFrontError(ecl, why);
    out_.dist_exchange_s += now_s() - t0;
}

DeviceFactorization Engine::run() {  // factorize.cpp:745-790
    for (int k = L_ + 1; k >= 1; --k) {
        StageStats st;
        st.stage = k;
        cur_stage_ = k;
        sprof_.emplace_back();
        sprof_.back().stage = k;
        const HostProf before = prof_;
        double t0 = now_s();
        if (dist_stage(k)) {
            // a split stage: every rank eliminates its own subtree's clusters; the top-separator
            // fronts they share are re-merged after every stage, and at the last split stage the
            // other subtrees' state goes to rank 0 (a rank whose elimination fails still reports)
            if (k == L_ + 1) dist_partition_state();
            start_rows_.assign(fr_.size(), std::vector<int>());
            for (size_t c = 0; c < fr_.size(); ++c)
                if (dist_top_[c] && alive_[c] && fr_[c].live) start_rows_[c] = fr_[c].rows;
            dist_touched_.clear();
            dist_tr_.clear();
            int ecl = -1;
            std::string why;
            try {
                eliminate_stage(k);
            } catch (const SingularFrontError& e) {
                ecl = e.cluster;
                why = e.reason;
            }
            dist_tseg_.emplace_back(k, out_.trailing_rows.size());
            dist_exchange(k, ecl, why);
            if (k == dist_kend_) {  // the rest runs on rank 0
                if (dist_->rank != 0) {
                    out_.dist_partial = true;
                    break;
                }
#ifdef _OPENMP
                if (const char* s = std::getenv("SPQR_HOST_THREADS_ROOT"))  // alone on the host now
                    if (std::atoi(s) > 0) omp_set_num_threads(std::atoi(s));
#endif
            }
        } else {
            eliminate_stage(k);
        }
        st.t_eliminate = now_s() - t0;
        digest(0);
        if (opt_.eps > 0.0 && k >= 2 && L_ + 1 - k >= opt_.skip_levels) {
            t0 = now_s();
            batch_ = out_.nbatches++;
            scale_all();
            st.t_scale = now_s() - t0;
            notify("scale", -1);
            t0 = now_s();
            sparsify_rows_all();
            notify("sparsify_rows", -1);
            batch_ = out_.nbatches++;
            sparsify_cols_all();
            st.t_sparsify = now_s() - t0;
            notify("sparsify_cols", -1);
        }
        snapshot(st);
        if (k >= 2) {
            t0 = now_s();
            merge_level();
            st.t_merge = now_s() - t0;
            notify("merge", -1);
        }
        st.nnz_w = out_.nnz_w();
        out_.stages.push_back(st);
        for (int i = 0; i < HostProf::N; ++i) sprof_.back().t[i] = prof_.t[i] - before.t[i];
    }
    if (!out_.dist_partial)
        for (size_t c = 0; c < fr_.size(); ++c)
            if (alive_[c] && fr_[c].live) out_.trailing_rows.insert(out_.trailing_rows.end(), fr_[c].rows.begin(), fr_[c].rows.end());
    for (size_t c = 0; c < fr_.size(); ++c) dfree(fr_[c].mat, fr_[c].big);
    sync();
    out_.ctr.t_qr_ms = out_.ctr.k_ms[K_QR];
    if (std::getenv("SPQR_PROF")) {
        for (int i = 0; i < HostProf::N; ++i)
            std::fprintf(stderr, "[spqr prof] %-14s %8.3f s  (%lld)\n", HostProf::name(i), prof_.t[i], prof_.n[i]);
        for (auto& p : nprof_.v) std::fprintf(stderr, "[spqr prof]   %-28s %8.3f s\n", p.first, p.second);
        std::fprintf(stderr, "[spqr prof] per stage:");
        for (int i = 0; i < HostProf::N; ++i) std::fprintf(stderr, " %s", HostProf::name(i));
        std::fprintf(stderr, "\n");
        for (auto& sp : sprof_) {
            std::fprintf(stderr, "[spqr prof] stage %2d", sp.stage);
            for (int i = 0; i < HostProf::N; ++i) std::fprintf(stderr, " %6.3f", sp.t[i]);
            std::fprintf(stderr, "\n");
        }
        for (auto& sp : sprof_)
            std::fprintf(stderr,
                         "[spqr prof] stage %2d waves %3d scol_waves %3d elims %6lld S_elems %10lld S_max %lldx%lld | "
                         "mat fronts %7lld rows %9lld elems %11lld max %lldx%lld\n",
                         sp.stage, sp.waves, sp.scol_waves, sp.elims, sp.s_elems, sp.s_max_rows, sp.s_max_cols, sp.mat_fronts,
                         sp.mat_rows, sp.mat_elems, sp.max_front_rows, sp.max_front_cols);
        for (int t = 0; t < K_NTAGS; ++t)
            std::fprintf(stderr, "[spqr prof] kernel %-9s %8.2f ms %6lld launches %10.1f MB\n", ktag_name(t), out_.ctr.k_ms[t],
                         out_.ctr.k_launches[t], out_.ctr.k_bytes[t] / 1e6);
        static const char* rn[5] = {"narrow", "coop", "tall", "smem+large", "cluster"};
        for (int r = 0; r < 5; ++r)
            std::fprintf(stderr, "[spqr prof] cpqr route %-10s %8.2f ms %6lld launches %8.0f problems\n", rn[r],
                         out_.ctr.route_ms[r], out_.ctr.route_launches[r], out_.ctr.route_probs[r]);
    }
    return std::move(out_);
}

}  // namespace

void sampler_start();
void sampler_stop();

DeviceFactorization gpu_factorize(const Csc& A, const ClusterHierarchy& h, const std::vector<int>& owner,
                                  const FactorizeOptions& opt, cudaStream_t st, const FactorizeObserver* obs) {
    if (A.m < A.n) throw std::invalid_argument("matrix must have at least as many rows as columns");
    if (static_cast<Index>(owner.size()) != A.m) throw std::invalid_argument("row_owner size mismatch");
    sampler_start();
    static const bool prof = std::getenv("SPQR_PROF") != nullptr;
    const double t0 = now_s();
    DeviceFactorization F;
    double t1 = 0, t2 = 0;
    {
        Engine e(A, h, owner, opt, st, obs);
        t1 = now_s();
        F = e.run();
        t2 = now_s();
    }
    if (prof)
        std::fprintf(stderr, "[spqr prof] engine construct %.3f s  run %.3f s  teardown %.3f s\n", t1 - t0, t2 - t1,
                     now_s() - t2);
    sampler_stop();
    return F;
}

}  // namespace spqr
