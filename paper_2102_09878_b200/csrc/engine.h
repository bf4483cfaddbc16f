// GPU factorization engine: Algorithm 1 of spaQR (proj/src/factorize.cpp) with
// every FP64 front in HBM and one batched launch per phase per stage.
#pragma once

#include <cuda_runtime.h>

#include <functional>
#include <memory>
#include <vector>

#include "devmem.h"
#include "spqr.h"

namespace spqr {

// One factor of W (transforms.h:16-30) held on the device.
struct DevWFactor {
    int kind = 0;         // 0 TriangularScale ([R | C]), 1 ColumnRotation (V, tau, sign)
    int batch = 0;        // factors of one batch act on mutually independent column sets
    int cluster = -1;     // cluster whose step produced the factor
    int c = 0, k = 0;     // |cols|; |coupled| (kind 0) or reflector count (kind 1)
    long long cols_off = 0, coupled_off = 0;  // into DeviceFactorization::idx
    double* a = nullptr;  // kind 0: c x (c+k), ld c.  kind 1: V c x k, ld c
    double* tau = nullptr;
    double* sign = nullptr;
    bool scale_only = false;  // kind 0 from scale_all: no coupling, C is the empty 0 x 0 block (factorize.cpp:479-482)
};

enum KTag { K_ASSEMBLE = 0, K_STATS, K_QR, K_TRSM, K_CPQR, K_SCATTER, K_NTAGS };
inline const char* ktag_name(int t) {
    static const char* n[K_NTAGS] = {"assemble", "stats", "front_qr", "trsm", "cpqr", "scatter"};
    return n[t];
}

struct EngineCounters {
    double k_ms[K_NTAGS] = {0};       // device time per kernel family (CUDA events on the engine stream)
    double k_bytes[K_NTAGS] = {0};    // algorithmic HBM bytes (read + write) per kernel family
    long long k_launches[K_NTAGS] = {0};
    long long launches = 0, syncs = 0, h2d_bytes = 0, d2h_bytes = 0;
    double qr_flops = 0, qr_bytes = 0, cpqr_flops = 0, cpqr_bytes = 0;  // algorithmic work (SURVEY 8(d) formulas)
    double cpqr_redundant_flops = 0, cpqr_redundant_bytes = 0;         // discarded speculative sparsify_cols work
    double t_qr_ms = 0;  // device time of the batched front-QR launches (CUDA events)
    long long qr_launches = 0;
    long long elim_waves = 0;  // dependency waves of eliminations summed over stages
    double route_ms[5] = {0}, route_probs[5] = {0};  // CPQR by route: narrow, coop, tall, smem+large, cluster
    long long route_launches[5] = {0};
};

// Subtree-split accounting (FactorizeOptions::ranks > 1): per stage, the
// algorithmic flops of the work each rank would own (eliminations, scaling QR, CPQR) and
// the bytes that would cross ranks, by phase: 0 stack gathers / scatter-backs of rows held by
// another rank's front, 1 R_p shipped to holders on other ranks (scale_all's B_m R_p^-1),
// 2 holder blocks gathered into G and written back (sparsify_cols), 3 fronts moved to a
// parent owned by another rank (merge; the top levels gather onto rank 0).
struct RankStats {
    int ranks = 0;
    std::vector<int> owner;                      // per cluster
    std::vector<std::vector<double>> flops;      // [stage position][rank]
    std::vector<std::vector<double>> cross;      // [stage position][phase]
};

// The outcome of spaqr_factorize (transforms.h:53-72) with W resident in HBM.
struct DeviceFactorization {
    Index M = 0, N = 0;
    double eps = 0.0;
    std::vector<DevWFactor> W;
    std::vector<int> idx;  // cols / coupled lists of all factors
    std::vector<Index> pivot_row, dropped_rows, trailing_rows;
    std::vector<StageStats> stages;
    std::unique_ptr<DeviceArena> warena;
    // Q (store_q, transforms.h:34-37,57): RowReflect factors as rotations on row ids (kind 1,
    // cols = rows, chronological); q_apply_t walks them forward, q_apply backward
    bool has_q = false;
    std::vector<DevWFactor> Q;
    std::vector<int> qidx;
    std::unique_ptr<DeviceArena> qarena;
    int nbatches = 0;
    EngineCounters ctr;
    RankStats rank;
    // distributed factorization: on ranks > 0 the result stops after the split stages, whose
    // subtree was sent to rank 0 (which holds the whole factorization)
    bool dist_partial = false;
    double dist_exchange_s = 0.0;   // time in the split stages' exchanges (export / receive + import)
    long long dist_bytes = 0;       // host-transport bytes sent + received, plus value bytes read over peer memory
    long long nnz_w() const;
};

// Read-only engine state handed to an observer after each phase (EngineView,
// factorize.h:31-36), materialised on the host: every live front's rows and key blocks
// (column-major nrows x width each, keys ascending), the active columns per cluster and the
// row accounting.  The GPU engine eliminates a stage in dependency waves, so one
// "eliminate" notification covers a whole wave (`wave`, ascending; detail = its first id).
struct EngineView {
    std::vector<int> front_cluster, rows_ptr{0}, rows, keys_ptr{0}, keys, key_width;
    std::vector<long long> block_off;
    std::vector<double> values;
    std::vector<int> cols_ptr{0}, cols;
    std::vector<int> wave;
    long long pivots = 0, dropped = 0, trailing = 0;
};
// FactorizeObserver::on_phase (factorize.h:40-43): phase is "eliminate", "scale",
// "sparsify_rows", "sparsify_cols" or "merge".
using FactorizeObserver = std::function<void(const char* phase, int stage, int detail, const EngineView& v)>;

DeviceFactorization gpu_factorize(const Csc& A, const ClusterHierarchy& h, const std::vector<int>& owner,
                                  const FactorizeOptions& opt, cudaStream_t st, const FactorizeObserver* obs = nullptr);

}  // namespace spqr
