// Host orchestration of the level-by-level generalized LDL^T (the hot path)
// and the C ABI of libh2ldl.so (include/h2ldl.h).
//
// Algorithm: the reference engine `_Engine` (gldl.py:179-602), re-expressed
// as a sequence of batched device launches.  For one wave of s shifts the
// engine keeps, per cluster of the current level, s-batched device blocks:
//   diag[i]  m_i x m_i          (gldl.py:229-256)
//   offd(i,j) m_i x m_j  i<j    dense near field / deferred pairs
//   coup(i,j) rS_i x rS_j       skeleton couplings of low-rank pairs
//   fill(i,j) m_i x m_j         fill-in created by elimination
// and walks the reference's schedule: per level, clusters ascending:
// recompress(i) -> eliminate(i); fold fills into couplings; merge to
// parents; BK of the root.  Every step is one or a few launches over all
// blocks it touches and all shifts of the wave.
//
// Shift batching (north star (b)): the structure (which blocks exist and
// their dimensions) is shared by all shifts of a wave.  The only
// data-dependent structure is the recompression rank t; the wave uses
// t = max over its shifts, each shift rotating with its own reflectors -
// a shift then keeps >= the directions the reference keeps, i.e. it is at
// least as accurate, and the inertia is unchanged for shifts farther than
// the construction tolerance from the spectrum.
//
// Live-row rule: a partner eliminated earlier in the level only contributes
// its skeleton rows to the panel and only its skeleton rows are updated -
// the reference carries its (exactly zero) redundant rows through the
// products (gldl.py:365-409); skipping them changes no value.
#include <algorithm>
#include <unordered_map>
#include <chrono>
#include <cmath>
#include <cstdio>
#include <cstring>
#include <map>
#include <mutex>
#include <memory>
#include <thread>
#include <set>
#include <stdexcept>
#include <string>
#include <vector>

#include "common.cuh"
#include "host_util.h"

namespace h2l {

using Pair = std::pair<int, int>;



static inline int64_t pad4(int64_t v) { return (v + 3) / 4 * 4; }
void launch_pack_counts(const int64_t *counts, const int *status, int64_t *out, int s, cudaStream_t st);

// s-batched device block (row-major, ld = cols)
struct Blk {
    double *p = nullptr;
    int rows = 0, cols = 0;
    int64_t bs = 0;
    double *at(int r, int c) const { return p + (int64_t)r * cols + c; }
};

// linear host(pinned)->device staging of task lists; reset at stream syncs
struct Staging {
    char *h = nullptr, *d = nullptr;
    size_t cap = 0, off = 0;
    void init(size_t bytes) {
        cap = bytes;
        CK(cudaMallocHost(&h, cap));
        CK(cudaMalloc(&d, cap));
    }
    void release() {
        if (h) cudaFreeHost(h);
        if (d) cudaFree(d);
        h = d = nullptr;
    }
};

struct Cl {
    int m = 0, nR = 0, nS = 0, r0 = 0;
};

class Wave {
public:
    explicit Wave(int device) : dev_(device) {
        CK(cudaSetDevice(dev_));
        cudaDeviceProp prop;
        CK(cudaGetDeviceProperties(&prop, dev_));
        if (prop.major < 10) throw CudaFail(H2L_ENODEV, "device is not sm_100 class");
        CK(cudaStreamCreateWithFlags(&st_, cudaStreamNonBlocking));
        // private stream-ordered pool per wave: blocks never migrate between the
        // streams of concurrent waves
        cudaMemPoolProps props{};
        props.allocType = cudaMemAllocationTypePinned;
        props.location.type = cudaMemLocationTypeDevice;
        props.location.id = dev_;
        CK(cudaMemPoolCreate(&pool_, &props));
        uint64_t thr = UINT64_MAX;
        CK(cudaMemPoolSetAttribute(pool_, cudaMemPoolAttrReleaseThreshold, &thr));
        stage_.init(size_t(64) << 20);
        for (int k = 0; k < 2; ++k) CK(cudaEventCreate(&ev_call_[k]));
    }
    ~Wave() {
        cudaSetDevice(dev_);
        cudaStreamSynchronize(st_);
        free_payload();
        for (auto &e : ev_pool_) cudaEventDestroy(e);
        for (int k = 0; k < 2; ++k) cudaEventDestroy(ev_call_[k]);
        stage_.release();
        cudaStreamDestroy(st_);
        cudaMemPoolDestroy(pool_);
    }

    // pool high-water mark (reset at the start of each call)
    void reset_mem_high() {
        uint64_t z = 0;
        CK(cudaMemPoolSetAttribute(pool_, cudaMemPoolAttrReservedMemHigh, &z));
    }
    double mem_high() {
        uint64_t v = 0;
        CK(cudaMemPoolGetAttribute(pool_, cudaMemPoolAttrReservedMemHigh, &v));
        return (double)v;
    }
    void set_option(const std::string &k, int64_t v) {
        if (k == "max_batch") max_batch_ = (int)std::max<int64_t>(1, v);
        else if (k == "time_kernels") time_kernels_ = (int)v;  // 0 off, 1 every kind, 2 Schur only
        else if (k == "borrow_arena") borrow_arena_ = v != 0;
        else if (k == "elim_order") elim_order_ = (int)v;
        else if (k == "qr_budget") qr_budget_ = v != 0;
        else if (k == "block_cache") block_cache_ = (int)std::max<int64_t>(0, std::min<int64_t>(2, v));
        else if (k == "block_classes") block_classes_ = v != 0;
        else if (k == "block_cache_mb") bcache_cap_ = std::max<int64_t>(0, v) << 20;
        else if (k == "schedule") schedule_ = (int)std::max<int64_t>(0, std::min<int64_t>(3, v));
        else if (k == "window") window_ = (int)std::max<int64_t>(1, v);
        else if (k == "group_mem_mb") group_mem_mb_ = std::max<int64_t>(1, v);
        else if (k == "group_max") group_max_ = (int)std::max<int64_t>(1, v);
        else if (k == "schur_arith") schur_arith_ = v == 1 ? 1 : 0;
        else throw CudaFail(H2L_EINVAL, "unknown option " + k);
    }

    // ------------------------------------------------------------------ upload
    void upload(const h2l_plan *pl) {
        CK(cudaSetDevice(dev_));
        free_payload();
        if (!pl || pl->n <= 0 || pl->depth < 0 || pl->depth > 30)
            throw CudaFail(H2L_EINVAL, "invalid plan header");
        n_ = pl->n;
        depth_ = pl->depth;
        kind_ = pl->kind;
        eps_ = pl->eps;
        scale0_ = pl->scale0;
        const int nodes = (1 << (depth_ + 1)) - 1;
        ranges_.assign(pl->ranges, pl->ranges + 2 * nodes);
        brank_.assign(pl->basis_rank, pl->basis_rank + nodes);
        bdim_.assign(pl->basis_dim, pl->basis_dim + nodes);
        boff_.assign(pl->basis_off, pl->basis_off + nodes);
        dense_.clear();
        for (int e = 0; e < pl->n_dense; ++e) dense_.push_back({pl->dense[2 * e], pl->dense[2 * e + 1]});
        lowrank_.clear();
        deferred_.clear();
        coup_off_.clear();
        for (int e = 0; e < pl->n_lowrank; ++e) {
            int l = pl->lowrank[3 * e], i = pl->lowrank[3 * e + 1], j = pl->lowrank[3 * e + 2];
            lowrank_[l].push_back({i, j});
            coup_off_[{l, i * 1000003LL + j}] = pl->lowrank_off[e];
        }
        for (int e = 0; e < pl->n_deferred; ++e)
            deferred_[pl->deferred[3 * e]].push_back({pl->deferred[3 * e + 1], pl->deferred[3 * e + 2]});
        cudaPointerAttributes pa{};
        const bool on_device = cudaPointerGetAttributes(&pa, pl->arena) == cudaSuccess &&
                               pa.type == cudaMemoryTypeDevice && pa.device == dev_;
        cudaGetLastError();
        if (borrow_arena_ && on_device) {
            // "borrow_arena": the caller's device arena is used in place and must
            // outlive the engine (the Python layer keeps the device-built H alive)
            arena_ = const_cast<double *>(pl->arena);
            owns_arena_ = false;
        } else {
            CK(cudaMalloc(&arena_, sizeof(double) * std::max<int64_t>(1, pl->arena_len)));
            owns_arena_ = true;
            // host or device arena (unified addressing); stream-ordered on st_ and
            // synced before any kernel reads it
            CK(cudaMemcpyAsync(arena_, pl->arena, sizeof(double) * pl->arena_len, cudaMemcpyDefault,
                               st_));
            CK(cudaStreamSynchronize(st_));
        }
        const int L = depth_;
        const int nleaf = 1 << L;
        // ---- skeleton prologue (K1): S = Q^T A Q, shift independent (compress.py:99-127)
        int64_t tot = 0;
        std::vector<int64_t> doff(nleaf), ooff(dense_.size());
        for (int i = 0; i < nleaf; ++i) { doff[i] = tot; tot += pad4((int64_t)lsize(i) * lsize(i)); }
        for (size_t e = 0; e < dense_.size(); ++e) {
            ooff[e] = tot;
            tot += pad4((int64_t)lsize(dense_[e].first) * lsize(dense_[e].second));
        }
        CK(cudaMalloc(&skel_, sizeof(double) * std::max<int64_t>(1, tot)));
        skel_diag_.assign(nleaf, nullptr);
        skel_off_.clear();
        // batched congruences: up to CH blocks per pair of grouped GEMM launches
        // (tmp_q = Q_a^T A_q, then S_q = tmp_q Q_b), identity bases as copies
        struct Cg { const double *A; int ra, cb; const double *Qa, *Qb; double *C; };
        std::vector<Cg> jobs;
        for (int i = 0; i < nleaf; ++i) {
            skel_diag_[i] = skel_ + doff[i];
            const int m = lsize(i);
            if (m) jobs.push_back({arena_ + pl->diag_off[i], m, m, leaf_basis(i), leaf_basis(i), skel_diag_[i]});
        }
        for (size_t e = 0; e < dense_.size(); ++e) {
            const int i = dense_[e].first, j = dense_[e].second;
            double *dst = skel_ + ooff[e];
            skel_off_[dense_[e]] = dst;
            jobs.push_back({arena_ + pl->dense_off[e], lsize(i), lsize(j), leaf_basis(i), leaf_basis(j), dst});
        }
        int64_t blk = 1;
        for (auto &q : jobs) blk = std::max<int64_t>(blk, pad4((int64_t)q.ra * q.cb));
        const int CH = (int)std::max<int64_t>(1, std::min<int64_t>(1024, (int64_t(1) << 28) / blk));
        double *tmp = nullptr;
        CK(cudaMalloc(&tmp, sizeof(double) * blk * std::min<size_t>(CH, jobs.size() + 1)));
        const int s_save = s_;
        s_ = 1;
        for (size_t q0 = 0; q0 < jobs.size(); q0 += CH) {
            const size_t q1 = std::min(jobs.size(), q0 + CH);
            GemmBatch g1, g2;
            CopyBatch c1, c2;
            for (size_t q = q0; q < q1; ++q) {
                const Cg &jb = jobs[q];
                double *t = tmp + (int64_t)(q - q0) * blk;
                const double *left = jb.A;
                if (jb.Qa) {
                    add_gemm(g1, gm(jb.Qa, 0, jb.ra, 1, jb.A, 0, jb.cb, 0, t, 0, jb.cb, jb.ra, jb.cb,
                                    jb.ra, 1.0, 0.0), 1);
                    left = t;
                }
                if (jb.Qb)
                    add_gemm(g2, gm(left, 0, jb.cb, 0, jb.Qb, 0, jb.cb, 0, jb.C, 0, jb.cb, jb.ra, jb.cb,
                                    jb.cb, 1.0, 0.0), 1);
                else if (jb.Qa)
                    add_copy(c2, cp(left, 0, jb.cb, jb.C, 0, jb.cb, jb.ra, jb.cb));
                else
                    add_copy(c1, cp(jb.A, 0, jb.cb, jb.C, 0, jb.cb, jb.ra, jb.cb));
            }
            flush(c1);
            flush(g1, 1);
            flush(g2, 1);
            flush(c2);
        }
        s_ = s_save;
        CK(cudaStreamSynchronize(st_));
        stage_.off = 0;
        cudaFree(tmp);
        uploaded_ = true;
    }

    // share the uploaded payload of `o` (read-only; `o` keeps ownership)
    void adopt(const Wave &o) {
        CK(cudaSetDevice(dev_));
        free_payload();
        n_ = o.n_; depth_ = o.depth_; kind_ = o.kind_; eps_ = o.eps_; scale0_ = o.scale0_;
        ranges_ = o.ranges_; boff_ = o.boff_; brank_ = o.brank_; bdim_ = o.bdim_;
        dense_ = o.dense_; lowrank_ = o.lowrank_; deferred_ = o.deferred_; coup_off_ = o.coup_off_;
        arena_ = o.arena_; skel_ = o.skel_; skel_diag_ = o.skel_diag_; skel_off_ = o.skel_off_;
        max_batch_ = o.max_batch_; time_kernels_ = o.time_kernels_; schedule_ = o.schedule_; window_ = o.window_; group_mem_mb_ = o.group_mem_mb_; group_max_ = o.group_max_; elim_order_ = o.elim_order_; qr_budget_ = o.qr_budget_; block_cache_ = o.block_cache_; block_classes_ = o.block_classes_; bcache_cap_ = o.bcache_cap_; schur_arith_ = o.schur_arith_;
        owns_payload_ = false;
        uploaded_ = o.uploaded_;
    }
    cudaStream_t stream() const { return st_; }
    // after an exception inside a call: drop every working block and per-wave buffer
    // (errors are swallowed: a sticky CUDA error leaves nothing to recover)
    void abort_cleanup() {
        cudaSetDevice(dev_);
        cudaStreamSynchronize(st_);
        cudaGetLastError();
        const bool in_arena = !guard_mode() && !barena_.slabs.empty();
        auto drop = [&](Blk &b) {
            if (b.p && !(in_arena && barena_.live.count((char *)b.p)))
                cudaFreeAsync(guard_mode() ? b.p - GUARD : b.p, st_);
            b = Blk{};
        };
        for (auto &b : diag_) drop(b);
        for (auto &kv : offd_) drop(kv.second);
        for (auto &kv : coup_) drop(kv.second);
        for (auto &kv : fill_) drop(kv.second);
        diag_.clear(); offd_.clear(); coup_.clear(); fill_.clear();
        live_.clear();
        for (auto &kv : bcache_)
            for (double *p : kv.second) cudaFreeAsync(p, st_);
        bcache_.clear();
        bcache_bytes_ = 0;
        arena_release_all(false);
        release_oz_scratch();
        for (void *p : {(void *)d_mu_, (void *)d_tol_, (void *)d_dropped_, (void *)d_counts_,
                        (void *)d_status_, (void *)d_rank_})
            if (p) cudaFreeAsync(p, st_);
        d_mu_ = d_tol_ = d_dropped_ = nullptr;
        d_counts_ = nullptr;
        d_status_ = d_rank_ = nullptr;
        cudaStreamSynchronize(st_);
        cudaGetLastError();
        stage_.off = 0;
        st_acc_ = nullptr;
        nc_ = 0;
        offp_.clear(); fillp_.clear(); pendf_.clear();
    }
    int max_batch() const { return max_batch_; }
    // run one wave (<= max_batch shifts) and accumulate into acc (stream-ordered, synchronous)
    // dev_out (nullable): device rows [s][4] = (neg, zero, pos, status) instead of the
    // host counts / status (h2l_inertia_device)
    void run(const double *mu, int s, int64_t *counts, int32_t *status, h2l_stats &acc,
             int64_t *dev_out = nullptr) {
        if (!uploaded_) throw CudaFail(H2L_ESTATE, "h2l_inertia before h2l_upload");
        CK(cudaSetDevice(dev_));
        run_wave(mu, s, counts, status, acc, dev_out);
    }

    std::string err;

private:
    bool owns_payload_ = true, owns_arena_ = true, borrow_arena_ = false;
    cudaMemPool_t pool_ = nullptr;
    int dev_;
    cudaStream_t st_ = nullptr;
    Staging stage_;
    int max_batch_ = 64;
    int time_kernels_ = 0;
    int elim_order_ = 0;
    int schedule_ = 1;                // 0 one cluster per group, 1 ascending wavefronts, 2 colours,
                                      // 3 colours of consecutive windows of the order
    int window_ = 64;
    int64_t group_mem_mb_ = 8192;     // temporaries of one group's eliminations
    int group_max_ = 512;
    int t_level_max_ = -1;  // largest recompression rank of the current level (-1: none yet)
    bool qr_budget_ = true;
    int schur_arith_ = 1;             // 0 DMMA fp64, 1 (default) INT8 tensor cores, Ozaki slices (k_schur_oz.cu)
    void *oz_scratch_ = nullptr;      // slice buffers of the INT8 Schur update (per wave)
    size_t oz_scratch_cap_ = 0;
    void release_oz_scratch() {
        if (oz_scratch_) cudaFreeAsync(oz_scratch_, st_);
        oz_scratch_ = nullptr;
        oz_scratch_cap_ = 0;
    }
    bool uploaded_ = false;
    cudaEvent_t ev_call_[2];
    std::vector<cudaEvent_t> ev_pool_;
    size_t ev_used_ = 0;
    std::vector<std::pair<int, double>> ev_marks_;  // (event index of start, kind)

    // plan
    int n_ = 0, depth_ = 0, kind_ = 0;
    double eps_ = 0, scale0_ = 0;
    std::vector<int64_t> ranges_, boff_;
    std::vector<int> brank_, bdim_;
    std::vector<Pair> dense_;
    std::map<int, std::vector<Pair>> lowrank_, deferred_;
    std::map<std::pair<int, long long>, int64_t> coup_off_;
    double *arena_ = nullptr, *skel_ = nullptr;
    std::vector<double *> skel_diag_;
    std::map<Pair, double *> skel_off_;

    // per-wave state
    int s_ = 0;
    double *d_mu_ = nullptr, *d_tol_ = nullptr, *d_dropped_ = nullptr;
    int64_t *d_counts_ = nullptr;
    int *d_status_ = nullptr, *d_rank_ = nullptr;
    std::vector<Cl> cl_;
    std::vector<Blk> diag_;
    std::vector<int> tile_map_, seg_of_, seg_start_;
    std::vector<SchurTarget> schur_tbl_;
    std::vector<char> elim_, pend_diag_;
    std::set<Pair> pend_off_;          // pending dense leaf blocks (large levels)
    // flat pair index of the current level (nc_ <= FLAT_MAX): O(1) block lookups
    // for the ~R^2/2 segment pairs of every elimination step
    static constexpr int FLAT_MAX = 2048;
    int nc_ = 0;
    std::vector<Blk *> offp_, fillp_;
    std::vector<char> pendf_;
    int64_t npend_ = 0, npend_diag_ = 0;
    bool flat() const { return nc_ <= FLAT_MAX; }
    size_t pidx(const Pair &k) const { return (size_t)k.first * nc_ + k.second; }
    Blk *off_get(const Pair &k) {
        if (flat()) return offp_[pidx(k)];
        auto it = offd_.find(k);
        return it == offd_.end() ? nullptr : &it->second;
    }
    Blk *fill_get(const Pair &k) {
        if (flat()) return fillp_[pidx(k)];
        auto it = fill_.find(k);
        return it == fill_.end() ? nullptr : &it->second;
    }
    Blk *off_put(const Pair &k, const Blk &b) {
        Blk *p = &(offd_[k] = b);
        if (flat()) offp_[pidx(k)] = p;
        return p;
    }
    Blk *fill_put(const Pair &k, const Blk &b) {
        Blk *p = &(fill_[k] = b);
        if (flat()) fillp_[pidx(k)] = p;
        return p;
    }
    void fill_erase(const Pair &k) {
        fill_.erase(k);
        if (flat()) fillp_[pidx(k)] = nullptr;
    }
    bool pend_has(const Pair &k) const {
        if (flat()) return k.first < nc_ && k.second < nc_ && pendf_[pidx(k)];
        return pend_off_.count(k) != 0;
    }
    bool pend_test_clear(const Pair &k) {
        if (flat()) {
            char &f = pendf_[pidx(k)];
            if (!f) return false;
            f = 0;
            --npend_;
            return true;
        }
        auto it = pend_off_.find(k);
        if (it == pend_off_.end()) return false;
        pend_off_.erase(it);
        --npend_;
        return true;
    }
    std::map<Pair, Blk> offd_, coup_, fill_;
    std::vector<std::set<Pair>> adj_off_, adj_fill_, adj_coup_;
    h2l_stats *st_acc_ = nullptr;

    // ---------------------------------------------------------------- helpers
    static int node(int level, int i) { return (1 << level) - 1 + i; }
    int csize(int level, int i) const {
        const int nd = node(level, i);
        return (int)(ranges_[2 * nd + 1] - ranges_[2 * nd]);
    }
    int lsize(int i) const { return csize(depth_, i); }
    // arena pointer of the square leaf basis or nullptr when Q = I (rank 0)
    const double *leaf_basis(int i) const {
        const int nd = node(depth_, i);
        if (boff_[nd] < 0 || brank_[nd] <= 0) return nullptr;
        return arena_ + boff_[nd];
    }

    void free_payload() {
        if (owns_payload_) {
            if (arena_ && owns_arena_) cudaFree(arena_);
            if (skel_) cudaFree(skel_);
        }
        arena_ = skel_ = nullptr;
        uploaded_ = false;
        owns_payload_ = true;
    }

    // Task lists reach the device through a pinned ring and one H2D copy per
    // launch.  Every array a launch reads is reserved in ONE region: a ring
    // overflow (stream sync + reset, or growth) can only happen before the
    // region is handed out, never between two arrays of the same launch.
    struct StageRegion {
        char *h = nullptr, *d = nullptr;
        size_t n = 0;
    };
    StageRegion stage_begin(size_t nbytes) {
        const size_t bytes = (nbytes + 255) / 256 * 256;
        if (stage_.off + bytes > stage_.cap) {
            sync();
            if (bytes > stage_.cap) {
                stage_.release();
                stage_.init(bytes * 2);
            }
        }
        StageRegion r{stage_.h + stage_.off, stage_.d + stage_.off, nbytes};
        stage_.off += bytes;
        return r;
    }
    void stage_commit(const StageRegion &r) {
        if (r.n) CK(cudaMemcpyAsync(r.d, r.h, r.n, cudaMemcpyHostToDevice, st_));
    }
    const void *stage(const void *src, size_t nbytes) {
        StageRegion r = stage_begin(nbytes);
        std::memcpy(r.h, src, nbytes);
        stage_commit(r);
        return r.d;
    }
    // several host arrays packed into one staged region (16-byte aligned parts)
    struct Pack {
        std::vector<char> h;
        size_t add(const void *p, size_t n) {
            const size_t off = (h.size() + 15) / 16 * 16;
            h.resize(off + n);
            if (n) std::memcpy(h.data() + off, p, n);
            return off;
        }
    };
    // H2L_GEMMSTATS: flop-weighted histogram of Schur GEMM shapes (printed per wave)
    std::map<std::string, double> ghist_;
    static bool gemmstats_on() {
        static const bool on = getenv("H2L_GEMMSTATS") != nullptr;
        return on;
    }
    template <class GB>
    void gemm_hist(const GB &b) {
        if (!gemmstats_on()) return;
        auto bucket = [](int v) { int q = 16; while (q < v) q *= 2; return q; };
        for (auto &t : b.t) {
            char key[64];
            snprintf(key, sizeof key, "M<=%d N<=%d K<=%d", bucket(t.M), bucket(t.N), bucket(t.K));
            ghist_[key] += 2.0 * t.M * t.N * (double)t.K * s_;
        }
        for (auto &t : b.t)
            ghist_["#padded flops"] += 2.0 * ((t.M + 63) / 64 * 64) * ((t.N + 63) / 64 * 64) * (double)t.K * s_;
        ghist_["#launch tiles"] += b.tiles;
        ghist_["#launches"] += 1;
    }
    void gemm_hist_print() {
        if (!gemmstats_on()) return;
        std::vector<std::pair<double, std::string>> v;
        double tot = 0;
        for (auto &kv : ghist_) if (kv.first[0] != '#') { v.push_back({kv.second, kv.first}); tot += kv.second; }
        std::sort(v.rbegin(), v.rend());
        fprintf(stderr, "schur gemm: %.3g flops (%.3g tile-padded), %.0f launches, %.0f tiles (per shift-row)\n",
                tot, ghist_["#padded flops"], ghist_["#launches"], ghist_["#launch tiles"]);
        for (size_t q = 0; q < v.size() && q < 25; ++q)
            fprintf(stderr, "  %-28s %5.1f%%\n", v[q].second.c_str(), 100.0 * v[q].first / tot);
        ghist_.clear();
    }
    // H2L_MEMTRACE: pool usage (current / high-water) at level boundaries
    void memtrace(const char *what, int level) {
        static const bool on = getenv("H2L_MEMTRACE") != nullptr;
        if (!on) return;
        CK(cudaStreamSynchronize(st_));
        uint64_t cur = 0, hi = 0;
        CK(cudaMemPoolGetAttribute(pool_, cudaMemPoolAttrUsedMemCurrent, &cur));
        CK(cudaMemPoolGetAttribute(pool_, cudaMemPoolAttrUsedMemHigh, &hi));
        fprintf(stderr, "memtrace %s level %d: used %.2f GB high %.2f GB\n", what, level, cur / 1e9,
                hi / 1e9);
    }
    void dbg_sync(const char *what = "") {
        if (guard_mode()) {
            CK(cudaStreamSynchronize(st_));
            last_launch_ = what;
            check_guards();
        }
    }
    void sync() {
        const auto t0 = std::chrono::steady_clock::now();
        CK(cudaStreamSynchronize(st_));
        wait_ms_ += std::chrono::duration<double, std::milli>(std::chrono::steady_clock::now() - t0).count();
        stage_.off = 0;
    }
    // H2L_HOSTPROF: host time blocked in stream syncs vs the wave's wall time
    double wait_ms_ = 0.0, host_rec_ms_ = 0.0, host_elim_ms_ = 0.0;
    static bool hostprof_on() {
        static const bool on = getenv("H2L_HOSTPROF") != nullptr;
        return on;
    }
    // H2L_HOSTPROF host-time buckets: 0 pool alloc, 1 pool free, 2 schedule, 3 BK setup,
    // 4 panel segments, 5 panel solve / GEMM task lists, 6 Schur tables (incl. fill creation),
    // 7 Schur staging + launch, 8 compaction, 9 task-list flushes
    double hp_ms_[12] = {};
    long long hp_n_[12] = {};
    int hp_cur_ = -1;
    std::chrono::steady_clock::time_point hp_t_;
    void hp_switch(int k) {   // sequential sections: time since the last switch goes to the last bucket
        if (!hostprof_on()) return;
        const auto now = std::chrono::steady_clock::now();
        if (hp_cur_ >= 0) {
            hp_ms_[hp_cur_] += std::chrono::duration<double, std::milli>(now - hp_t_).count();
            hp_n_[hp_cur_]++;
        }
        hp_cur_ = k;
        hp_t_ = now;
    }
    struct HostTimer {
        Wave *w;
        int k;
        std::chrono::steady_clock::time_point t0;
        HostTimer(Wave *w_, int k_) : w(hostprof_on() ? w_ : nullptr), k(k_) {
            if (w) t0 = std::chrono::steady_clock::now();
        }
        ~HostTimer() {
            if (w) {
                w->hp_ms_[k] += std::chrono::duration<double, std::milli>(std::chrono::steady_clock::now() - t0).count();
                w->hp_n_[k]++;
            }
        }
    };

    // debug (H2L_DEBUG_GUARD): every block gets GUARD doubles of 0xff canary on both
    // sides, checked after every launch by dbg_sync()
    static constexpr int64_t GUARD = 512;
    static bool guard_mode() {
        static const bool g = getenv("H2L_DEBUG_GUARD") != nullptr;
        return g;
    }
    std::map<double *, int64_t> live_;  // interior pointer -> interior doubles
    std::string last_launch_;
    void check_guards() {
        std::vector<unsigned char> buf(sizeof(double) * GUARD);
        for (auto &kv : live_) {
            for (int side = 0; side < 2; ++side) {
                const double *g = side == 0 ? kv.first - GUARD : kv.first + kv.second;
                CK(cudaMemcpy(buf.data(), g, buf.size(), cudaMemcpyDeviceToHost));
                for (size_t q = 0; q < buf.size(); ++q)
                    if (buf[q] != 0xff) {
                        fprintf(stderr, "GUARD %p: %s overwrote %s guard of block %p (+%lld doubles) at byte %zu after [%s]\n",
                                (void *)this, side ? "tail" : "head", side ? "tail" : "head", (void *)kv.first,
                                (long long)kv.second, q, last_launch_.c_str());
                        CK(cudaMemset((void *)g, 0xff, buf.size()));
                        break;
                    }
            }
        }
    }
    // ---- block arena (block_cache = 2, default): working blocks are carved out of large
    // slabs by a best-fit free list with coalescing, on the host.  A config-4 wave makes
    // ~1.7M block allocations and as many frees (every elimination compacts every block
    // of the cluster); through the stream-ordered pool that was half of the wave's wall
    // time.  One stream per wave makes the reuse of a freed range stream-ordered.
    struct Arena {
        static constexpr size_t SLAB = size_t(512) << 20, GRAN = 256;
        std::vector<std::pair<char *, size_t>> slabs;
        std::map<char *, size_t> by_addr;                 // free ranges
        std::set<std::pair<size_t, char *>> by_size;
        std::unordered_map<char *, size_t> live;
        void erase_free(std::map<char *, size_t>::iterator it) {
            by_size.erase({it->second, it->first});
            by_addr.erase(it);
        }
        void add_free(char *p, size_t n) {
            auto nx = by_addr.lower_bound(p);
            if (nx != by_addr.end() && p + n == nx->first) {   // merge with the next range
                n += nx->second;
                auto dead = nx++;
                erase_free(dead);
            }
            if (nx != by_addr.begin()) {                        // merge with the previous one
                auto pv = std::prev(nx);
                if (pv->first + pv->second == p) {
                    p = pv->first;
                    n += pv->second;
                    erase_free(pv);
                }
            }
            by_addr.emplace_hint(nx, p, n);
            by_size.emplace(n, p);
        }
        char *take(size_t n) {                                   // nullptr: no free range fits
            auto it = by_size.lower_bound({n, nullptr});
            if (it == by_size.end()) return nullptr;
            char *p = it->second;
            const size_t have = it->first;
            by_addr.erase(p);
            by_size.erase(it);
            if (have > n) {
                by_addr[p + n] = have - n;
                by_size.emplace(have - n, p + n);
            }
            live[p] = n;
            return p;
        }
        void give(char *p) {
            auto it = live.find(p);
            if (it == live.end()) return;
            const size_t n = it->second;
            live.erase(it);
            add_free(p, n);
        }
    } barena_;
    double *arena_alloc(int64_t nd) {
        const size_t n = ((size_t)nd * sizeof(double) + Arena::GRAN - 1) / Arena::GRAN * Arena::GRAN;
        char *p = barena_.take(n);
        if (!p) {
            // a new slab; its last GRAN bytes are never handed out, so ranges of two slabs
            // are never adjacent and never merge
            HostTimer ht(this, 0);
            size_t want = std::max(n, Arena::SLAB);
            char *base = nullptr;
            cudaError_t e = cudaMallocFromPoolAsync((void **)&base, want + Arena::GRAN, pool_, st_);
            if (e == cudaErrorMemoryAllocation && want > n) {
                cudaGetLastError();
                want = n;
                e = cudaMallocFromPoolAsync((void **)&base, want + Arena::GRAN, pool_, st_);
            }
            CK(e);
            barena_.slabs.emplace_back(base, want + Arena::GRAN);
            barena_.add_free(base, want);
            p = barena_.take(n);
        }
        return (double *)p;
    }
    void arena_release_all(bool throwing = true) {
        for (auto &sl : barena_.slabs) {
            cudaError_t e = cudaFreeAsync(sl.first, st_);
            if (throwing) CK(e);
        }
        barena_ = Arena{};
    }

    Blk alloc(int rows, int cols, bool zero) {
        Blk b;
        b.rows = rows;
        b.cols = cols;
        b.bs = pad4((int64_t)rows * cols);
        if (rows > 0 && cols > 0) {
            if (guard_mode()) {
                double *base;
                const int64_t inner = b.bs * s_;
                CK(cudaMallocFromPoolAsync((void **)&base, sizeof(double) * (inner + 2 * GUARD), pool_, st_));
                CK(cudaMemsetAsync(base, 0xff, sizeof(double) * (inner + 2 * GUARD), st_));
                b.p = base + GUARD;
                live_[b.p] = inner;
            } else if (block_cache_ == 2) {
                b.p = arena_alloc(b.bs * s_);
            } else {
                const int64_t nd = size_class(b.bs * s_);
                auto it = block_cache_ ? bcache_.find(nd) : bcache_.end();
                if (it != bcache_.end() && !it->second.empty()) {
                    b.p = it->second.back();
                    it->second.pop_back();
                    bcache_bytes_ -= nd * (int64_t)sizeof(double);
                } else {
                    HostTimer ht(this, 0);
                    cudaError_t e = cudaMallocFromPoolAsync((void **)&b.p, sizeof(double) * nd, pool_, st_);
                    if (e == cudaErrorMemoryAllocation && bcache_bytes_ > 0) {
                        // the cached free blocks are the only memory this wave can give back
                        cudaGetLastError();
                        flush_block_cache();
                        CK(cudaStreamSynchronize(st_));
                        e = cudaMallocFromPoolAsync((void **)&b.p, sizeof(double) * nd, pool_, st_);
                    }
                    CK(e);
                }
            }
            if (zero) CK(cudaMemsetAsync(b.p, 0, sizeof(double) * b.bs * s_, st_));
        }
        return b;
    }
    void release(Blk &b) {
        if (b.p) {
            if (guard_mode()) {
                CK(cudaStreamSynchronize(st_));
                check_guards();
                live_.erase(b.p);
                CK(cudaFreeAsync(b.p - GUARD, st_));
            } else if (block_cache_ == 2) {
                barena_.give((char *)b.p);
            } else {
                // same-size blocks are re-issued from a host-side free list (one stream:
                // stream order makes reuse safe); the pool call per block costs more
                // host time than the kernels of small fronts
                const int64_t nd = size_class(b.bs * s_), by = nd * (int64_t)sizeof(double);
                if (block_cache_ && bcache_bytes_ + by <= bcache_cap_) {
                    bcache_[nd].push_back(b.p);
                    bcache_bytes_ += by;
                } else {
                    HostTimer ht(this, 1);
                    CK(cudaFreeAsync(b.p, st_));
                }
            }
        }
        b = Blk{};
    }
    // Blocks are allocated in size classes (8 per octave: <= 12.5 % slack) so that the
    // blocks a moving front retires (compaction shrinks every block of an eliminated
    // cluster) are re-issued to the blocks it creates: on config 4 (~1M block
    // allocations per wave) the pool calls were most of the step's host time.
    int64_t bcache_cap_ = int64_t(2) << 30;
    int block_classes_ = 1;
    int64_t size_class(int64_t nd) const {
        if (!block_classes_ || nd <= 64) return nd;
        int lg = 63 - __builtin_clzll((unsigned long long)nd);
        const int64_t step = int64_t(1) << (lg - 3);
        return (nd + step - 1) / step * step;
    }
    std::unordered_map<int64_t, std::vector<double *>> bcache_;
    int64_t bcache_bytes_ = 0;
    int block_cache_ = 2;   // 0 pool call per block, 1 free lists per size class, 2 arena
    void flush_block_cache() {
        for (auto &kv : bcache_)
            for (double *p : kv.second) CK(cudaFreeAsync(p, st_));
        bcache_.clear();
        bcache_bytes_ = 0;
    }

    // -------------------------------------------------- batched task builders
    struct CopyBatch {
        std::vector<CopyTask> t;
        std::vector<int> pre;
        int tiles = 0;
    };
    struct GemmBatch {
        std::vector<GemmTask> t;
        std::vector<int> pre;
        int tiles = 0;
        double flops = 0;
    };

    static void add_copy(CopyBatch &b, const CopyTask &t) {
        const int k = copy_tiles(t.rows, t.cols);
        if (!k) return;
        b.pre.push_back(b.tiles);
        b.t.push_back(t);
        b.tiles += k;
    }
    // dst <- op(src) (rows x cols) ; helpers
    static CopyTask cp(const double *src, int64_t ss, int lds, double *dst, int64_t ds, int ldd,
                       int rows, int cols, int trans = 0, int acc = 0, double alpha = 1.0) {
        CopyTask t{};
        t.src = src; t.dst = dst; t.sstride = ss; t.dstride = ds;
        t.rows = rows; t.cols = cols; t.lds = lds; t.ldd = ldd;
        t.trans = trans; t.acc = acc; t.alpha = alpha;
        return t;
    }
    static CopyTask zero(double *dst, int64_t ds, int ldd, int rows, int cols) {
        return cp(nullptr, 0, 0, dst, ds, ldd, rows, cols);
    }
    void flush(CopyBatch &b, const double *mu = nullptr) {
        if (!b.t.empty()) {
            Pack pk;
            const size_t o1 = pk.add(b.t.data(), sizeof(CopyTask) * b.t.size());
            const size_t o2 = pk.add(b.pre.data(), sizeof(int) * b.pre.size());
            const char *d = (const char *)stage(pk.h.data(), pk.h.size());
            const CopyTask *dt = (const CopyTask *)(d + o1);
            const int *dp = (const int *)(d + o2);
            {
                Timed tm(this, 5);
                launch_copy_prefixed(dt, dp, (int)b.t.size(), b.tiles, s_ ? s_ : 1, mu, st_);
            }
            CK(cudaGetLastError());
            dbg_sync("copy");
            if (st_acc_) st_acc_->launches++;
        }
        b = CopyBatch{};
    }
    static void add_gemm(GemmBatch &b, const GemmTask &t, int nshift) {
        const int k = gemm_tiles(t.M, t.N);
        if (!k) return;
        b.pre.push_back(b.tiles);
        b.t.push_back(t);
        b.tiles += k;
        b.flops += 2.0 * t.M * t.N * (double)t.K * nshift;
    }
    static GemmTask gm(const double *A, int64_t sA, int lda, int tA, const double *B, int64_t sB,
                       int ldb, int tB, double *C, int64_t sC, int ldc, int M, int N, int K,
                       double alpha, double beta) {
        GemmTask t{};
        t.A = A; t.B = B; t.C = C; t.sA = sA; t.sB = sB; t.sC = sC;
        t.M = M; t.N = N; t.K = K; t.lda = lda; t.ldb = ldb; t.ldc = ldc;
        t.tA = tA; t.tB = tB; t.alpha = alpha; t.beta = beta;
        return t;
    }
    cudaEvent_t next_event() {
        if (ev_used_ == ev_pool_.size()) {
            cudaEvent_t e;
            CK(cudaEventCreate(&e));
            ev_pool_.push_back(e);
        }
        return ev_pool_[ev_used_++];
    }
    // kind: 1 = Schur update, 0 = other
    void flush(GemmBatch &b, int nshift, int kind = 0) {
        if (!b.t.empty()) {
            Pack pk;
            const size_t o1 = pk.add(b.t.data(), sizeof(GemmTask) * b.t.size());
            const size_t o2 = pk.add(b.pre.data(), sizeof(int) * b.pre.size());
            size_t o3 = 0;
            const bool map = b.t.size() > 32;  // tile -> task map: one load per CTA instead of a search
            if (map) {
                tile_map_.resize(b.tiles);
                for (size_t q = 0; q < b.t.size(); ++q) {
                    const int e = q + 1 < b.t.size() ? b.pre[q + 1] : b.tiles;
                    std::fill(tile_map_.begin() + b.pre[q], tile_map_.begin() + e, (int)q);
                }
                o3 = pk.add(tile_map_.data(), sizeof(int) * tile_map_.size());
            }
            const char *d = (const char *)stage(pk.h.data(), pk.h.size());
            const GemmTask *dt = (const GemmTask *)(d + o1);
            const int *dp = (const int *)(d + o2);
            const int *dm = map ? (const int *)(d + o3) : nullptr;
            {
                Timed tm(this, kind);
                launch_gemm(dt, dp, (int)b.t.size(), b.tiles, nshift, st_, kind == 1, dm);
                if (kind == 1) gemm_hist(b);
            }
            CK(cudaGetLastError());
            dbg_sync(kind == 1 ? "gemm-schur" : (kind == 2 ? "gemm-rot" : "gemm-panel"));
            if (st_acc_) {
                st_acc_->launches++;
                st_acc_->gemm_flops_exec += b.flops;
                if (kind == 2) st_acc_->flops += b.flops;  // rotations / merges: executed == algorithmic
            }
        }
        b = GemmBatch{};
    }
    cudaEvent_t mark(int kind) {
        ev_marks_.push_back({(int)ev_used_, (double)kind});
        return next_event();
    }
    // kinds: 0 panel GEMMs, 1 Schur GEMM, 2 rotation/merge GEMMs, 3 BK, 4 panel solve,
    //        5 copies, 6 QR (pqr + form)
    struct Timed {
        Wave *w;
        bool on;
        Timed(Wave *w_, int kind)
            : w(w_), on(w_->time_kernels_ == 1 || (w_->time_kernels_ == 2 && kind == 1)) {
            if (on) CK(cudaEventRecord(w->mark(kind), w->st_));
        }
        ~Timed() {
            if (on) cudaEventRecord(w->next_event(), w->st_);
        }
    };

    Blk &pair_block(std::map<Pair, Blk> &store, int a, int b) { return store[{a, b}]; }

    // ------------------------------------------------------------------ wave
    void run_wave(const double *mu, int s, int64_t *counts, int32_t *status, h2l_stats &acc,
                  int64_t *dev_out) {
        const auto wall0 = std::chrono::steady_clock::now();
        wait_ms_ = host_rec_ms_ = host_elim_ms_ = 0.0;
        for (int q = 0; q < 12; ++q) hp_ms_[q] = 0.0, hp_n_[q] = 0;
        s_ = s;
        st_acc_ = &acc;
        ev_used_ = 0;
        ev_marks_.clear();
        std::vector<double> tol(s);
        for (int z = 0; z < s; ++z) tol[z] = eps_ * (scale0_ + std::fabs(mu[z]));
        CK(cudaMallocFromPoolAsync((void **)&d_mu_, sizeof(double) * s, pool_, st_));
        CK(cudaMallocFromPoolAsync((void **)&d_tol_, sizeof(double) * s, pool_, st_));
        CK(cudaMallocFromPoolAsync((void **)&d_dropped_, sizeof(double) * s, pool_, st_));
        CK(cudaMallocFromPoolAsync((void **)&d_counts_, sizeof(int64_t) * 3 * s, pool_, st_));
        CK(cudaMallocFromPoolAsync((void **)&d_status_, sizeof(int) * s, pool_, st_));
        CK(cudaMallocFromPoolAsync((void **)&d_rank_, sizeof(int) * s, pool_, st_));
        CK(cudaMemcpyAsync(d_mu_, stage(mu, sizeof(double) * s), sizeof(double) * s,
                           cudaMemcpyDeviceToDevice, st_));
        CK(cudaMemcpyAsync(d_tol_, stage(tol.data(), sizeof(double) * s), sizeof(double) * s,
                           cudaMemcpyDeviceToDevice, st_));
        CK(cudaMemsetAsync(d_counts_, 0, sizeof(int64_t) * 3 * s, st_));
        CK(cudaMemsetAsync(d_status_, 0, sizeof(int) * s, st_));

        if (depth_ == 0) {
            Blk root = alloc(lsize(0), lsize(0), false);
            CopyBatch c;
            CopyTask t = cp(skel_diag_[0], 0, root.cols, root.p, root.bs, root.cols, root.rows,
                            root.cols);
            t.shift_diag = 1;
            add_copy(c, t);
            flush(c, d_mu_);
            factor_root(root);
            release(root);
        } else {
            assemble_leaf();
            int level = depth_;
            Blk root;
            while (true) {
                process_level(level);
                memtrace("level done", level);
                if (kind_ == H2L_FLAT) {
                    root = merge_flat();
                    break;
                }
                if (level == 1) {
                    root = merge_pairwise(1, true);
                    break;
                }
                merge_pairwise(level, false);
                memtrace("merged", level);
                --level;
            }
            factor_root(root);
            release(root);
            clear_level();
        }
        gemm_hist_print();
        // timings of Schur launches
        std::vector<int64_t> hc(3 * s);
        std::vector<int> hs(s);
        if (dev_out) {
            launch_pack_counts(d_counts_, d_status_, dev_out, s, st_);
            CK(cudaGetLastError());
            st_acc_->launches++;
        } else {
            CK(cudaMemcpyAsync(hc.data(), d_counts_, sizeof(int64_t) * 3 * s, cudaMemcpyDeviceToHost, st_));
            CK(cudaMemcpyAsync(hs.data(), d_status_, sizeof(int) * s, cudaMemcpyDeviceToHost, st_));
        }
        sync();
        for (auto &mk : ev_marks_) {
            float ms = 0.f;
            CK(cudaEventElapsedTime(&ms, ev_pool_[mk.first], ev_pool_[mk.first + 1]));
            const int kd = (int)mk.second;
            if (kd >= 0 && kd < 8) acc.ms_kind[kd] += ms;
            if (kd == 1) acc.ms_schur += ms;
            if (kd == 3) acc.ms_bk += ms;
        }
        if (!dev_out) {
            std::memcpy(counts, hc.data(), sizeof(int64_t) * 3 * s);
            for (int z = 0; z < s; ++z) status[z] = hs[z] ? H2L_SHIFT_SINGULAR : H2L_SHIFT_OK;
        }
        release_oz_scratch();
        arena_release_all();
        for (double *p : {d_mu_, d_tol_, d_dropped_}) CK(cudaFreeAsync(p, st_));
        CK(cudaFreeAsync(d_counts_, st_));
        CK(cudaFreeAsync(d_status_, st_));
        CK(cudaFreeAsync(d_rank_, st_));
        d_mu_ = d_tol_ = d_dropped_ = nullptr;
        d_counts_ = nullptr;
        d_status_ = d_rank_ = nullptr;
        sync();
        if (hostprof_on())
            fprintf(stderr, "hostprof: wave of %d shifts: wall %.1f ms, blocked in syncs %.1f ms, "
                    "host in recompress %.1f ms (incl. syncs), in eliminate %.1f ms\n", s,
                    std::chrono::duration<double, std::milli>(std::chrono::steady_clock::now() - wall0).count(),
                    wait_ms_, host_rec_ms_, host_elim_ms_);
        if (hostprof_on()) {
            static const char *nm[12] = {"pool_alloc", "pool_free", "schedule", "bk_setup", "panel_segs",
                                         "panel_tasks", "schur_tables", "schur_launch", "compaction",
                                         "flushes", "", ""};
            fprintf(stderr, "hostprof buckets (ms, calls):");
            for (int q = 0; q < 10; ++q) fprintf(stderr, " %s %.1f (%lld)", nm[q], hp_ms_[q], hp_n_[q]);
            fprintf(stderr, "\n");
        }
        st_acc_ = nullptr;
    }

    void clear_level() {
        for (auto &b : diag_) release(b);
        for (auto &kv : offd_) release(kv.second);
        for (auto &kv : coup_) release(kv.second);
        for (auto &kv : fill_) release(kv.second);
        diag_.clear();
        offd_.clear();
        coup_.clear();
        fill_.clear();
        flush_block_cache();
    }

    void reset_adjacency(int nclus) {
        nc_ = nclus;
        const size_t nn = flat() ? (size_t)nclus * nclus : 0;
        offp_.assign(nn, nullptr);
        fillp_.assign(nn, nullptr);
        pendf_.assign(nn, 0);
        pend_off_.clear();
        npend_ = 0;
        adj_off_.assign(nclus, {});
        adj_fill_.assign(nclus, {});
        adj_coup_.assign(nclus, {});
        elim_.assign(nclus, 0);
    }

    // load couplings of `level` from the arena into s-batched blocks
    void load_couplings(int level, CopyBatch &c) {
        auto it = lowrank_.find(level);
        if (it == lowrank_.end()) return;
        for (auto &pr : it->second) {
            const int i = pr.first, j = pr.second;
            const int ri = brank_[node(level, i)], rj = brank_[node(level, j)];
            Blk b = alloc(ri, rj, false);
            const int64_t off = coup_off_.at({level, i * 1000003LL + j});
            if (b.p) add_copy(c, cp(arena_ + off, 0, rj, b.p, b.bs, rj, ri, rj));
            coup_[pr] = b;
            adj_coup_[i].insert(pr);
            adj_coup_[j].insert(pr);
        }
    }

    // Leaf blocks are materialised lazily (just before the first elimination that
    // touches them) from the shift-independent skeleton blocks: together with the
    // compaction of eliminated clusters only the moving front is held per shift.
    void assemble_leaf() {
        const int L = depth_, nl = 1 << L;
        clear_level();
        cl_.assign(nl, Cl{});
        diag_.assign(nl, Blk{});
        reset_adjacency(nl);
        pend_diag_.assign(nl, 0);
        npend_diag_ = 0;
        for (int i = 0; i < nl; ++i) {
            const int m = lsize(i);
            if (m == 0) continue;
            const int r = std::max(0, brank_[node(L, i)]);
            cl_[i] = Cl{m, m - r, r, r};
            pend_diag_[i] = 1;
            ++npend_diag_;
        }
        for (auto &pr : dense_) {
            off_put(pr, Blk{});
            if (flat()) pendf_[pidx(pr)] = 1;
            else pend_off_.insert(pr);
            ++npend_;
            adj_off_[pr.first].insert(pr);
            adj_off_[pr.second].insert(pr);
        }
        CopyBatch c;
        load_couplings(L, c);
        flush(c);
    }
    void ensure_diag(int i, CopyBatch &c) {
        if (i >= (int)pend_diag_.size() || !pend_diag_[i]) return;
        pend_diag_[i] = 0;
        --npend_diag_;
        const int m = lsize(i);
        diag_[i] = alloc(m, m, false);
        CopyTask t = cp(skel_diag_[i], 0, m, diag_[i].p, diag_[i].bs, m, m, m);
        t.shift_diag = 1;
        add_copy(c, t);
    }
    void ensure_off(const Pair &pr, CopyBatch &c) {
        if (!pend_test_clear(pr)) return;
        Blk b = alloc(lsize(pr.first), lsize(pr.second), false);
        add_copy(c, cp(skel_off_.at(pr), 0, b.cols, b.p, b.bs, b.cols, b.rows, b.cols));
        off_put(pr, b);
    }
    // every block the recompression and elimination of i can touch
    void ensure_front(int i, CopyBatch &c) {
        if (npend_ == 0 && npend_diag_ == 0) return;
        ensure_diag(i, c);
        std::vector<int> partners;
        for (auto &k : adj_off_[i]) {
            partners.push_back(k.first == i ? k.second : k.first);
            ensure_off(k, c);
        }
        std::sort(partners.begin(), partners.end());
        for (size_t x = 0; x < partners.size(); ++x) {
            ensure_diag(partners[x], c);
            if (npend_)
                for (size_t y = x + 1; y < partners.size(); ++y)
                    ensure_off({partners[x], partners[y]}, c);
        }
    }
    void ensure_all() {
        CopyBatch c;
        for (int i = 0; i < (int)pend_diag_.size(); ++i) ensure_diag(i, c);
        for (auto &pr : dense_) ensure_off(pr, c);
        flush(c, d_mu_);
    }

    // ------------------------------------------------------ elimination schedule
    // Groups of clusters of one level that are eliminated together (one launch
    // per kernel kind for the whole group).  Two clusters may share a group
    // only if their eliminations touch disjoint blocks: with N(i) = {i} and its
    // near-field partners, eliminating i writes diag/offd/fill blocks inside
    // N(i) x N(i) and rotates / compacts the fills of i, so i and i' conflict
    // when N(i) and N(i') intersect or a fill (i, i') exists when the level
    // starts (fills created during the level join two partners of one cluster,
    // which already intersect).  Couplings both may pad are composed on the host.
    //   schedule 0: one cluster per group, ascending (the reference, gldl.py:262-266)
    //               or low-degree first (elim_order 1);
    //   schedule 1: wavefronts of the ascending order's dependency DAG -- every
    //               cluster runs after all earlier conflicting ones, so each
    //               shift factors exactly what the ascending sweep factors;
    //   schedule 2: colour classes of a greedy distance-2 colouring (ascending
    //               first-fit): a re-ordered elimination, far fewer groups.
    std::vector<std::vector<int>> make_schedule(int level) {
        const int nc = 1 << level;
        std::vector<int> order;
        for (int i = 0; i < nc; ++i)
            if (cl_[i].m > 0) order.push_back(i);
        if (elim_order_ == 1)
            std::stable_sort(order.begin(), order.end(), [&](int a, int b) {
                return adj_off_[a].size() + adj_fill_[a].size() < adj_off_[b].size() + adj_fill_[b].size();
            });
        std::vector<std::vector<int>> groups;
        if (schedule_ == 0 || order.size() <= 1) {
            for (int i : order) groups.push_back({i});
            return groups;
        }
        const int W = (nc + 63) / 64;
        std::vector<uint64_t> N((size_t)nc * W, 0), F((size_t)nc * W, 0);
        auto setb = [&](std::vector<uint64_t> &v, int r, int b) { v[(size_t)r * W + (b >> 6)] |= 1ull << (b & 63); };
        for (int i = 0; i < nc; ++i) {
            setb(N, i, i);
            for (auto &k : adj_off_[i]) setb(N, i, k.first == i ? k.second : k.first);
            for (auto &k : adj_fill_[i]) setb(F, i, k.first == i ? k.second : k.first);
        }
        auto inter = [&](const std::vector<uint64_t> &a, int ra, const uint64_t *b) {
            for (int w = 0; w < W; ++w)
                if (a[(size_t)ra * W + w] & b[w]) return true;
            return false;
        };
        std::vector<int> gid(nc, -1);
        if (schedule_ == 1) {
            // wavefront w(i) = 1 + max w(i') over earlier conflicting i'
            std::vector<int> om(nc, -1);  // max wavefront of a processed cluster whose N holds x
            for (int i : order) {
                int w = 0;
                for (int x = 0; x < nc; ++x)
                    if ((N[(size_t)i * W + (x >> 6)] >> (x & 63)) & 1) w = std::max(w, om[x] + 1);
                for (auto &k : adj_fill_[i]) {
                    const int f = k.first == i ? k.second : k.first;
                    if (gid[f] >= 0) w = std::max(w, gid[f] + 1);
                }
                gid[i] = w;
                for (int x = 0; x < nc; ++x)
                    if ((N[(size_t)i * W + (x >> 6)] >> (x & 63)) & 1) om[x] = std::max(om[x], w);
            }
        } else {
            // first-fit colouring: colour c holds the union of its members' N and its
            // members.  Schedule 3 colours consecutive windows of the order separately
            // (groups: window 0's colours, then window 1's, ...): the eliminated clusters
            // stay a moving front, so materialised blocks and fills stay local as in the
            // ascending sweep (schedule 2 spreads them over the whole level at once)
            const int win = schedule_ == 3 ? std::max(1, window_) : (int)order.size();
            int base = 0;
            for (size_t w0 = 0; w0 < order.size(); w0 += win) {
                std::vector<std::vector<uint64_t>> U, Mb;
                const size_t w1 = std::min(order.size(), w0 + win);
                for (size_t q = w0; q < w1; ++q) {
                    const int i = order[q];
                    int c = 0;
                    for (; c < (int)U.size(); ++c)
                        if (!inter(N, i, U[c].data()) && !inter(F, i, Mb[c].data())) break;
                    if (c == (int)U.size()) {
                        U.emplace_back(W, 0);
                        Mb.emplace_back(W, 0);
                    }
                    for (int w = 0; w < W; ++w) U[c][w] |= N[(size_t)i * W + w];
                    Mb[c][i >> 6] |= 1ull << (i & 63);
                    gid[i] = base + c;
                }
                base += (int)U.size();
            }
        }
        int ng = 0;
        for (int i : order) ng = std::max(ng, gid[i] + 1);
        std::vector<std::vector<int>> byg(ng);
        for (int i : order) byg[gid[i]].push_back(i);
        // split a group by the temporaries its eliminations hold at once
        const double budget = (double)group_mem_mb_ * 1048576.0;
        for (auto &g : byg) {
            std::sort(g.begin(), g.end());
            std::vector<int> cur;
            double bytes = 0.0;
            for (int i : g) {
                const Cl &ci = cl_[i];
                double R = ci.nS;
                for (auto &k : adj_off_[i]) R += cl_[k.first == i ? k.second : k.first].m;
                int c = 0;
                for (auto &k : adj_fill_[i]) {
                    const Blk *f = fill_get(k);
                    if (f) c += k.first == i ? f->cols : f->rows;
                }
                const double m = ci.m;
                // panel + products, recompression buffers, and the fills the elimination
                // can create between its partners (upper bound: every partner pair)
                double fills = 0.0;
                {
                    std::vector<int> ps;
                    for (auto &k : adj_off_[i]) ps.push_back(k.first == i ? k.second : k.first);
                    for (size_t x = 0; x < ps.size(); ++x)
                        for (size_t y = x + 1; y < ps.size(); ++y) {
                            const Pair key{std::min(ps[x], ps[y]), std::max(ps[x], ps[y])};
                            if (!off_get(key) && !fill_get(key) && !pend_has(key))
                                fills += (double)cl_[ps[x]].m * cl_[ps[y]].m;
                        }
                }
                const double b = 8.0 * s_ * (2.0 * R * m + 2.0 * (double)c * m + 6.0 * m * m + fills);
                if (!cur.empty() && (bytes + b > budget || (int)cur.size() >= group_max_)) {
                    groups.push_back(cur);
                    cur.clear();
                    bytes = 0.0;
                }
                cur.push_back(i);
                bytes += b;
            }
            if (!cur.empty()) groups.push_back(cur);
        }
        return groups;
    }

    void process_level(int level) {
        const bool leaf = level == depth_;
        t_level_max_ = -1;
        std::vector<std::vector<int>> groups;
        {
            HostTimer ht(this, 2);
            groups = make_schedule(level);
        }
        st_acc_->groups += (int64_t)groups.size();
        for (const auto &g : groups) {
            if (leaf && (npend_ || npend_diag_)) {
                CopyBatch c;
                for (int i : g) ensure_front(i, c);
                flush(c, d_mu_);
            }
            const auto h0 = std::chrono::steady_clock::now();
            recompress_group(g);
            const auto h1 = std::chrono::steady_clock::now();
            eliminate_group(g);
            const auto h2 = std::chrono::steady_clock::now();
            host_rec_ms_ += std::chrono::duration<double, std::milli>(h1 - h0).count();
            host_elim_ms_ += std::chrono::duration<double, std::milli>(h2 - h1).count();
        }
        if (leaf) ensure_all();
        // fold fills of this level's low-rank pairs into the couplings (gldl.py:284-294)
        auto it = lowrank_.find(level);
        if (it != lowrank_.end()) {
            CopyBatch c;
            std::vector<Pair> done;
            for (auto &pr : it->second) {
                Blk *fp = fill_get(pr);
                if (!fp) continue;
                Blk &C = coup_.at(pr);
                Blk &F = *fp;
                const int a = pr.first, b = pr.second;
                const int ra = cl_[a].nR, rb = cl_[b].nR;
                if (C.p)
                    add_copy(c, cp(F.at(ra, rb), F.bs, F.cols, C.p, C.bs, C.cols, C.rows, C.cols, 0, 1));
                done.push_back(pr);
            }
            flush(c);
            for (auto &pr : done) {
                release(*fill_get(pr));
                fill_erase(pr);
                adj_fill_[pr.first].erase(pr);
                adj_fill_[pr.second].erase(pr);
            }
        }
    }

    // ------------------------------------------------------- recompression K7-K9
    void row_transform(const Blk &src, Blk &dst, const double *Tr, int64_t trs, int nR, int nS,
                       int t, GemmBatch &g, CopyBatch &c) {
        // dst rows: [0,newR) = Tr[0:newR] src[0:nR]; [newR,newR+nS) = src[nR:]; [newR+nS,m) = Tr[newR:] src[0:nR]
        const int newR = nR - t, cols = src.cols;
        add_gemm(g, gm(Tr, trs, nR, 0, src.p, src.bs, cols, 0, dst.p, dst.bs, cols, newR, cols, nR,
                       1.0, 0.0), s_);
        add_gemm(g, gm(Tr + (int64_t)newR * nR, trs, nR, 0, src.p, src.bs, cols, 0,
                       dst.at(newR + nS, 0), dst.bs, cols, t, cols, nR, 1.0, 0.0), s_);
        add_copy(c, cp(src.at(nR, 0), src.bs, cols, dst.at(newR, 0), dst.bs, cols, nS, cols));
    }
    void col_transform(const Blk &src, Blk &dst, const double *Tr, int64_t trs, int nR, int nS,
                       int t, GemmBatch &g, CopyBatch &c) {
        // dst cols: [0,newR) = src[:,0:nR] Tr[0:newR]^T ; [newR,newR+nS) = src[:,nR:] ; rest = src[:,0:nR] Tr[newR:]^T
        const int newR = nR - t, rows = src.rows, m = src.cols;
        add_gemm(g, gm(src.p, src.bs, m, 0, Tr, trs, nR, 1, dst.p, dst.bs, m, rows, newR, nR, 1.0,
                       0.0), s_);
        add_gemm(g, gm(src.p, src.bs, m, 0, Tr + (int64_t)newR * nR, trs, nR, 1,
                       dst.at(0, newR + nS), dst.bs, m, rows, t, nR, 1.0, 0.0), s_);
        add_copy(c, cp(src.at(0, nR), src.bs, m, dst.at(0, newR), dst.bs, m, rows, nS));
    }

    // Q^T of the full column-pivoted QR of the n x n Gram matrix M (M is consumed),
    // one cluster: the deflation pass and the fallback beyond distributed shared memory
    void gram_order(Blk &M, int n, Blk &QT, double *tau, int *piv, int *used, double *norms,
                    int64_t ts, const int *d_active, int kmax) {
        if (pqr_cluster_size(n)) {
            CK(launch_pqr_cluster(M.p, M.bs, n, tau, piv, ts, d_active, s_, st_, kmax));
            CK(launch_form_q_rows(M.p, M.bs, n, tau, ts, QT.p, QT.bs, d_active, s_, st_, kmax));
        } else {
            // M is symmetric: its row-major storage is also its "columns as rows" layout
            CK(launch_pqr(M.p, M.bs, n, n, n, tau, piv, used, norms, ts, ts, d_tol_, d_rank_,
                          d_dropped_, d_active, -2, s_, st_));
            // all n reflectors; with t = n form_tr's row map is the identity (QT = Q^T)
            CK(launch_form_tr(M.p, M.bs, n, tau, piv, ts, n, n, QT.p, QT.bs, d_active, s_, st_));
        }
        st_acc_->launches += 2;
    }

    // M (n x n) = A^T A for A = c x n (row stride ld, shift stride sA), one cluster
    void gram(const double *A, int64_t sA, int ld, int n, int c, Blk &M) {
        GemmBatch g;
        add_gemm(g, gm(A, sA, ld, 1, A, sA, ld, 0, M.p, M.bs, n, n, n, c, 1.0, 0.0), s_);
        flush(g, s_, 6);
    }

    // one cluster's recompression state (recompress_group)
    struct RecJob {
        int i = 0, nR = 0, c = 0, kmax = 0, t = 0;
        std::vector<Pair> ks;
        Blk GT, M, QT, DT;
        double *tau = nullptr, *norms = nullptr, *part = nullptr, *P = nullptr;
        int *piv = nullptr, *used = nullptr;
        int parts = 1;
        double dropped = 0.0;
    };

    // Recompression of every cluster of a group (gldl.py:296-347), each kernel
    // kind one launch over all clusters x shifts.  Rank reveal: the reference
    // runs a column-pivoted QR of the fill rows G (n_R x c); here the directions
    // are ordered by a pivoted QR of the Gram matrix M = G G^T (cluster kernel)
    // and the rank is taken from the EXACT energies of D = Q^T G with the
    // reference's tail rule (k_rrqr.cu).  One readback per group decides the
    // ranks (block sizes are host-side structure).
    void recompress_group(const std::vector<int> &grp) {
        std::vector<RecJob> J;
        for (int i : grp) {
            const Cl &ci = cl_[i];
            if (ci.nR == 0 || adj_fill_[i].empty()) continue;
            RecJob j;
            j.i = i;
            j.nR = ci.nR;
            j.ks.assign(adj_fill_[i].begin(), adj_fill_[i].end());
            for (auto &k : j.ks) j.c += (k.first == i) ? fill_get(k)->cols : fill_get(k)->rows;
            J.push_back(std::move(j));
        }
        if (J.empty()) return;
        const int nj = (int)J.size();
        // ---- G^T (c x nR) of every job: row q = column q of G
        {
            CopyBatch cb;
            for (auto &j : J) {
                if (j.c == 0) continue;
                j.GT = alloc(j.c, j.nR, false);
                int q0 = 0;
                for (auto &k : j.ks) {
                    Blk &F = *fill_get(k);
                    if (k.first == j.i) {  // F[:nR, :] -> GT rows = columns of F
                        add_copy(cb, cp(F.p, F.bs, F.cols, j.GT.at(q0, 0), j.GT.bs, j.nR, F.cols, j.nR, 1));
                        q0 += F.cols;
                    } else {               // F[:, :nR]^T -> GT rows = rows of F
                        add_copy(cb, cp(F.p, F.bs, F.cols, j.GT.at(q0, 0), j.GT.bs, j.nR, F.rows, j.nR, 0));
                        q0 += F.rows;
                    }
                }
            }
            flush(cb);
        }
        // per-job rank outputs: ranks [nj][s], r1 [nj][s] (ints), dropped [nj][s]
        int *d_act, *d_ri;
        double *d_rd;
        CK(cudaMallocFromPoolAsync((void **)&d_act, sizeof(int) * s_, pool_, st_));
        CK(cudaMallocFromPoolAsync((void **)&d_ri, sizeof(int) * 2 * nj * s_, pool_, st_));
        CK(cudaMallocFromPoolAsync((void **)&d_rd, sizeof(double) * nj * s_, pool_, st_));
        CK(cudaMemsetAsync(d_ri, 0, sizeof(int) * 2 * nj * s_, st_));
        CK(cudaMemsetAsync(d_rd, 0, sizeof(double) * nj * s_, st_));
        activity_from_status(d_act);
        auto rank_of = [&](int q) { return d_ri + (int64_t)q * s_; };
        auto r1_of = [&](int q) { return d_ri + (int64_t)(nj + q) * s_; };
        auto drop_of = [&](int q) { return d_rd + (int64_t)q * s_; };
        for (auto &j : J) {
            if (j.c == 0) continue;
            const int64_t ts = pad4(j.nR);
            j.M = alloc(j.nR, j.nR, false);
            j.QT = alloc(j.nR, j.nR, false);
            j.DT = alloc(j.c, j.nR, false);
            CK(cudaMallocFromPoolAsync((void **)&j.tau, sizeof(double) * ts * s_, pool_, st_));
            CK(cudaMallocFromPoolAsync((void **)&j.norms, sizeof(double) * ts * s_, pool_, st_));
            CK(cudaMallocFromPoolAsync((void **)&j.piv, sizeof(int) * ts * s_, pool_, st_));
            CK(cudaMallocFromPoolAsync((void **)&j.used, sizeof(int) * ts * s_, pool_, st_));
            CK(cudaMallocFromPoolAsync((void **)&j.part,
                                       sizeof(double) * tail_rank_part_doubles(j.c, j.nR) * s_, pool_, st_));
            // the ordering is budgeted: kmax pivots (1.5x the largest rank this level has
            // needed + 32, all of them for the level's first group); a rank within 8 of the
            // budget redoes the ordering with every pivot.  The leading kmax reflectors of
            // a pivoted QR do not depend on how many follow, so the rank equals the full
            // ordering's; only the (dropped) complement's basis differs.
            j.kmax = (t_level_max_ < 0 || !qr_budget_)
                         ? j.nR : std::min(j.nR, t_level_max_ + std::max(32, t_level_max_ / 2));
        }
        std::vector<int> pend;
        for (int q = 0; q < nj; ++q)
            if (J[q].c > 0) pend.push_back(q);
        std::vector<int> hri(2 * (size_t)nj * s_), hact(s_);
        std::vector<double> hrd((size_t)nj * s_);
        while (!pend.empty()) {
            // ---- M = G G^T = GT^T GT: split-K partial products (one grouped launch) summed
            // in a fixed order (one launch), so small groups still fill the SMs
            {
                int tiles = 0;
                for (int q : pend) tiles += gemm_tiles(J[q].nR, J[q].nR);
                const int want = std::max(1, (2 * 148 * 4 + tiles - 1) / std::max(1, tiles));
                GemmBatch g;
                std::vector<SumJob> sj;
                int64_t maxcount = 0;
                for (int q : pend) {
                    RecJob &j = J[q];
                    const int n = j.nR;
                    int parts = std::max(1, std::min((j.c + 511) / 512, want));
                    const int chunk = (j.c + parts - 1) / parts;
                    parts = (j.c + chunk - 1) / chunk;
                    j.parts = parts;
                    if (parts <= 1) {
                        add_gemm(g, gm(j.GT.p, j.GT.bs, n, 1, j.GT.p, j.GT.bs, n, 0, j.M.p, j.M.bs, n, n, n,
                                       j.c, 1.0, 0.0), s_);
                        continue;
                    }
                    const int64_t ps = pad4((int64_t)n * n);
                    if (!j.P) CK(cudaMallocFromPoolAsync((void **)&j.P, sizeof(double) * ps * parts * s_, pool_, st_));
                    for (int p = 0; p < parts; ++p) {
                        const int k0 = p * chunk, kc = std::min(chunk, j.c - k0);
                        add_gemm(g, gm(j.GT.p + (int64_t)k0 * n, j.GT.bs, n, 1, j.GT.p + (int64_t)k0 * n,
                                       j.GT.bs, n, 0, j.P + p * ps, ps * parts, n, n, n, kc, 1.0, 0.0), s_);
                    }
                    sj.push_back(SumJob{j.P, ps * parts, ps, j.M.p, j.M.bs, (int64_t)n * n, parts, 0});
                    maxcount = std::max<int64_t>(maxcount, (int64_t)n * n);
                }
                flush(g, s_, 6);
                if (!sj.empty()) {
                    const SumJob *dj = (const SumJob *)stage(sj.data(), sizeof(SumJob) * sj.size());
                    Timed tm(this, 6);
                    launch_sum_partials_multi(dj, (int)sj.size(), maxcount, s_, st_);
                    CK(cudaGetLastError());
                    st_acc_->launches++;
                }
            }
            // ---- ordering: pivoted QR of every M (cluster kernel) and Q^T
            {
                std::vector<PqrJob> pj;
                int nmax = 0;
                for (int q : pend) {
                    RecJob &j = J[q];
                    if (!pqr_cluster_size(j.nR)) {
                        st_acc_->paths[3]++;
                        Timed tm(this, 7);
                        gram_order(j.M, j.nR, j.QT, j.tau, j.piv, j.used, j.norms, pad4(j.nR), d_act,
                                   j.kmax);
                        continue;
                    }
                    if (pqr_cluster_size(j.nR) == 16) st_acc_->paths[2]++;
                    pj.push_back(PqrJob{j.M.p, j.M.bs, j.tau, j.piv, pad4(j.nR), j.QT.p, j.QT.bs, j.nR,
                                        j.kmax});
                    nmax = std::max(nmax, j.nR);
                }
                if (!pj.empty()) {
                    const PqrJob *dj = (const PqrJob *)stage(pj.data(), sizeof(PqrJob) * pj.size());
                    Timed tm(this, 7);
                    CK(launch_pqr_cluster_multi(dj, (int)pj.size(), nmax, d_act, s_, st_));
                    CK(launch_form_q_rows_multi(dj, (int)pj.size(), nmax, d_act, s_, st_));
                    st_acc_->launches += 2;
                }
            }
            // ---- D^T = GT Q (Q[k][n] = QT[n][k]) and the exact tail energies
            {
                GemmBatch g;
                for (int q : pend) {
                    RecJob &j = J[q];
                    add_gemm(g, gm(j.GT.p, j.GT.bs, j.nR, 0, j.QT.p, j.QT.bs, j.nR, 1, j.DT.p, j.DT.bs,
                                   j.nR, j.c, j.nR, j.nR, 1.0, 0.0), s_);
                }
                flush(g, s_, 6);
                std::vector<RankJob> rj;
                int cmax = 0, nmax = 0;
                for (int q : pend) {
                    RecJob &j = J[q];
                    rj.push_back(RankJob{j.DT.p, j.DT.bs, j.part, rank_of(q), r1_of(q), drop_of(q), j.c, j.nR});
                    cmax = std::max(cmax, j.c);
                    nmax = std::max(nmax, j.nR);
                }
                const RankJob *dj = (const RankJob *)stage(rj.data(), sizeof(RankJob) * rj.size());
                Timed tm(this, 6);
                CK(launch_tail_rank_multi(dj, (int)rj.size(), cmax, nmax, d_tol_, d_act, s_, st_));
                st_acc_->launches += 2;
            }
            auto readback = [&] {
                CK(cudaMemcpyAsync(hri.data(), d_ri, sizeof(int) * hri.size(), cudaMemcpyDeviceToHost, st_));
                CK(cudaMemcpyAsync(hrd.data(), d_rd, sizeof(double) * hrd.size(), cudaMemcpyDeviceToHost, st_));
                CK(cudaMemcpyAsync(hact.data(), d_act, sizeof(int) * s_, cudaMemcpyDeviceToHost, st_));
                sync();
            };
            readback();
            // ---- deflation pass: the Gram ordering only resolves directions whose
            // energy is above ~1e-16 of the largest; re-order the rest from their own
            // Gram matrix (per cluster; rare).  Skipped when the first pass already drops
            // every direction past r1: the tail sums from any r <= r1 then include the
            // whole (rotation-invariant) energy of that subspace.
            bool defl = false;
            for (int q : pend) {
                RecJob &j = J[q];
                const int nR = j.nR;
                int r1 = nR, t1 = 0;
                for (int z = 0; z < s_; ++z)
                    if (hact[z]) {
                        r1 = std::min(r1, hri[(size_t)(nj + q) * s_ + z]);
                        t1 = std::max(t1, hri[(size_t)q * s_ + z]);
                    }
                const int nT = nR - r1;
                if (!(nT > 1 && t1 > r1)) continue;
                defl = true;
                Blk M2 = alloc(nT, nT, false), Q2T = alloc(nT, nT, false);
                Blk DT2 = alloc(j.c, nT, false), QT2 = alloc(nT, nR, false);
                gram(j.DT.p + r1, j.DT.bs, nR, nT, j.c, M2);  // M2 = D_tail D_tail^T
                {
                    Timed tm(this, 6);
                    gram_order(M2, nT, Q2T, j.tau, j.piv, j.used, j.norms, pad4(nR), d_act,
                               std::min(nT, j.kmax));
                }
                {
                    GemmBatch g;  // DT2 = D_tail^T Q2 ; QT2 = Q2^T QT[r1:, :]
                    add_gemm(g, gm(j.DT.p + r1, j.DT.bs, nR, 0, Q2T.p, Q2T.bs, nT, 1, DT2.p, DT2.bs,
                                   nT, j.c, nT, nT, 1.0, 0.0), s_);
                    add_gemm(g, gm(Q2T.p, Q2T.bs, nT, 0, j.QT.at(r1, 0), j.QT.bs, nR, 0, QT2.p,
                                   QT2.bs, nR, nT, nR, nT, 1.0, 0.0), s_);
                    flush(g, s_, 6);
                }
                CopyBatch cc;
                add_copy(cc, cp(DT2.p, DT2.bs, nT, j.DT.p + r1, j.DT.bs, nR, j.c, nT));
                add_copy(cc, cp(QT2.p, QT2.bs, nR, j.QT.at(r1, 0), j.QT.bs, nR, nT, nR));
                flush(cc);
                {
                    Timed tm(this, 6);
                    CK(launch_tail_rank(j.DT.p, j.DT.bs, j.c, nR, j.part, d_tol_, rank_of(q),
                                        drop_of(q), nullptr, d_act, s_, st_));
                    st_acc_->launches += 2;
                }
                for (Blk *b : {&M2, &Q2T, &DT2, &QT2}) release(*b);
            }
            if (defl) readback();
            std::vector<int> redo;
            for (int q : pend) {
                RecJob &j = J[q];
                j.t = 0;
                j.dropped = 0.0;
                for (int z = 0; z < s_; ++z)
                    if (hact[z]) {
                        j.t = std::max(j.t, hri[(size_t)q * s_ + z]);
                        j.dropped += hrd[(size_t)q * s_ + z];
                    }
                if (j.kmax < j.nR && j.t + 8 >= j.kmax) {
                    j.kmax = j.nR;
                    redo.push_back(q);
                }
            }
            pend.swap(redo);
        }
        for (auto &j : J) {
            if (j.c == 0) continue;
            st_acc_->dropped_fro += j.dropped;
            t_level_max_ = std::max(t_level_max_, j.t);
            st_acc_->recompressions++;
            // algorithmic QR of G (nR x c), survey §8d: 2 c nR^2 - 2/3 nR^3 (for c >= nR)
            const double a = std::max(j.c, j.nR), b = std::min(j.c, j.nR);
            st_acc_->flops += (2.0 * a * b * b - 2.0 / 3.0 * b * b * b) * s_;
        }
        // ---- rotations of every job with t > 0: Tr = [U_r^T ; U_s^T] = QT rows [t, nR) then [0, t)
        std::vector<int> rot;
        for (int q = 0; q < nj; ++q)
            if (J[q].c > 0 && J[q].t > 0) rot.push_back(q);
        if (!rot.empty()) {
            std::vector<Blk> Tr(nj);
            CopyBatch rc;
            for (int q : rot) {
                RecJob &j = J[q];
                Tr[q] = alloc(j.nR, j.nR, false);
                add_copy(rc, cp(j.QT.at(j.t, 0), j.QT.bs, j.nR, Tr[q].p, Tr[q].bs, j.nR, j.nR - j.t, j.nR));
                add_copy(rc, cp(j.QT.p, j.QT.bs, j.nR, Tr[q].at(j.nR - j.t, 0), Tr[q].bs, j.nR, j.t, j.nR));
            }
            flush(rc);
            std::vector<int> ids, ts;
            std::vector<const Blk *> trs;
            for (int q : rot) {
                ids.push_back(J[q].i);
                ts.push_back(J[q].t);
                trs.push_back(&Tr[q]);
            }
            apply_rotations(ids, trs, ts);
            // per-shift truncation: a shift whose own rank r_z < t drops the fill content
            // of directions [r_z, t) as the reference does at that shift (gldl.py:341-347);
            // the directions stay in the skeleton (a congruence: same matrix, same inertia)
            if (s_ > 1) {
                std::vector<TailZeroJob> tz;
                for (int q : rot) {
                    RecJob &j = J[q];
                    const Cl &ci = cl_[j.i];  // already rotated: nR' = nR - t, nS' = nS + t
                    const int base = ci.nR + (ci.nS - j.t);
                    for (auto &k : adj_fill_[j.i]) {
                        Blk *F = fill_get(k);
                        if (!F || !F->p) continue;
                        if (k.first == j.i)
                            tz.push_back(TailZeroJob{F->p, F->bs, rank_of(q), F->cols, F->cols, base, j.t, 0, 0});
                        else
                            tz.push_back(TailZeroJob{F->p, F->bs, rank_of(q), F->cols, F->rows, base, j.t, 1, 0});
                    }
                }
                if (!tz.empty()) {
                    const TailZeroJob *dj = (const TailZeroJob *)stage(tz.data(), sizeof(TailZeroJob) * tz.size());
                    Timed tm(this, 5);
                    CK(launch_tail_zero(dj, (int)tz.size(), s_, st_));
                    st_acc_->launches++;
                }
            }
            for (int q : rot) release(Tr[q]);
        }
        // ---- discard what is left in the redundant rows of the fills (gldl.py:341-347)
        {
            CopyBatch z;
            for (auto &j : J) {
                const int keep = cl_[j.i].nR;
                if (keep == 0) continue;
                for (auto &k : j.ks) {
                    Blk &F = *fill_get(k);
                    if (k.first == j.i) add_copy(z, zero(F.p, F.bs, F.cols, keep, F.cols));
                    else add_copy(z, zero(F.p, F.bs, F.cols, F.rows, keep));
                }
            }
            flush(z);
        }
        for (auto &j : J) {
            for (void *p : {(void *)j.tau, (void *)j.norms, (void *)j.piv, (void *)j.used, (void *)j.part,
                            (void *)j.P})
                if (p) CK(cudaFreeAsync(p, st_));
            for (Blk *b : {&j.M, &j.QT, &j.DT, &j.GT}) release(*b);
        }
        for (void *p : {(void *)d_act, (void *)d_ri, (void *)d_rd}) CK(cudaFreeAsync(p, st_));
    }

    void activity_from_status(int *d_active);

    // Basis rotations of several clusters (gldl.py:313-339): diag, offd, fill rows /
    // columns by T, couplings zero-padded.  The clusters of a group share no offd or
    // fill block; a coupling padded by two of them is padded once to its final size.
    void apply_rotations(const std::vector<int> &ids, const std::vector<const Blk *> &Trs,
                         const std::vector<int> &ts) {
        GemmBatch g1, g2;
        CopyBatch c1, c2;
        std::vector<Blk> Y(ids.size()), Z(ids.size());
        std::vector<std::pair<Blk *, Blk>> repl;
        for (size_t q = 0; q < ids.size(); ++q) {
            const int i = ids[q], t = ts[q];
            const Cl &ci = cl_[i];
            const Blk &Tr = *Trs[q];
            Y[q] = alloc(ci.m, ci.m, false);
            Z[q] = alloc(ci.m, ci.m, false);
            row_transform(diag_[i], Y[q], Tr.p, Tr.bs, ci.nR, ci.nS, t, g1, c1);  // Y = T D
            for (auto *store : {&offd_, &fill_}) {
                auto &adj = (store == &offd_) ? adj_off_[i] : adj_fill_[i];
                for (auto &k : adj) {
                    Blk &B = (store == &offd_) ? *off_get(k) : *fill_get(k);
                    Blk N = alloc(B.rows, B.cols, false);
                    if (k.first == i) row_transform(B, N, Tr.p, Tr.bs, ci.nR, ci.nS, t, g1, c1);
                    else col_transform(B, N, Tr.p, Tr.bs, ci.nR, ci.nS, t, g1, c1);
                    repl.push_back({&B, N});
                }
            }
        }
        flush(g1, s_, 2);
        flush(c1);
        for (size_t q = 0; q < ids.size(); ++q) {
            const int i = ids[q];
            const Cl &ci = cl_[i];
            col_transform(Y[q], Z[q], Trs[q]->p, Trs[q]->bs, ci.nR, ci.nS, ts[q], g2, c2);  // Z = Y T^T
        }
        // couplings: zero-pad by t rows / columns (gldl.py:324-330)
        std::map<Pair, std::pair<int, int>> pads;
        for (size_t q = 0; q < ids.size(); ++q) {
            const int i = ids[q];
            for (auto &k : adj_coup_[i]) {
                auto &pd = pads[k];
                if (k.first == i) pd.first += ts[q];
                else pd.second += ts[q];
            }
        }
        std::vector<std::pair<Blk *, Blk>> crepl;
        for (auto &kv : pads) {
            Blk &C = coup_.at(kv.first);
            Blk N = alloc(C.rows + kv.second.first, C.cols + kv.second.second, true);
            if (C.p && N.p) add_copy(c2, cp(C.p, C.bs, C.cols, N.p, N.bs, N.cols, C.rows, C.cols));
            crepl.push_back({&C, N});
        }
        flush(g2, s_, 2);
        flush(c2);
        for (size_t q = 0; q < ids.size(); ++q) {
            const int i = ids[q];
            release(diag_[i]);
            release(Y[q]);
            diag_[i] = Z[q];
            Cl &ci = cl_[i];
            ci.nR -= ts[q];
            ci.nS += ts[q];
            st_acc_->rank_added += ts[q];
        }
        for (auto &r : repl) { release(*r.first); *r.first = r.second; }
        for (auto &r : crepl) { release(*r.first); *r.first = r.second; }
    }

    // --------------------------------------------------------- elimination K2-K6
    // one row segment of the elimination panel B = [D_SR ; partner slices]
    struct Seg {
        int who, lo, len, row;   // cluster, first live row, live rows, first panel row
        const double *src;       // source block (shift 0)
        int64_t ss;              // shift stride of the source
        int lds, trans, r0;      // panel row r = src row (r0 + r), or column when trans
    };
    // op(segment) as the left operand (len x nR) of a GEMM
    static void seg_as_A(const Seg &g, const double **A, int *lda, int *tA) {
        if (g.trans) { *A = g.src + g.r0; *lda = g.lds; *tA = 1; }
        else { *A = g.src + (int64_t)g.r0 * g.lds; *lda = g.lds; *tA = 0; }
    }

    struct ElimJob {
        int i = 0, nR = 0, nS = 0, m = 0, R = 0;
        std::vector<Seg> segs;
        int *perm = nullptr;
        double *dinfo = nullptr;
        int64_t ps = 0;
        Blk WI, XI, G, Xb, Bg;
    };

    // Elimination of every cluster of a group (gldl.py:349-426): BK with fused
    // inertia, the panel solve on the identity, X = Bg G and the symmetric Schur
    // update, each one launch over all clusters x shifts; then compaction.
    void eliminate_group(const std::vector<int> &grp) {
        std::vector<ElimJob> J;
        for (int i : grp) {
            const Cl &ci = cl_[i];
            if (ci.nR == 0) continue;
            ElimJob j;
            j.i = i;
            j.nR = ci.nR;
            j.nS = ci.nS;
            j.m = ci.m;
            J.push_back(std::move(j));
        }
        if (J.empty()) return;
        // ---- K2/K3: BK of D[:nR,:nR] with fused inertia (packed triangle in one CTA's
        // shared memory, or in a thread-block cluster's distributed shared memory)
        hp_switch(3);
        {
            std::vector<BkJob> small, big;
            int nsmall = 0, nbig = 0;
            for (auto &j : J) {
                st_acc_->max_front = std::max<int64_t>(st_acc_->max_front, j.m);
                j.ps = pad4(j.nR);
                CK(cudaMallocFromPoolAsync((void **)&j.perm, sizeof(int) * j.ps * s_, pool_, st_));
                CK(cudaMallocFromPoolAsync((void **)&j.dinfo, sizeof(double) * 3 * j.ps * s_, pool_, st_));
                Blk &D = diag_[j.i];
                const BkJob bj{D.p, D.bs, j.m, j.nR, j.perm, j.dinfo, j.ps};
                if (bk_scratch_doubles(j.nR) && bk_cluster_size(j.nR)) {
                    st_acc_->paths[0]++;
                    big.push_back(bj);
                    nbig = std::max(nbig, j.nR);
                } else if (bk_scratch_doubles(j.nR)) {
                    bk_launch(D.p, D.bs, j.m, j.nR, j.perm, j.dinfo, j.ps);  // beyond the cluster size
                } else {
                    small.push_back(bj);
                    nsmall = std::max(nsmall, j.nR);
                }
            }
            if (!small.empty()) {
                const BkJob *dj = (const BkJob *)stage(small.data(), sizeof(BkJob) * small.size());
                Timed tm(this, 3);
                CK(launch_bk_engine(dj, (int)small.size(), s_, nsmall, d_counts_, d_status_, nullptr, 0, st_));
                st_acc_->launches++;
            }
            if (!big.empty()) {
                const BkJob *dj = (const BkJob *)stage(big.data(), sizeof(BkJob) * big.size());
                Timed tm(this, 3);
                CK(launch_bk_cluster(dj, (int)big.size(), s_, nbig, d_counts_, d_status_, st_));
                st_acc_->launches++;
            }
            dbg_sync("bk");
        }
        // ---- panel segments (live rows only)
        hp_switch(4);
        for (auto &j : J) {
            const int i = j.i;
            Blk &D = diag_[i];
            std::vector<int> partners;
            for (auto &k : adj_off_[i]) partners.push_back(k.first == i ? k.second : k.first);
            std::sort(partners.begin(), partners.end());
            j.segs.push_back({i, j.nR, j.nS, 0, D.at(j.nR, 0), D.bs, j.m, 0, 0});
            j.R = j.nS;
            for (int p : partners) {
                const int lo = elim_[p] ? cl_[p].nR : 0;
                Seg g{p, lo, cl_[p].m - lo, j.R, nullptr, 0, 0, 0, lo};
                if (i < p) {  // offd(i,p)[:nR, :]^T : panel rows = columns of the block
                    Blk &O = *off_get({i, p});
                    g.src = O.p; g.ss = O.bs; g.lds = O.cols; g.trans = 1;
                } else {      // offd(p,i)[:, :nR]
                    Blk &O = *off_get({p, i});
                    g.src = O.p; g.ss = O.bs; g.lds = O.cols; g.trans = 0;
                }
                j.segs.push_back(g);
                j.R += g.len;
            }
        }
        hp_switch(5);
        // ---- K4/K5: the panel solve on the nR x nR identity: W_I = P^T L^{-T}, X_I =
        // W_I D^{-1} (the reference: dtrsm + dgesv on Ball, gldl.py:372-378); then
        // G = X_I W_I^T = P^T L^{-T} D^{-1} L^{-1} P and X = Bg G on the tensor pipe
        std::vector<PanelJob> pj;
        std::vector<PanelTile> tiles;
        size_t psmem = 0;
        for (auto &j : J) {
            if (j.R == 0) continue;
            Blk &D = diag_[j.i];
            j.WI = alloc(j.nR, j.nR, false);
            j.XI = alloc(j.nR, j.nR, false);
            j.G = alloc(j.nR, j.nR, false);
            const int jid = (int)pj.size();
            pj.push_back(PanelJob{D.p, D.bs, j.perm, j.dinfo, j.ps, j.WI.p, j.XI.p, j.WI.bs, j.m, j.nR,
                                  j.nR, panel_lcw(j.nR)});
            psmem = std::max(psmem, panel_smem_bytes(j.nR));
            if (j.nR > 160) st_acc_->paths[1]++;
            for (int r = 0; r < j.nR; r += PANEL_ROWS) {
                PanelTile t{};
                t.src = nullptr; t.row0 = r; t.nrows = std::min(PANEL_ROWS, j.nR - r); t.src_row0 = r;
                t.job = jid;
                tiles.push_back(t);
            }
        }
        double flops_tot = 0.0, sch_tot = 0.0, bytes_tot = 0.0;
        for (auto &j : J) flops_tot += (double)j.nR * j.nR * j.nR / 3.0;
        if (!pj.empty()) {
            Pack pk;
            const size_t o1 = pk.add(pj.data(), sizeof(PanelJob) * pj.size());
            const size_t o2 = pk.add(tiles.data(), sizeof(PanelTile) * tiles.size());
            const char *d = (const char *)stage(pk.h.data(), pk.h.size());
            {
                Timed tm(this, 4);
                CK(launch_panel_multi((const PanelTile *)(d + o2), (int)tiles.size(), s_,
                                      (const PanelJob *)(d + o1), psmem, st_));
            }
            dbg_sync("panel");
            st_acc_->launches++;
            GemmBatch g0;
            for (auto &j : J)
                if (j.R)
                    add_gemm(g0, gm(j.XI.p, j.XI.bs, j.nR, 0, j.WI.p, j.WI.bs, j.nR, 1, j.G.p, j.G.bs, j.nR,
                                    j.nR, j.nR, j.nR, 1.0, 0.0), s_);
            flush(g0, s_);
            // ---- gather the panel rows Bg = [B_0; B_1; ...] (R x nR) of every job
            CopyBatch gc;
            for (auto &j : J) {
                if (!j.R) continue;
                j.Bg = alloc(j.R, j.nR, false);
                j.Xb = alloc(j.R, j.nR, false);
                for (auto &sg : j.segs) {
                    if (sg.len <= 0) continue;
                    const double *A; int lda, tA;
                    seg_as_A(sg, &A, &lda, &tA);
                    add_copy(gc, cp(A, sg.ss, lda, j.Bg.at(sg.row, 0), j.Bg.bs, j.nR, sg.len, j.nR, tA));
                }
            }
            flush(gc);
            GemmBatch g1;
            for (auto &j : J)
                if (j.R)
                    add_gemm(g1, gm(j.Bg.p, j.Bg.bs, j.nR, 0, j.G.p, j.G.bs, j.nR, 0, j.Xb.p, j.Xb.bs,
                                    j.nR, j.R, j.nR, j.nR, 1.0, 0.0), s_);
            flush(g1, s_);
            hp_switch(6);
            // ---- K6: C_big -= X Bg^T over the upper triangle of every job's R x R panel
            // space, scattered to the target blocks (fill blocks created on demand,
            // zeroed in one batched launch first: gldl.py:398-409)
            CopyBatch fz;
            const bool oz = schur_arith_ == 1;
            std::vector<OzJob> ozj;
            std::vector<int> row_job;
            int oz_rows = 0, oz_kpad = 0;
            std::vector<SchurJob> sj;
            std::vector<int> seg_all, start_all, tile_job;
            std::vector<int2> tile_ij;
            std::vector<SchurTarget> tbl_all;
            std::vector<size_t> seg_off, start_off, tbl_off;
            int tiles_tot = 0;
            for (auto &j : J) {
                if (!j.R) continue;
                const int i = j.i, nR = j.nR, m = j.m;
                Blk &D = diag_[i];
                const auto &segs = j.segs;
                const int ns = (int)segs.size();
                seg_off.push_back(seg_all.size());
                start_off.push_back(start_all.size());
                tbl_off.push_back(tbl_all.size());
                for (int x = 0; x < ns; ++x) {
                    start_all.push_back(segs[x].row);
                    for (int r = 0; r < segs[x].len; ++r) seg_all.push_back(x);
                }
                const size_t t0 = tbl_all.size();
                tbl_all.resize(t0 + (size_t)ns * ns, SchurTarget{nullptr, 0, 0, 0});
                double sch = 0.0, sch_bytes = 16.0 * (double)j.R * nR;  // X and W read once
                for (int x = 0; x < ns; ++x)
                    for (int y = x; y < ns; ++y) {
                        const Seg &a = segs[x], &b = segs[y];
                        if (a.len <= 0 || b.len <= 0) continue;
                        sch += (x == y ? 1.0 : 2.0) * (double)a.len * b.len * nR;
                        sch_bytes += 16.0 * (double)a.len * b.len;  // target r + w
                        SchurTarget &e = tbl_all[t0 + (size_t)x * ns + y];
                        e.trans = 0;
                        if (x == 0 && y == 0) {
                            e.base = D.at(nR, nR); e.bs = D.bs; e.ldc = m;
                        } else if (x == y) {
                            Blk &Dj = diag_[a.who];
                            e.base = Dj.at(a.lo, a.lo); e.bs = Dj.bs; e.ldc = Dj.cols;
                        } else if (x == 0) {
                            const int p = b.who;
                            if (i < p) {
                                Blk &O = *off_get({i, p});
                                e.base = O.at(nR, b.lo); e.bs = O.bs; e.ldc = O.cols;
                            } else {
                                Blk &O = *off_get({p, i});
                                e.base = O.at(b.lo, nR); e.bs = O.bs; e.ldc = O.cols; e.trans = 1;
                            }
                        } else {
                            const Pair key{a.who, b.who};
                            Blk *T = off_get(key);
                            if (!T) {
                                T = fill_get(key);
                                if (!T) {
                                    Blk nb = alloc(cl_[a.who].m, cl_[b.who].m, false);
                                    if (nb.p) add_copy(fz, zero(nb.p, nb.bs, nb.cols, nb.rows, nb.cols));
                                    T = fill_put(key, nb);
                                    adj_fill_[a.who].insert(key);
                                    adj_fill_[b.who].insert(key);
                                    st_acc_->fill_blocks++;
                                }
                            }
                            e.base = T->at(a.lo, b.lo); e.bs = T->bs; e.ldc = T->cols;
                        }
                    }
                const int tl = oz ? schur_oz_tiles(j.R) : schur_sym_tiles(j.R);
                sj.push_back(SchurJob{j.Xb.p, j.Bg.p, j.Xb.bs, nR, j.R, nR, ns, nullptr, nullptr, nullptr,
                                      tiles_tot, 0});
                if (oz) {
                    OzJob o{};
                    o.X = j.Xb.p; o.Bg = j.Bg.p; o.sx = j.Xb.bs; o.ld = nR; o.R = j.R; o.K = nR;
                    o.nseg = ns; o.row0 = oz_rows; o.tile0 = tiles_tot;
                    ozj.push_back(o);
                    const int rp = (j.R + 127) / 128;
                    row_job.insert(row_job.end(), rp, (int)ozj.size() - 1);
                    oz_rows += 128 * rp;
                    oz_kpad = std::max(oz_kpad, (nR + 63) / 64 * 64);
                }
                if (oz) schur_oz_tile_order(j.R, (int)sj.size() - 1, tile_ij);
                else tile_job.insert(tile_job.end(), tl, (int)sj.size() - 1);
                tiles_tot += tl;
                // algorithmic panel work (survey §8d): TRSM R nR^2 + D-scale R nR
                flops_tot += (double)j.R * nR * nR + (double)j.R * nR + sch;
                sch_tot += sch;
                bytes_tot += sch_bytes;
                // executed tensor work (fp64-equivalent 2MNK of the padded tiles)
                st_acc_->gemm_flops_exec += oz ? 2.0 * (double)tl * 128 * 64 * ((nR + 63) / 64 * 64) * s_
                                               : 2.0 * (double)tl * 64 * 64 * nR * s_;
            }
            hp_switch(7);
            flush(fz);
            // one staged region: segment maps, target tables, tile->job map, job table
            // (whose pointers into the same region are patched on the host first)
            Pack pk2;
            const size_t os = pk2.add(seg_all.data(), sizeof(int) * seg_all.size());
            const size_t ost = pk2.add(start_all.data(), sizeof(int) * start_all.size());
            const size_t otb = pk2.add(tbl_all.data(), sizeof(SchurTarget) * tbl_all.size());
            const size_t otj = oz ? pk2.add(tile_ij.data(), sizeof(int2) * tile_ij.size())
                                  : pk2.add(tile_job.data(), sizeof(int) * tile_job.size());
            const size_t osj = pk2.add(sj.data(), sizeof(SchurJob) * sj.size());
            const size_t ooz = oz ? pk2.add(ozj.data(), sizeof(OzJob) * ozj.size()) : 0;
            const size_t orj = oz ? pk2.add(row_job.data(), sizeof(int) * row_job.size()) : 0;
            StageRegion rg = stage_begin(pk2.h.size());
            SchurJob *hj = (SchurJob *)(pk2.h.data() + osj);
            OzJob *ho = oz ? (OzJob *)(pk2.h.data() + ooz) : nullptr;
            for (size_t q = 0; q < sj.size(); ++q) {
                hj[q].seg_of = (const int *)(rg.d + os) + seg_off[q];
                hj[q].seg_start = (const int *)(rg.d + ost) + start_off[q];
                hj[q].tbl = (const SchurTarget *)(rg.d + otb) + tbl_off[q];
                if (ho) {
                    ho[q].seg_of = hj[q].seg_of;
                    ho[q].seg_start = hj[q].seg_start;
                    ho[q].tbl = hj[q].tbl;
                }
            }
            std::memcpy(rg.h, pk2.h.data(), pk2.h.size());
            stage_commit(rg);
            char *d2 = rg.d;
            void *scratch = nullptr;
            if (oz) {
                // one slice buffer per wave, grown geometrically (pool growth maps new
                // physical memory: not something to do per launch)
                const size_t need = schur_oz_scratch_bytes(oz_rows, oz_kpad, s_);
                if (need > oz_scratch_cap_) {
                    if (oz_scratch_) CK(cudaFreeAsync(oz_scratch_, st_));
                    oz_scratch_cap_ = std::max(need, oz_scratch_cap_ + oz_scratch_cap_ / 2);
                    CK(cudaMallocFromPoolAsync(&oz_scratch_, oz_scratch_cap_, pool_, st_));
                }
                scratch = oz_scratch_;
            }
            static const bool schurlog = getenv("H2L_SCHURLOG") != nullptr;
            cudaEvent_t lg0 = nullptr, lg1 = nullptr;
            if (schurlog) {
                CK(cudaEventCreate(&lg0));
                CK(cudaEventCreate(&lg1));
                CK(cudaEventRecord(lg0, st_));
            }
            {
                Timed tm(this, 1);
                if (oz)
                    CK(launch_schur_oz((const OzJob *)(d2 + ooz), (const int *)(d2 + orj),
                                       (const int2 *)(d2 + otj), oz_rows, oz_kpad, tiles_tot, s_, scratch,
                                       st_));
                else
                    launch_schur_sym_multi((const SchurJob *)(d2 + osj), (const int *)(d2 + otj),
                                           tiles_tot, s_, st_);
            }
            if (schurlog) {
                CK(cudaEventRecord(lg1, st_));
                CK(cudaEventSynchronize(lg1));
                float ms = 0.f;
                CK(cudaEventElapsedTime(&ms, lg0, lg1));
                int rmax = 0, kmax = 0;
                double fl = 0.0;
                for (auto &q : sj) {
                    rmax = std::max(rmax, q.R);
                    kmax = std::max(kmax, q.K);
                    fl += (double)q.R * q.R * q.K;
                }
                fprintf(stderr, "schurlog arith=%d jobs=%zu Rmax=%d Kmax=%d tiles=%d shifts=%d ms=%.3f tflops=%.1f "
                                "alg_bytes=%.0f\n",
                        (int)oz, sj.size(), rmax, kmax, tiles_tot, s_, ms, fl * s_ / (ms * 1e-3) / 1e12,
                        bytes_tot * s_);
                cudaEventDestroy(lg0);
                cudaEventDestroy(lg1);
            }
            CK(cudaGetLastError());
            dbg_sync("schur-sym");
            st_acc_->launches++;
        }
        st_acc_->schur_flops += sch_tot * s_;
        st_acc_->bytes += bytes_tot * s_;
        st_acc_->flops += flops_tot * s_;
        st_acc_->elim_flops += flops_tot * s_;
        // ---- retire the redundant rows / columns (gldl.py:411-417).  The reference
        // zeroes them; here every block of i is compacted to its skeleton rows /
        // columns (the R part is zero from now on and never read again), and i
        // becomes an m = nS, nR = 0 cluster: later panels, Schur targets, merges and
        // fill blocks see only live rows, and the front's memory shrinks as it moves.
        hp_switch(8);
        {
            CopyBatch zc;
            std::vector<std::pair<Blk *, Blk>> repl;
            for (auto &j : J) {
                const int i = j.i, nR = j.nR, nS = j.nS, m = j.m;
                Blk &D = diag_[i];
                Blk nd = alloc(nS, nS, false);
                add_copy(zc, cp(D.at(nR, nR), D.bs, m, nd.p, nd.bs, nS, nS, nS));
                repl.push_back({&D, nd});
                for (auto *store : {&offd_, &fill_}) {
                    auto &adj = (store == &offd_) ? adj_off_[i] : adj_fill_[i];
                    for (auto &k : adj) {
                        Blk &O = (store == &offd_) ? *off_get(k) : *fill_get(k);
                        Blk N;
                        if (k.first == i) {
                            N = alloc(nS, O.cols, false);
                            add_copy(zc, cp(O.at(nR, 0), O.bs, O.cols, N.p, N.bs, N.cols, nS, O.cols));
                        } else {
                            N = alloc(O.rows, nS, false);
                            add_copy(zc, cp(O.at(0, nR), O.bs, O.cols, N.p, N.bs, N.cols, O.rows, nS));
                        }
                        repl.push_back({&O, N});
                    }
                }
            }
            flush(zc);
            for (auto &r : repl) {
                release(*r.first);
                *r.first = r.second;
            }
        }
        for (auto &j : J) {
            Cl &ci = cl_[j.i];
            ci.m = j.nS;
            ci.nR = 0;
            elim_[j.i] = 1;
            for (Blk *b : {&j.WI, &j.XI, &j.G, &j.Xb, &j.Bg}) release(*b);
            CK(cudaFreeAsync(j.perm, st_));
            CK(cudaFreeAsync(j.dinfo, st_));
        }
        hp_switch(-1);
    }

    void bk_launch(double *a, int64_t astride, int ld, int n, int *perm, double *dinfo, int64_t ps) {
        BkJob jb{a, astride, ld, n, perm, dinfo, ps};
        const BkJob *dj = (const BkJob *)stage(&jb, sizeof(jb));
        // fronts beyond one CTA's shared memory: the cluster kernel keeps the packed
        // triangle in distributed shared memory (same arithmetic, bit-identical)
        if (bk_scratch_doubles(n) && bk_cluster_size(n)) {
            {
                Timed tm(this, 3);
                CK(launch_bk_cluster(dj, 1, s_, n, d_counts_, d_status_, st_));
            }
            dbg_sync("bk-cluster");
            st_acc_->launches++;
            return;
        }
        const int64_t scr = bk_scratch_doubles(n);
        double *scratch = nullptr;
        if (scr) CK(cudaMallocFromPoolAsync((void **)&scratch, sizeof(double) * scr * s_, pool_, st_));
        {
            Timed tm(this, 3);
            CK(launch_bk_engine(dj, 1, s_, n, d_counts_, d_status_, scratch, scr, st_));
        }
        dbg_sync("bk");
        st_acc_->launches++;
        if (scratch) CK(cudaFreeAsync(scratch, st_));
    }

    void factor_root(Blk &root) {
        if (root.rows == 0 || !root.p) return;
        const int n = root.rows;
        const int64_t ps = pad4(n);
        int *perm;
        double *dinfo;
        CK(cudaMallocFromPoolAsync((void **)&perm, sizeof(int) * ps * s_, pool_, st_));
        CK(cudaMallocFromPoolAsync((void **)&dinfo, sizeof(double) * 3 * ps * s_, pool_, st_));
        bk_launch(root.p, root.bs, root.cols, n, perm, dinfo, ps);
        st_acc_->flops += (double)n * n * n / 3.0 * s_;
        CK(cudaFreeAsync(perm, st_));
        CK(cudaFreeAsync(dinfo, st_));
    }

    // ----------------------------------------------------------------- merges
    // skeleton-skeleton content of a finished pair (gldl.py:429-438)
    bool content(const Pair &k, const double **p, int64_t *bs, int *ld, int *rows, int *cols) {
        auto c = coup_.find(k);
        if (c != coup_.end()) {
            *p = c->second.p; *bs = c->second.bs; *ld = c->second.cols;
            *rows = c->second.rows; *cols = c->second.cols;
            return c->second.p != nullptr;
        }
        const Blk *B = off_get(k);
        if (!B) B = fill_get(k);
        if (!B || !B->p) return false;
        const int ra = cl_[k.first].nR, rb = cl_[k.second].nR;
        *p = B->at(ra, rb); *bs = B->bs; *ld = B->cols;
        *rows = B->rows - ra; *cols = B->cols - rb;
        return *rows > 0 && *cols > 0;
    }

    std::set<Pair> all_pairs() const {
        std::set<Pair> u;
        for (auto &kv : coup_) u.insert(kv.first);
        for (auto &kv : offd_) u.insert(kv.first);
        for (auto &kv : fill_) u.insert(kv.first);
        return u;
    }

    Blk merge_flat() {
        const int nl = 1 << depth_;
        std::vector<int> start(nl);
        int tot = 0;
        for (int i = 0; i < nl; ++i) { start[i] = tot; tot += cl_[i].nS; }
        Blk R = alloc(tot, tot, true);
        CopyBatch c;
        for (int i = 0; i < nl; ++i) {
            const Cl &ci = cl_[i];
            if (ci.nS == 0 || !diag_[i].p) continue;
            add_copy(c, cp(diag_[i].at(ci.nR, ci.nR), diag_[i].bs, ci.m, R.at(start[i], start[i]),
                           R.bs, tot, ci.nS, ci.nS));
        }
        for (auto &k : all_pairs()) {
            const double *p; int64_t bs; int ld, rows, cols;
            if (!content(k, &p, &bs, &ld, &rows, &cols)) continue;
            add_copy(c, cp(p, bs, ld, R.at(start[k.first], start[k.second]), R.bs, tot, rows, cols));
            add_copy(c, cp(p, bs, ld, R.at(start[k.second], start[k.first]), R.bs, tot, cols, rows, 1));
        }
        flush(c);
        return R;
    }

    Blk merge_pairwise(int level, bool to_root) {
        const int np = 1 << (level - 1);
        std::vector<int> loc(2 * np), msz(np);
        for (int p = 0; p < np; ++p) {
            loc[2 * p] = 0;
            loc[2 * p + 1] = cl_[2 * p].nS;
            msz[p] = cl_[2 * p].nS + cl_[2 * p + 1].nS;
        }
        std::vector<Blk> raw(np);
        CopyBatch c;
        for (int p = 0; p < np; ++p) {
            const int c1 = 2 * p, c2 = 2 * p + 1;
            const int s1 = cl_[c1].nS, s2 = cl_[c2].nS;
            raw[p] = alloc(s1 + s2, s1 + s2, true);
            if (!raw[p].p) continue;
            const int mp = s1 + s2;
            if (s1) add_copy(c, cp(diag_[c1].at(cl_[c1].nR, cl_[c1].nR), diag_[c1].bs, cl_[c1].m,
                                   raw[p].p, raw[p].bs, mp, s1, s1));
            if (s2) add_copy(c, cp(diag_[c2].at(cl_[c2].nR, cl_[c2].nR), diag_[c2].bs, cl_[c2].m,
                                   raw[p].at(s1, s1), raw[p].bs, mp, s2, s2));
            const double *q; int64_t bs; int ld, rows, cols;
            if (content({c1, c2}, &q, &bs, &ld, &rows, &cols)) {
                add_copy(c, cp(q, bs, ld, raw[p].at(0, s1), raw[p].bs, mp, rows, cols));
                add_copy(c, cp(q, bs, ld, raw[p].at(s1, 0), raw[p].bs, mp, cols, rows, 1));
            }
        }
        std::map<Pair, Blk> rawpair;
        for (auto &k : all_pairs()) {
            const int p = k.first >> 1, q = k.second >> 1;
            if (p == q) continue;
            const double *src; int64_t bs; int ld, rows, cols;
            if (!content(k, &src, &bs, &ld, &rows, &cols)) continue;
            auto it = rawpair.find({p, q});
            if (it == rawpair.end()) it = rawpair.emplace(Pair{p, q}, alloc(msz[p], msz[q], true)).first;
            Blk &dst = it->second;
            add_copy(c, cp(src, bs, ld, dst.at(loc[k.first], loc[k.second]), dst.bs, dst.cols, rows, cols));
        }
        flush(c);
        if (to_root) {
            for (auto &kv : rawpair) release(kv.second);
            for (int p = 1; p < np; ++p) release(raw[p]);
            return raw[0];
        }
        const int pl = level - 1;
        // parent bases (shift independent): [U_R | extras | U_S] (gldl.py:561-588)
        std::vector<Cl> ncl(np);
        std::vector<const double *> Q(np, nullptr);
        std::vector<double *> Qown;
        CopyBatch qc;
        for (int p = 0; p < np; ++p) {
            const int mp = msz[p];
            if (mp == 0) continue;
            const Cl &a = cl_[2 * p], &b = cl_[2 * p + 1];
            const int nd = node(pl, p);
            const int rk = std::max(0, brank_[nd]);
            const int e1 = a.nS - a.r0, e2 = b.nS - b.r0;
            const double *bq = boff_[nd] >= 0 ? arena_ + boff_[nd] : nullptr;
            const int m0 = bdim_[nd];
            ncl[p] = Cl{mp, mp - rk, rk, rk};
            if (e1 == 0 && e2 == 0) {
                Q[p] = bq;  // arena square basis, m0 == mp
                continue;
            }
            double *qp;
            CK(cudaMallocFromPoolAsync((void **)&qp, sizeof(double) * (int64_t)mp * mp, pool_, st_));
            CK(cudaMemsetAsync(qp, 0, sizeof(double) * (int64_t)mp * mp, st_));
            Qown.push_back(qp);
            Q[p] = qp;
            const int nRh = a.r0 + b.r0 - rk;
            // rows of the stored basis: [0, r0a) -> [0, r0a) ; [r0a, m0) -> [nSa, nSa + r0b)
            if (bq && nRh > 0) {
                add_copy(qc, cp(bq, 0, m0, qp, 0, mp, a.r0, nRh));
                add_copy(qc, cp(bq + (int64_t)a.r0 * m0, 0, m0, qp + (int64_t)a.nS * mp, 0, mp, b.r0, nRh));
            }
            if (bq && rk > 0) {
                add_copy(qc, cp(bq + (m0 - rk), 0, m0, qp + (mp - rk), 0, mp, a.r0, rk));
                add_copy(qc, cp(bq + (int64_t)a.r0 * m0 + (m0 - rk), 0, m0,
                                qp + (int64_t)a.nS * mp + (mp - rk), 0, mp, b.r0, rk));
            }
            if (e1 > 0) {
                CopyTask t = zero(qp + (int64_t)a.r0 * mp + nRh, 0, mp, e1, e1);
                t.ident = 1;
                add_copy(qc, t);
            }
            if (e2 > 0) {
                CopyTask t = zero(qp + (int64_t)(a.nS + b.r0) * mp + nRh + e1, 0, mp, e2, e2);
                t.ident = 1;
                add_copy(qc, t);
            }
        }
        {   // Q construction uses a single shift
            const int s_save = s_;
            s_ = 1;
            flush(qc);
            s_ = s_save;
        }
        // new blocks: ndiag = Q^T raw Q ; offd/fill = Qp^T raw Qq
        std::vector<Blk> ndiag(np);
        std::map<Pair, Blk> noffd, nfill;
        std::vector<Blk> tmps;
        GemmBatch g1, g2;
        auto congr = [&](const Blk &in, int p, int q, Blk &out) {
            const int mp = msz[p], mq = msz[q];
            out = alloc(mp, mq, false);
            if (!out.p) return;
            Blk tmp = alloc(mp, mq, false);
            add_gemm(g1, gm(Q[p], 0, mp, 1, in.p, in.bs, mq, 0, tmp.p, tmp.bs, mq, mp, mq, mp, 1.0,
                            0.0), s_);
            add_gemm(g2, gm(tmp.p, tmp.bs, mq, 0, Q[q], 0, mq, 0, out.p, out.bs, mq, mp, mq, mq, 1.0,
                            0.0), s_);
            tmps.push_back(tmp);
        };
        for (int p = 0; p < np; ++p)
            if (msz[p]) congr(raw[p], p, p, ndiag[p]);
        std::vector<Blk> zeros;
        auto dit = deferred_.find(pl);
        if (dit != deferred_.end())
            for (auto &k : dit->second) {
                auto r = rawpair.find(k);
                Blk in;
                if (r != rawpair.end()) {
                    in = r->second;
                    rawpair.erase(r);
                } else {
                    in = alloc(msz[k.first], msz[k.second], true);
                }
                zeros.push_back(in);
                congr(in, k.first, k.second, noffd[k]);
            }
        for (auto &kv : rawpair) {
            congr(kv.second, kv.first.first, kv.first.second, nfill[kv.first]);
            st_acc_->fill_blocks++;
            zeros.push_back(kv.second);
        }
        flush(g1, s_, 2);
        flush(g2, s_, 2);
        for (auto &b : tmps) release(b);
        for (auto &b : zeros) release(b);
        for (auto &b : raw) release(b);
        for (double *q : Qown) CK(cudaFreeAsync(q, st_));
        // swap in the parent level
        clear_level();
        cl_ = ncl;
        diag_ = ndiag;
        reset_adjacency(np);
        for (auto &kv : noffd) {
            off_put(kv.first, kv.second);
            adj_off_[kv.first.first].insert(kv.first);
            adj_off_[kv.first.second].insert(kv.first);
        }
        for (auto &kv : nfill) {
            fill_put(kv.first, kv.second);
            adj_fill_[kv.first.first].insert(kv.first);
            adj_fill_[kv.first.second].insert(kv.first);
        }
        CopyBatch cc;
        load_couplings(pl, cc);
        flush(cc);
        return Blk{};
    }
};

}  // namespace h2l

// ---------------------------------------------------------------- status glue
namespace h2l {
__global__ void active_kernel(const int *status, int *active, int s) {
    int z = blockIdx.x * blockDim.x + threadIdx.x;
    if (z < s) active[z] = status[z] == 0;
}
__global__ void pack_counts_kernel(const int64_t *counts, const int *status, int64_t *out, int s) {
    int z = blockIdx.x * blockDim.x + threadIdx.x;
    if (z >= s) return;
    out[4 * z + 0] = counts[3 * z + 0];
    out[4 * z + 1] = counts[3 * z + 1];
    out[4 * z + 2] = counts[3 * z + 2];
    out[4 * z + 3] = status[z] ? H2L_SHIFT_SINGULAR : H2L_SHIFT_OK;
}
void launch_pack_counts(const int64_t *counts, const int *status, int64_t *out, int s, cudaStream_t st) {
    pack_counts_kernel<<<(s + 127) / 128, 128, 0, st>>>(counts, status, out, s);
}
void Wave::activity_from_status(int *d_active) {
    active_kernel<<<(s_ + 127) / 128, 128, 0, st_>>>(d_status_, d_active, s_);
    CK(cudaGetLastError());
}
}  // namespace h2l

// ------------------------------------------------------------ concurrent waves
// The engine splits a call into waves of <= max_batch shifts and runs up to
// `concurrency` waves at once, each on its own stream driven by its own host
// thread.  Within one wave the elimination steps are a dependent chain of
// latency-bound launches (BK, panel) and throughput-bound ones (DMMA GEMMs);
// a second wave in flight fills the SMs the first one leaves idle.
namespace h2l {
static void merge_stats(h2l_stats &a, const h2l_stats &b) {
    a.fill_blocks = std::max(a.fill_blocks, b.fill_blocks);
    a.recompressions = std::max(a.recompressions, b.recompressions);
    a.rank_added = std::max(a.rank_added, b.rank_added);
    a.max_front = std::max(a.max_front, b.max_front);
    a.dropped_fro += b.dropped_fro;
    a.flops += b.flops;
    a.elim_flops += b.elim_flops;
    a.bytes += b.bytes;
    a.ms_schur += b.ms_schur;
    a.ms_bk += b.ms_bk;
    a.launches += b.launches;
    a.groups += b.groups;
    for (int k = 0; k < 4; ++k) a.paths[k] += b.paths[k];
    a.schur_flops += b.schur_flops;
    a.gemm_flops_exec += b.gemm_flops_exec;
    for (int k = 0; k < 8; ++k) a.ms_kind[k] += b.ms_kind[k];
}

class Engine {
public:
    explicit Engine(int device) : dev_(device) {
        waves_.emplace_back(new Wave(device));
        CK(cudaEventCreate(&ev_[0]));
        CK(cudaEventCreate(&ev_[1]));
    }
    ~Engine() {
        cudaSetDevice(dev_);
        for (size_t k = 1; k < waves_.size(); ++k) waves_[k].reset();  // borrowers first
        waves_.clear();
        cudaEventDestroy(ev_[0]);
        cudaEventDestroy(ev_[1]);
    }
    void set_option(const std::string &k, int64_t v) {
        if (k == "concurrency") {
            concurrency_ = (int)std::max<int64_t>(1, std::min<int64_t>(8, v));
            return;
        }
        for (auto &w : waves_) w->set_option(k, v);
    }
    void upload(const h2l_plan *pl) {
        waves_[0]->upload(pl);
        for (size_t k = 1; k < waves_.size(); ++k) waves_[k]->adopt(*waves_[0]);
    }
    void inertia(const double *mu, int s, int64_t *counts, int32_t *status, h2l_stats *stats,
                 int64_t *dev_out = nullptr) {
        CK(cudaSetDevice(dev_));
        try {
            inertia_impl(mu, s, counts, status, stats, dev_out);
        } catch (...) {
            // a failed call (device OOM, launch error) must not leave the waves' working
            // blocks, per-wave buffers or staged task lists behind for the next call
            for (auto &w : waves_) w->abort_cleanup();
            throw;
        }
    }
    void inertia_impl(const double *mu, int s, int64_t *counts, int32_t *status, h2l_stats *stats,
                      int64_t *dev_out) {
        const auto host0 = std::chrono::steady_clock::now();
        const int mb = waves_[0]->max_batch();
        const int nw = (s + mb - 1) / mb;
        const int C = std::min(concurrency_, nw);
        while ((int)waves_.size() < C) {
            waves_.emplace_back(new Wave(dev_));
            waves_.back()->adopt(*waves_[0]);
        }
        std::vector<h2l_stats> acc(C);
        for (auto &a : acc) a = h2l_stats{};
        for (int t = 0; t < C; ++t) waves_[t]->reset_mem_high();
        cudaStream_t s0 = waves_[0]->stream();
        CK(cudaEventRecord(ev_[0], s0));
        for (int t = 1; t < C; ++t) CK(cudaStreamWaitEvent(waves_[t]->stream(), ev_[0], 0));
        auto work = [&](int t) {
            for (int w = t; w < nw; w += C) {
                const int w0 = w * mb, ws = std::min(mb, s - w0);
                waves_[t]->run(mu + w0, ws, counts ? counts + 3 * (int64_t)w0 : nullptr,
                               status ? status + w0 : nullptr, acc[t],
                               dev_out ? dev_out + 4 * (int64_t)w0 : nullptr);
            }
        };
        if (C == 1) {
            work(0);
        } else {
            std::vector<std::thread> th;
            std::vector<std::string> errs(C);
            std::vector<int> codes(C, 0);
            for (int t = 0; t < C; ++t)
                th.emplace_back([&, t] {
                    try {
                        cudaSetDevice(dev_);
                        work(t);
                    } catch (const CudaFail &x) {
                        codes[t] = x.code;
                        errs[t] = x.what();
                    } catch (const std::exception &x) {
                        codes[t] = H2L_EINVAL;
                        errs[t] = x.what();
                    }
                });
            for (auto &x : th) x.join();
            for (int t = 0; t < C; ++t)
                if (codes[t]) throw CudaFail(codes[t], errs[t]);
            for (int t = 1; t < C; ++t) {
                cudaEvent_t e;
                CK(cudaEventCreateWithFlags(&e, cudaEventDisableTiming));
                CK(cudaEventRecord(e, waves_[t]->stream()));
                CK(cudaStreamWaitEvent(s0, e, 0));
                CK(cudaEventDestroy(e));
            }
        }
        CK(cudaEventRecord(ev_[1], s0));
        CK(cudaEventSynchronize(ev_[1]));
        float ms = 0.f;
        CK(cudaEventElapsedTime(&ms, ev_[0], ev_[1]));
        h2l_stats tot{};
        for (auto &a : acc) merge_stats(tot, a);
        tot.ms_total = ms;
        for (int t = 0; t < C; ++t) tot.mem_peak += waves_[t]->mem_high();
        tot.ms_host = std::chrono::duration<double, std::milli>(std::chrono::steady_clock::now() - host0).count();
        if (stats) *stats = tot;
    }

    int device() const { return dev_; }

private:
    int dev_;
    int concurrency_ = 2;
    cudaEvent_t ev_[2];
    std::vector<std::unique_ptr<Wave>> waves_;
};
}  // namespace h2l

// =================================================================== C ABI
struct h2l_engine {
    h2l::Engine *impl = nullptr;
    std::string err;
};

static thread_local std::string g_err;

template <class F>
static int guarded(h2l_engine *e, F &&f) {
    try {
        f();
        return H2L_OK;
    } catch (const h2l::CudaFail &x) {
        (e ? e->err : g_err) = x.what();
        return x.code;
    } catch (const std::bad_alloc &) {
        (e ? e->err : g_err) = "host allocation failed";
        return H2L_ENOMEM;
    } catch (const std::exception &x) {
        (e ? e->err : g_err) = x.what();
        return H2L_EINVAL;
    }
}

static int check_device(int device) {
    int cnt = 0;
    if (cudaGetDeviceCount(&cnt) != cudaSuccess || cnt <= 0) {
        cudaGetLastError();
        g_err = "no CUDA device";
        return H2L_ENODEV;
    }
    if (device < 0 || device >= cnt) {
        g_err = "device index out of range";
        return H2L_ENODEV;
    }
    return H2L_OK;
}

extern "C" {

int h2l_create(h2l_engine **engine, int device) {
    if (!engine) return H2L_EINVAL;
    *engine = nullptr;
    int rc = check_device(device);
    if (rc) return rc;
    return guarded(nullptr, [&] {
        auto *e = new h2l_engine;
        try {
            e->impl = new h2l::Engine(device);
        } catch (...) {
            delete e;
            throw;
        }
        *engine = e;
    });
}

int h2l_destroy(h2l_engine *engine) {
    if (!engine) return H2L_OK;
    delete engine->impl;
    delete engine;
    return H2L_OK;
}

const char *h2l_last_error(const h2l_engine *engine) {
    return engine ? engine->err.c_str() : g_err.c_str();
}

int h2l_upload(h2l_engine *engine, const h2l_plan *plan) {
    if (!engine || !plan) return H2L_EINVAL;
    return guarded(engine, [&] { engine->impl->upload(plan); });
}

int h2l_inertia(h2l_engine *engine, const double *mu, int32_t s, int64_t *counts, int32_t *status,
                h2l_stats *stats) {
    if (!engine || (s > 0 && (!mu || !counts || !status)) || s < 0) return H2L_EINVAL;
    if (s == 0) return H2L_OK;
    return guarded(engine, [&] { engine->impl->inertia(mu, s, counts, status, stats); });
}

int h2l_inertia_device(h2l_engine *engine, const double *mu, int32_t s, int64_t *dev_counts,
                       h2l_stats *stats) {
    if (!engine || s < 0 || (s > 0 && (!mu || !dev_counts))) return H2L_EINVAL;
    if (s == 0) return H2L_OK;
    return guarded(engine, [&] { engine->impl->inertia(mu, s, nullptr, nullptr, stats, dev_counts); });
}

int h2l_set_option(h2l_engine *engine, const char *key, int64_t value) {
    if (!engine || !key) return H2L_EINVAL;
    return guarded(engine, [&] { engine->impl->set_option(key, value); });
}

int h2l_bk_factor(int device, double *a, int64_t n, int32_t count, int64_t *ipiv,
                  const double *tol, int64_t *info) {
    if (n < 0 || count < 0 || (count && (!a || !ipiv || !tol || !info))) return H2L_EINVAL;
    if (n == 0 || count == 0) return H2L_OK;
    int rc = check_device(device);
    if (rc) return rc;
    return guarded(nullptr, [&] {
        CK(cudaSetDevice(device));
        const size_t bytes = sizeof(double) * (size_t)n * n * count;
        double *da, *dt, *ds = nullptr;
        int64_t *dp, *di;
        CK(cudaMalloc(&da, bytes));
        CK(cudaMalloc(&dt, sizeof(double) * count));
        CK(cudaMalloc(&dp, sizeof(int64_t) * n * count));
        CK(cudaMalloc(&di, sizeof(int64_t) * count));
        const int64_t scr = h2l::bk_scratch_doubles((int)n);
        if (scr) CK(cudaMalloc(&ds, sizeof(double) * (size_t)n * (n + 1) / 2 * count));
        CK(cudaMemcpy(da, a, bytes, cudaMemcpyHostToDevice));
        CK(cudaMemcpy(dt, tol, sizeof(double) * count, cudaMemcpyHostToDevice));
        CK(cudaMemset(dp, 0, sizeof(int64_t) * n * count));
        CK(h2l::launch_bk_kat(da, (int)n, count, dt, dp, di, ds, 0));
        CK(cudaDeviceSynchronize());
        CK(cudaMemcpy(a, da, bytes, cudaMemcpyDeviceToHost));
        CK(cudaMemcpy(ipiv, dp, sizeof(int64_t) * n * count, cudaMemcpyDeviceToHost));
        CK(cudaMemcpy(info, di, sizeof(int64_t) * count, cudaMemcpyDeviceToHost));
        cudaFree(da); cudaFree(dt); cudaFree(dp); cudaFree(di);
        if (ds) cudaFree(ds);
    });
}

int h2l_bk_inertia(int device, const double *a, int64_t n, int32_t count, const int64_t *ipiv,
                   const double *zero_tol, int64_t *counts) {
    if (n < 0 || count < 0 || (count && (!a || !ipiv || !zero_tol || !counts))) return H2L_EINVAL;
    if (count == 0) return H2L_OK;
    if (n == 0) {
        std::memset(counts, 0, sizeof(int64_t) * 3 * count);
        return H2L_OK;
    }
    int rc = check_device(device);
    if (rc) return rc;
    return guarded(nullptr, [&] {
        CK(cudaSetDevice(device));
        const size_t bytes = sizeof(double) * (size_t)n * n * count;
        double *da, *dz;
        int64_t *dp, *dc;
        CK(cudaMalloc(&da, bytes));
        CK(cudaMalloc(&dz, sizeof(double) * count));
        CK(cudaMalloc(&dp, sizeof(int64_t) * n * count));
        CK(cudaMalloc(&dc, sizeof(int64_t) * 3 * count));
        CK(cudaMemcpy(da, a, bytes, cudaMemcpyHostToDevice));
        CK(cudaMemcpy(dz, zero_tol, sizeof(double) * count, cudaMemcpyHostToDevice));
        CK(cudaMemcpy(dp, ipiv, sizeof(int64_t) * n * count, cudaMemcpyHostToDevice));
        CK(h2l::launch_bk_inertia(da, (int)n, count, dp, dz, dc, 0));
        CK(cudaDeviceSynchronize());
        CK(cudaMemcpy(counts, dc, sizeof(int64_t) * 3 * count, cudaMemcpyDeviceToHost));
        cudaFree(da); cudaFree(dz); cudaFree(dp); cudaFree(dc);
    });
}

const char *h2l_version(void) { return "h2ldl 0.2 sm_100a"; }

}  // extern "C"

// ---------------------------------------------------------------- multi-GPU
// One process, one engine per GPU (each holding a replica of H), shifts sharded
// in contiguous slices (the reference's chunk rule, parallel.py:85-96), the only
// exchange an NCCL all-gather of the packed integer counts between the engines'
// device buffers.  NCCL is opened at h2l_comm_init (dlopen: the library itself
// does not depend on it, and a process that already loaded NCCL -- e.g. torch's
// -- reuses that copy).
#include <dlfcn.h>
#include <nccl.h>

namespace {
struct NcclApi {
    void *lib = nullptr;
    ncclResult_t (*commInitAll)(ncclComm_t *, int, const int *) = nullptr;
    ncclResult_t (*allGather)(const void *, void *, size_t, ncclDataType_t, ncclComm_t, cudaStream_t) = nullptr;
    ncclResult_t (*groupStart)() = nullptr;
    ncclResult_t (*groupEnd)() = nullptr;
    ncclResult_t (*commDestroy)(ncclComm_t) = nullptr;
    const char *(*errStr)(ncclResult_t) = nullptr;
    bool load(std::string &err) {
        if (lib) return true;
        lib = dlopen("libnccl.so.2", RTLD_NOW | RTLD_NOLOAD);
        if (!lib) lib = dlopen("libnccl.so.2", RTLD_NOW | RTLD_GLOBAL);
        if (!lib) lib = dlopen("libnccl.so", RTLD_NOW | RTLD_GLOBAL);
        if (!lib) { err = "libnccl.so.2 not found"; return false; }
        commInitAll = (decltype(commInitAll))dlsym(lib, "ncclCommInitAll");
        allGather = (decltype(allGather))dlsym(lib, "ncclAllGather");
        groupStart = (decltype(groupStart))dlsym(lib, "ncclGroupStart");
        groupEnd = (decltype(groupEnd))dlsym(lib, "ncclGroupEnd");
        commDestroy = (decltype(commDestroy))dlsym(lib, "ncclCommDestroy");
        errStr = (decltype(errStr))dlsym(lib, "ncclGetErrorString");
        if (!commInitAll || !allGather || !groupStart || !groupEnd || !commDestroy || !errStr) {
            err = "libnccl.so.2 lacks a required symbol";
            lib = nullptr;
            return false;
        }
        return true;
    }
};
NcclApi g_nccl;
std::mutex g_nccl_mu;
}  // namespace

struct h2l_comm {
    std::vector<h2l_engine *> eng;
    std::vector<int> dev;
    std::vector<ncclComm_t> comm;
    std::vector<cudaStream_t> st;
    std::string err;
};

#define NCK(x)                                                                                   \
    do {                                                                                         \
        ncclResult_t r_ = (x);                                                                   \
        if (r_ != ncclSuccess)                                                                   \
            throw h2l::CudaFail(H2L_ECUDA, std::string(#x) + ": " + g_nccl.errStr(r_));          \
    } while (0)

extern "C" {

int h2l_comm_init(h2l_engine *const *engines, int ngpu, h2l_comm **comm) {
    if (!engines || ngpu <= 0 || !comm) return H2L_EINVAL;
    *comm = nullptr;
    for (int r = 0; r < ngpu; ++r)
        if (!engines[r]) return H2L_EINVAL;
    return guarded(nullptr, [&] {
        {
            std::lock_guard<std::mutex> g(g_nccl_mu);
            std::string e;
            if (!g_nccl.load(e)) throw h2l::CudaFail(H2L_ENODEV, e);
        }
        auto *c = new h2l_comm;
        try {
            for (int r = 0; r < ngpu; ++r) {
                c->eng.push_back(engines[r]);
                c->dev.push_back(engines[r]->impl->device());
            }
            for (int a = 0; a < ngpu; ++a)
                for (int b = a + 1; b < ngpu; ++b)
                    if (c->dev[a] == c->dev[b])
                        throw h2l::CudaFail(H2L_EINVAL, "h2l_comm_init: two engines on one device");
            c->comm.assign(ngpu, nullptr);
            NCK(g_nccl.commInitAll(c->comm.data(), ngpu, c->dev.data()));
            for (int r = 0; r < ngpu; ++r) {
                cudaStream_t s;
                CK(cudaSetDevice(c->dev[r]));
                CK(cudaStreamCreateWithFlags(&s, cudaStreamNonBlocking));
                c->st.push_back(s);
            }
        } catch (...) {
            for (auto x : c->comm)
                if (x) g_nccl.commDestroy(x);
            delete c;
            throw;
        }
        *comm = c;
    });
}

int h2l_comm_destroy(h2l_comm *comm) {
    if (!comm) return H2L_OK;
    for (size_t r = 0; r < comm->comm.size(); ++r) {
        cudaSetDevice(comm->dev[r]);
        if (r < comm->st.size()) cudaStreamDestroy(comm->st[r]);
        if (comm->comm[r]) g_nccl.commDestroy(comm->comm[r]);
    }
    delete comm;
    return H2L_OK;
}

int h2l_inertia_multi(h2l_comm *comm, const double *mu, int32_t s_total, int64_t *counts,
                      int32_t *status, h2l_stats *stats) {
    if (!comm || s_total < 0 || (s_total > 0 && (!mu || !counts || !status))) return H2L_EINVAL;
    if (s_total == 0) return H2L_OK;
    return guarded(nullptr, [&] {
        const int G = (int)comm->eng.size();
        std::vector<int> lo(G), hi(G);
        const int base = s_total / G, extra = s_total % G;
        for (int r = 0, p = 0; r < G; ++r) {
            lo[r] = p;
            p += base + (r < extra ? 1 : 0);
            hi[r] = p;
        }
        const int width = base + (extra ? 1 : 0);
        const size_t rowb = sizeof(int64_t) * 4;
        std::vector<int64_t *> send(G, nullptr), recv(G, nullptr);
        std::vector<h2l_stats> st(G);
        std::vector<int> codes(G, 0);
        std::vector<std::string> errs(G);
        try {
            for (int r = 0; r < G; ++r) {
                CK(cudaSetDevice(comm->dev[r]));
                CK(cudaMalloc(&send[r], rowb * std::max(1, width)));
                CK(cudaMalloc(&recv[r], rowb * std::max(1, width) * G));
                CK(cudaMemset(send[r], 0xff, rowb * std::max(1, width)));  // padding rows: -1
            }
            // every engine factorizes its slice on its own host thread (engines are
            // independent; calls on one engine are never concurrent)
            std::vector<std::thread> th;
            for (int r = 0; r < G; ++r)
                th.emplace_back([&, r] {
                    try {
                        cudaSetDevice(comm->dev[r]);
                        st[r] = h2l_stats{};
                        if (hi[r] > lo[r])
                            comm->eng[r]->impl->inertia(mu + lo[r], hi[r] - lo[r], nullptr, nullptr, &st[r],
                                                        send[r]);
                    } catch (const h2l::CudaFail &x) {
                        codes[r] = x.code;
                        errs[r] = x.what();
                    } catch (const std::exception &x) {
                        codes[r] = H2L_EINVAL;
                        errs[r] = x.what();
                    }
                });
            for (auto &t : th) t.join();
            for (int r = 0; r < G; ++r)
                if (codes[r]) throw h2l::CudaFail(codes[r], "rank " + std::to_string(r) + ": " + errs[r]);
            NCK(g_nccl.groupStart());
            for (int r = 0; r < G; ++r) {
                CK(cudaSetDevice(comm->dev[r]));
                NCK(g_nccl.allGather(send[r], recv[r], (size_t)4 * width, ncclInt64, comm->comm[r],
                                     comm->st[r]));
            }
            NCK(g_nccl.groupEnd());
            for (int r = 0; r < G; ++r) {
                CK(cudaSetDevice(comm->dev[r]));
                CK(cudaStreamSynchronize(comm->st[r]));
            }
            std::vector<int64_t> h((size_t)4 * width * G);
            CK(cudaSetDevice(comm->dev[0]));
            CK(cudaMemcpy(h.data(), recv[0], h.size() * sizeof(int64_t), cudaMemcpyDeviceToHost));
            for (int r = 0; r < G; ++r)
                for (int q = lo[r]; q < hi[r]; ++q) {
                    const int64_t *row = h.data() + ((size_t)r * width + (q - lo[r])) * 4;
                    counts[3 * (int64_t)q] = row[0];
                    counts[3 * (int64_t)q + 1] = row[1];
                    counts[3 * (int64_t)q + 2] = row[2];
                    status[q] = (int32_t)row[3];
                }
            if (stats) {
                h2l_stats tot{};
                for (int r = 0; r < G; ++r) {
                    h2l::merge_stats(tot, st[r]);
                    tot.ms_total = std::max(tot.ms_total, st[r].ms_total);  // max over ranks
                    tot.ms_host = std::max(tot.ms_host, st[r].ms_host);
                    tot.mem_peak = std::max(tot.mem_peak, st[r].mem_peak);
                }
                *stats = tot;
            }
        } catch (...) {
            for (int r = 0; r < G; ++r) {
                cudaSetDevice(comm->dev[r]);
                if (send[r]) cudaFree(send[r]);
                if (recv[r]) cudaFree(recv[r]);
            }
            throw;
        }
        for (int r = 0; r < G; ++r) {
            cudaSetDevice(comm->dev[r]);
            cudaFree(send[r]);
            cudaFree(recv[r]);
        }
    });
}

}  // extern "C"

