// Tensor-scale C-ABI: the batched quantize pipeline (pipeline.cpp:65-115 of
// the reference, applied to a batch of independent tensors the way
// model.cpp:154-192 applies it to a model), tensor statistics, outlier
// detection, dequantisation and reconstruction error.
//
// Phase 1 (all tensors, grouped launches): K1 pass 1 -> merge -> pass 2 ->
// merge -> K2 count -> scan; one D2H of the per-tensor stats (sizes the COO
// buffers, reports non-finite inputs). Phase 2: K2 write, K3 per row-class,
// K3b, column finalize, column-ordered totals, K4. One more sync publishes
// the errors / invariant.
#include <algorithm>
#include <cstdio>
#include <cstdlib>
#include <cmath>
#include <cstring>
#include <map>
#include <memory>
#include <vector>

#include "runtime.hpp"

namespace ezq {

namespace {

constexpr unsigned long long kNoBad = ~0ull;

int64_t ceil_div(int64_t a, int64_t b) { return (a + b - 1) / b; }

// Columns per K3 CTA. The busiest SM processes ceil(groups / SMs) strips of
// `cb` columns; fewer concurrent warps than ~12 per SM leave the FP64/issue
// pipes idle during each step's reduction + Adam latency. Minimise
// (columns on the busiest SM) / warp-efficiency; ties go to wider strips.
int choose_k3_width(const K3Launch& base, const std::vector<int>& members, const int64_t* cols,
                    const DeviceInfo& di) {
    const int unit = (base.W == 1) ? 32 / base.L : 1;
    const int max_teams = (base.W == 1) ? 16 * unit : std::max(1, 16 / base.W);
    int best_cb = unit;
    double best = 1e300;
    for (int cb = unit; cb <= max_teams; cb += unit) {
        K3Launch t = base;
        set_k3_width(t, cb);
        // Warps of a CTA map to SMSPs by warp id % 4: only multiples of 4
        // warps keep the four schedulers equally loaded.
        if ((t.threads / 32) % 4 != 0) continue;
        if (!t.global_strip && t.smem > static_cast<size_t>(di.max_smem_optin)) break;
        const int cps_smem = t.global_strip ? 8 : static_cast<int>(di.smem_per_sm / (t.smem + 1024));
        const int cps = std::min({cps_smem, 2048 / t.threads, 8});
        if (cps < 1) break;
        int64_t groups = 0;
        for (int i : members) groups += ceil_div(cols[i], cb);
        const int64_t per_sm = ceil_div(groups, di.sms);
        const double warps = static_cast<double>(std::min<int64_t>(cps, per_sm)) * (t.threads / 32);
        const double eff = std::min(1.0, warps / 12.0);
        // A lone CTA per SM cannot hide its strip load and sequential-error
        // epilogue behind another CTA's Adam loop.
        const double overlap = (std::min<int64_t>(cps, per_sm) >= 2) ? 1.0 : 1.12;
        const double cost = static_cast<double>(per_sm * cb) / eff * overlap;
        if (cost <= best + 1e-9) {
            best = cost;
            best_cb = cb;
        }
    }
    return best_cb;
}

TStats fresh_stats() {
    TStats s;
    std::memset(&s, 0, sizeof(s));
    s.bad_index = kNoBad;
    return s;
}

// Uploads `h` into arena memory `d` (async; host vector must outlive the copy
// -> callers keep it alive until the next sync).
// Small host->device uploads go through a per-thread pinned staging buffer:
// a pageable cudaMemcpyAsync is host-synchronous and waits for the DMA
// engine, i.e. behind any large H2D copy in flight (the chunked host-input
// pipeline), which would serialize ingest and compute. The buffer is reused
// by the next call only after this call's stream synchronization.
struct Stager {
    char* base = nullptr;
    size_t cap = 0, off = 0;
    void reset(size_t need) {
        off = 0;
        if (need <= cap) return;
        if (base) host_free(base);
        cap = std::max(need, cap * 2);
        base = static_cast<char*>(host_alloc(cap));
        if (!base) cap = 0;
    }
};
thread_local Stager t_stage;

template <class T>
int upload(T* d, const std::vector<T>& h, cudaStream_t st) {
    if (h.empty()) return EZQ_OK;
    const size_t bytes = h.size() * sizeof(T);
    const size_t at = (t_stage.off + 15) & ~size_t(15);
    if (t_stage.base && at + bytes <= t_stage.cap) {
        std::memcpy(t_stage.base + at, h.data(), bytes);
        t_stage.off = at + bytes;
        // SM loads, not the DMA queue: no wait behind bulk H2D copies
        if (int e = ingest_h2d(d, t_stage.base + at, bytes, st)) return e;
    } else {
        EZQ_CK(cudaMemcpyAsync(d, h.data(), bytes, cudaMemcpyHostToDevice, st));
    }
    return EZQ_OK;
}

void free_qweight_arrays(ezq_qweight* q) {
    if (!q || !q->owned) return;
    if (q->mem == EZQ_MEM_DEVICE) {
        // Stream-ordered pool memory: no device-wide synchronisation.
        int dev = 0;
        cudaGetDevice(&dev);
        cudaStream_t st = thread_stream(dev);
        if (q->packed) cudaFreeAsync(q->packed, st);
        if (q->scales) cudaFreeAsync(q->scales, st);
        if (q->outliers) cudaFreeAsync(q->outliers, st);
    } else {
        host_free(q->packed);
        host_free(q->scales);
        host_free(q->outliers);
    }
    q->packed = nullptr;
    q->scales = nullptr;
    q->outliers = nullptr;
}

}  // namespace

// ---------------------------------------------------------------------------
// `d2h` (host outputs only): when non-null the artifact copies to host run
// on that stream and the call returns without waiting for them (the caller
// synchronizes it) -- the chunked host pipeline overlaps them with the next
// chunk's compute.
// `grid` (ezq_grid_oracle_batch): no artifacts; the brute-force grid oracle
// runs on the K3s tables and the per-column best grid scale / error are
// copied to grid->scale / grid->error (batch column order).
struct GridReq {
    int points;
    double* scale;
    double* error;
};

// reuse / stats_out (batched sigma sweep): the per-tensor stats of an
// earlier call over the same tensors are taken as given and only the
// sigma_n-dependent threshold is recomputed; stats_out receives this call's.
int quantize_batch(const float* const* Ws, const int64_t* rows, const int64_t* cols, int n,
                   const ezq_config* cfg, int mode, int in_mem, int out_mem, void* user_stream,
                   ezq_qweight** outs, int* failed, cudaStream_t d2h = nullptr, const GridReq* grid = nullptr,
                   const TStats* reuse = nullptr, TStats* stats_out = nullptr) {
    if (failed) *failed = -1;
    if (n <= 0) return clear_error();
    for (int i = 0; i < n; ++i) outs[i] = nullptr;
    if (mode < EZQ_MODE_EASYQUANT || mode > EZQ_MODE_OUTLIERS_ONLY)
        return set_error(EZQ_ERR_INVALID_ARGUMENT, "unknown quant mode " + std::to_string(mode));
    // DenseMatrix::validate shape check first (types.cpp:10-12).
    for (int i = 0; i < n; ++i) {
        if (rows[i] <= 0 || cols[i] <= 0) {
            if (failed) *failed = i;
            return set_error(EZQ_ERR_INVALID_ARGUMENT,
                             "matrix shape must be positive, got " + std::to_string(rows[i]) +
                                 "x" + std::to_string(cols[i]));
        }
    }
    std::string cfg_msg;
    const int cfg_status = validate_config(cfg, &cfg_msg);

    int dev;
    if (int s = bind_device(&dev)) return s;
    const DeviceInfo& di = device_info(dev);
    cudaStream_t st = pick_stream(user_stream, dev);

    // ---- sizes & host descriptors ----
    std::vector<TDesc> hd(n);
    std::vector<int64_t> chunk_base(n + 1), dblk_base(n + 1), pblk_base(n + 1);
    int64_t tot_chunks = 0, tot_dblk = 0, tot_pblk = 0, tot_cols = 0, tot_in = 0;
    for (int i = 0; i < n; ++i) {
        const int64_t N = rows[i] * cols[i];
        TDesc& d = hd[i];
        std::memset(&d, 0, sizeof(d));
        d.rows = rows[i];
        d.cols = cols[i];
        d.n = N;
        d.chunk_base = chunk_base[i] = tot_chunks;
        d.n_chunks = ceil_div(N, kStatsChunk);
        tot_chunks += d.n_chunks;
        d.dblk_base = dblk_base[i] = tot_dblk;
        d.n_dblk = ceil_div(N, kDetectBlock);
        tot_dblk += d.n_dblk;
        d.pblk_base = pblk_base[i] = tot_pblk;
        tot_pblk += ceil_div(N, kPackBlock);
        d.col_base = tot_cols;
        tot_cols += cols[i];
        // K3b packs unless k = 4 nibble pairs could straddle rows (odd cols)
        d.pack_fused = (cfg_status == EZQ_OK && (cfg->bits != 4 || cols[i] % 2 == 0)) ? 1 : 0;
        if (in_mem == EZQ_MEM_HOST) tot_in += N;
    }
    chunk_base[n] = tot_chunks;
    dblk_base[n] = tot_dblk;
    pblk_base[n] = tot_pblk;

    trace("qb: descriptors done");
    // ---- K3 plans: one launch per distinct row count ----
    const bool eq = mode == EZQ_MODE_EASYQUANT;
    std::map<int64_t, std::vector<int>> by_rows;
    for (int i = 0; i < n; ++i) by_rows[rows[i]].push_back(i);
    struct Plan {
        K3Launch kl;
        std::vector<K3Group> groups;
        size_t goff = 0;
        int grid = 0;
        int sorted_cpb = 0;  // > 0: K3s (sorted columns), columns per CTA
    };
    static const bool k3_sorted = std::getenv("EZQ_K3_STREAMING") == nullptr;  // A/B: streaming K3 only
    std::vector<Plan> plans;
    size_t tot_groups = 0, gstrip_floats = 0, k3s_work = 0;
    static const size_t k3s_work_env = [] {
        const char* e = std::getenv("EZQ_K3S_WORK_MB");
        return (e ? static_cast<size_t>(std::atoll(e)) : size_t(8192)) << 20;
    }();
    // The tables may take at most a sixteenth of the device memory (>= 128 MB;
    // smaller buffers only mean more, shorter waves). Total, not free, memory:
    // cudaMemGetInfo per call was measured to stall some calls by 20-60 ms.
    const size_t k3s_work_cap =
        std::min(k3s_work_env, std::max<size_t>(size_t(128) << 20, di.total_mem / 16));
    if (cfg_status == EZQ_OK) {
        for (auto& kv : by_rows) {
            Plan p;
            const int pieces = k3s_pieces(kv.first);
            if ((k3_sorted || grid) && eq && pieces > 0 && k3s_supported(cfg->bits)) {
                // K3s: a CTA sorts a group of columns (one row piece), then a
                // loop kernel runs the columns' Adam loops on the tables.
                const int64_t pr = k3s_piece_rows(kv.first);
                const int cpb = k3s_cpb(pr);
                p.sorted_cpb = cpb;
                const size_t per_group = k3s_slot_bytes(pr) * cpb;
                p.kl.rows = kv.first;
                for (int i : kv.second)
                    for (int64_t c0 = 0; c0 < cols[i]; c0 += cpb)
                        for (int q = 0; q < pieces; ++q)
                            p.groups.push_back({i, static_cast<int32_t>(c0),
                                                static_cast<int32_t>(std::min<int64_t>(cpb, cols[i] - c0)),
                                                static_cast<int32_t>(q * pr)});
                p.goff = tot_groups;
                tot_groups += p.groups.size();
                p.grid = static_cast<int>(p.groups.size());
                const size_t wave_groups =
                    std::max<size_t>(pieces, std::min<size_t>(p.groups.size(), k3s_work_cap / per_group));
                k3s_work = std::max(k3s_work, per_group * wave_groups + 512);
                plans.push_back(std::move(p));
                continue;
            }
            p.kl = plan_k3(kv.first, 0, di.sms, di.max_smem_optin);
            const int best_cb = choose_k3_width(p.kl, kv.second, cols, di);
            set_k3_width(p.kl, best_cb);
            for (int i : kv.second)
                for (int64_t c0 = 0; c0 < cols[i]; c0 += best_cb)
                    p.groups.push_back({i, static_cast<int32_t>(c0),
                                        static_cast<int32_t>(std::min<int64_t>(best_cb, cols[i] - c0)),
                                        0});
            p.goff = tot_groups;
            tot_groups += p.groups.size();
            p.grid = static_cast<int>(p.groups.size());
            if (p.kl.global_strip) {
                p.grid = std::min<int>(p.grid, di.sms * 2);
                gstrip_floats = std::max(gstrip_floats, static_cast<size_t>(p.grid) *
                                                            p.kl.teams * p.kl.rstride);
            }
            plans.push_back(std::move(p));
        }
    }
    // 32-column tiles for K3b.
    std::vector<int2> tiles;
    for (int i = 0; i < n; ++i)
        for (int64_t c0 = 0; c0 < cols[i]; c0 += 32) tiles.push_back(make_int2(i, (int)c0));
    // longest columns first: a K3b warp walks its tile's rows, so the tall
    // tensors' tiles go into the first waves instead of forming the tail
    std::stable_sort(tiles.begin(), tiles.end(),
                     [&](const int2& a, const int2& b) { return rows[a.x] > rows[b.x]; });
    std::vector<double> bc;
    bias_tables(cfg, bc);

    trace("qb: plans done");
    // ---- arena ----
    Arena ar;
    ar.reserve(sizeof(TStats) * n);
    ar.reserve(sizeof(TDesc) * n);
    for (int k = 0; k < 3; ++k) ar.reserve_n<int64_t>(n + 1);
    for (int k = 0; k < 3; ++k) ar.reserve_n<double>(tot_chunks);
    for (int k = 0; k < 2; ++k) ar.reserve_n<float>(tot_chunks);
    for (int k = 0; k < 2; ++k) ar.reserve_n<long long>(tot_dblk);
    ar.reserve_n<int32_t>(tot_dblk * (kDetectBlock / kDetectSeg));
    for (int k = 0; k < 5; ++k) ar.reserve_n<double>(tot_cols);
    ar.reserve_n<float>(tot_cols);
    ar.reserve_n<uint8_t>(tot_cols);
    ar.reserve_n<int32_t>(tot_cols);
    for (int k = 0; k < 2; ++k) ar.reserve_n<double>(tot_cols * kTieMax);
    ar.reserve_n<int2>(tiles.size());
    ar.reserve(sizeof(double) * bc.size());
    ar.reserve(sizeof(K3Group) * tot_groups);
    ar.reserve(sizeof(float) * tot_in);
    ar.reserve(sizeof(float) * gstrip_floats);
    ar.reserve(k3s_work);
    if (int s = ar.allocate(st)) return s;
    TStats* d_stats = ar.take<TStats>(n);
    TDesc* d_desc = ar.take<TDesc>(n);
    int64_t* d_chunk_base = ar.take<int64_t>(n + 1);
    int64_t* d_dblk_base = ar.take<int64_t>(n + 1);
    int64_t* d_pblk_base = ar.take<int64_t>(n + 1);
    Scratch sc;
    sc.p_sum = ar.take<double>(tot_chunks);
    sc.p_max = ar.take<double>(tot_chunks);
    sc.p_dev = ar.take<double>(tot_chunks);
    sc.p_mn = ar.take<float>(tot_chunks);
    sc.p_mx = ar.take<float>(tot_chunks);
    sc.blk_count = ar.take<long long>(tot_dblk);
    sc.blk_offset = ar.take<long long>(tot_dblk);
    sc.seg_off = ar.take<int32_t>(tot_dblk * (kDetectBlock / kDetectSeg));
    sc.s_rtn = ar.take<double>(tot_cols);
    sc.s_fin = ar.take<double>(tot_cols);
    sc.err_rtn = ar.take<double>(tot_cols);
    sc.err_fin = ar.take<double>(tot_cols);
    sc.inv = ar.take<double>(tot_cols);
    sc.invf = ar.take<float>(tot_cols);
    sc.repack = ar.take<uint8_t>(tot_cols);
    sc.tie_n = ar.take<int32_t>(tot_cols);
    sc.tie_s = ar.take<double>(tot_cols * kTieMax);
    sc.tie_e = ar.take<double>(tot_cols * kTieMax);
    double* d_bc = ar.take<double>(bc.size());
    K3Group* d_groups = ar.take<K3Group>(tot_groups);
    float* d_in = ar.take<float>(tot_in);
    float* d_gstrip = ar.take<float>(gstrip_floats);
    void* d_k3s_work = ar.take<unsigned char>(k3s_work);
    int2* d_tiles = ar.take<int2>(tiles.size());
    if (!ar.ok()) return set_error(EZQ_ERR_CUDA, "internal: arena overflow (quantize_batch)");

    trace("qb: arena done");
    // ---- inputs ----
    int64_t in_off = 0;
    for (int i = 0; i < n; ++i) {
        hd[i].st = d_stats + i;
        if (in_mem == EZQ_MEM_HOST) {
            float* dst = d_in + in_off;
            EZQ_CK(cudaMemcpyAsync(dst, Ws[i], sizeof(float) * hd[i].n, cudaMemcpyHostToDevice, st));
            hd[i].W = dst;
            in_off += hd[i].n;
        } else {
            hd[i].W = Ws[i];
        }
    }
    bool all_aligned = true;
    for (int i = 0; i < n; ++i) all_aligned &= (reinterpret_cast<uintptr_t>(hd[i].W) & 15) == 0;
    {
        size_t need = 64 * 16 + sizeof(TStats) * n + 2 * sizeof(TDesc) * n + 3 * sizeof(int64_t) * (n + 1) +
                      sizeof(double) * bc.size() + sizeof(int2) * tiles.size();
        for (auto& p : plans) need += sizeof(K3Group) * p.groups.size();
        t_stage.reset(need);
    }
    std::vector<TStats> hs(n, fresh_stats());
    if (reuse)
        for (int i = 0; i < n; ++i) {  // the sigma-independent stats; per-call fields fresh
            hs[i].sum = reuse[i].sum;
            hs[i].max_abs = reuse[i].max_abs;
            hs[i].mean = reuse[i].mean;
            hs[i].stddev = reuse[i].stddev;
            hs[i].ss = reuse[i].ss;
            hs[i].mn = reuse[i].mn;
            hs[i].mx = reuse[i].mx;
            hs[i].constant = reuse[i].constant;
        }
    if (int s = upload(d_stats, hs, st)) return s;
    if (int s = upload(d_desc, hd, st)) return s;
    if (int s = upload(d_chunk_base, chunk_base, st)) return s;
    if (int s = upload(d_dblk_base, dblk_base, st)) return s;
    if (int s = upload(d_pblk_base, pblk_base, st)) return s;
    if (int s = upload(d_bc, bc, st)) return s;
    if (int s = upload(d_tiles, tiles, st)) return s;
    for (auto& p : plans) {
        if (p.groups.empty()) continue;
        if (int s = upload(d_groups + p.goff, p.groups, st)) return s;
    }

    trace("qb: inputs done");
    // ---- phase 1 ----
    int64_t tot_elems = 0;
    for (int i = 0; i < n; ++i) tot_elems += hd[i].n;
    int pt = prof_begin("stats", st);
    if (reuse && cfg_status == EZQ_OK) {
        launch_stats_rethreshold(d_desc, n, cfg->sigma_n, mode != EZQ_MODE_RTN, st);
    } else {
        launch_stats_pass1(d_desc, d_chunk_base, n, tot_chunks, sc, st, all_aligned);
        launch_stats_fin1(d_desc, n, sc, st);
    }
    if (cfg_status == EZQ_OK) {
        if (!reuse) {
            launch_stats_pass2(d_desc, d_chunk_base, n, tot_chunks, sc, st, all_aligned);
            launch_stats_fin2(d_desc, n, sc, cfg->sigma_n, mode != EZQ_MODE_RTN, st);
        }
        prof_end(pt, st, reuse ? 0.0 : 8.0 * tot_elems);  // two reads of W
        if (mode != EZQ_MODE_RTN) {
            pt = prof_begin("detect", st);
            launch_detect_count(d_desc, d_dblk_base, n, tot_dblk, sc, st);
            launch_detect_scan(d_desc, n, sc, st);
            prof_end(pt, st, 4.0 * tot_elems);
        }
    } else {
        prof_end(pt, st, 4.0 * tot_elems);
    }
    EZQ_CK(cudaGetLastError());
    EZQ_CK(cudaMemcpyAsync(hs.data(), d_stats, sizeof(TStats) * n, cudaMemcpyDeviceToHost, st));
    trace("phase1 sync begin", n);
    EZQ_CK(cudaStreamSynchronize(st));
    trace("phase1 sync end", n);
    for (int i = 0; i < n; ++i) {
        if (hs[i].bad_index != kNoBad) {  // types.cpp:17-20
            if (failed) *failed = i;
            return set_error(EZQ_ERR_INVALID_ARGUMENT,
                             "non-finite element at flat index " + std::to_string(hs[i].bad_index),
                             static_cast<int64_t>(hs[i].bad_index));
        }
    }
    if (cfg_status != EZQ_OK) return set_error(cfg_status, cfg_msg);
    if (stats_out)
        for (int i = 0; i < n; ++i) stats_out[i] = hs[i];
    if (mode != EZQ_MODE_RTN) {
        for (int i = 0; i < n; ++i)
            if (rows[i] > UINT32_MAX || cols[i] > UINT32_MAX) {  // outliers.cpp:30-31
                if (failed) *failed = i;
                return set_error(EZQ_ERR_INVALID_ARGUMENT,
                                 "matrix dimensions exceed 32-bit coordinate range");
            }
    }

    trace("qb: phase1 checked");
    if (grid) {  // ---- grid oracle: tables + grid scan, no artifacts ----
        const CfgDev cd = make_cfg(cfg, mode, d_bc);
        for (auto& p : plans) {
            if (!p.sorted_cpb)
                return set_error(EZQ_ERR_INVALID_ARGUMENT, "grid oracle needs the sorted-column path (k <= 5, "
                                                           "rows <= 65536)");
            launch_k3_sorted(p.kl.rows, p.sorted_cpb, d_desc, d_groups + p.goff, static_cast<int>(p.groups.size()),
                             sc, cd, d_k3s_work, k3s_work, st, grid->points);
        }
        EZQ_CK(cudaGetLastError());
        EZQ_CK(cudaMemcpyAsync(grid->scale, sc.s_fin, sizeof(double) * tot_cols, cudaMemcpyDeviceToHost, st));
        EZQ_CK(cudaMemcpyAsync(grid->error, sc.err_fin, sizeof(double) * tot_cols, cudaMemcpyDeviceToHost, st));
        EZQ_CK(cudaStreamSynchronize(st));
        return clear_error();
    }
    // ---- outputs (device) ----
    struct Out {
        uint8_t* packed = nullptr;
        float* scales = nullptr;
        ezq_outlier* outl = nullptr;
    };
    std::vector<Out> dout(n);
    auto free_dout = [&]() {
        for (auto& o : dout) {
            if (o.packed) cudaFreeAsync(o.packed, st);
            if (o.scales) cudaFreeAsync(o.scales, st);
            if (o.outl) cudaFreeAsync(o.outl, st);
            o = Out{};
        }
    };
    for (int i = 0; i < n; ++i) {
        const int64_t pb = ezq_packed_size(hd[i].n, cfg->bits);
        cudaError_t e1 = cudaMallocAsync(&dout[i].packed, std::max<int64_t>(pb, 1), st);
        cudaError_t e2 = cudaMallocAsync(&dout[i].scales, sizeof(float) * cols[i], st);
        cudaError_t e3 = cudaSuccess;
        if (hs[i].n_out > 0) e3 = cudaMallocAsync(&dout[i].outl, sizeof(ezq_outlier) * hs[i].n_out, st);
        if (e1 != cudaSuccess || e2 != cudaSuccess || e3 != cudaSuccess) {
            free_dout();
            return cuda_error(cudaErrorMemoryAllocation, "output allocation");
        }
        hd[i].packed = dout[i].packed;
        hd[i].scales = dout[i].scales;
        hd[i].outliers = dout[i].outl;
    }
    if (int s = upload(d_desc, hd, st)) {
        free_dout();
        return s;
    }

    trace("qb: outputs allocated");
    // ---- phase 2 ----
    const CfgDev cd = make_cfg(cfg, mode, d_bc);
    EZQ_CK(cudaMemsetAsync(sc.tie_n, 0, sizeof(int32_t) * tot_cols, st));  // streaming-K3 columns: certified
    int64_t tot_out = 0;
    for (int i = 0; i < n; ++i) tot_out += hs[i].n_out;
    if (mode != EZQ_MODE_RTN) {
        const int p2 = prof_begin("detect", st);
        launch_detect_write(d_desc, d_dblk_base, n, tot_dblk, sc, st);
        prof_end(p2, st, 4.0 * tot_elems + 12.0 * tot_out);
    }
    trace("qb: detect launched");
    for (auto& p : plans) {
        // Algorithmic work: 7 flop (1 DMUL + 3 DFMA) per normal element-step.
        double normals = 0.0;
        for (auto& g : p.groups) (void)g;
        for (int i = 0; i < n; ++i)
            if (rows[i] == p.kl.rows) normals += static_cast<double>(hd[i].n - hs[i].n_out);
        const double steps1 = (mode == EZQ_MODE_EASYQUANT) ? cfg->steps + 1.0 : 0.0;
        if (p.sorted_cpb) {  // profiled inside ("qsort" / "qrange")
            launch_k3_sorted(p.kl.rows, p.sorted_cpb, d_desc, d_groups + p.goff, static_cast<int>(p.groups.size()),
                             sc, cd, d_k3s_work, k3s_work, st);
        } else {
            const int p3 = prof_begin("qrange_stream", st);
            launch_k3(p.kl, d_desc, d_groups + p.goff, static_cast<int>(p.groups.size()), sc, cd,
                      d_gstrip, p.grid, st);
            prof_end(p3, st, 7.0 * normals * steps1);
        }
        trace("qb: k3 plan launched", p.kl.rows);
    }
    int p4 = prof_begin("seqerr", st);
    launch_resolve_ties(d_desc, d_tiles, static_cast<int>(tiles.size()), sc, cd, st);
    launch_seq_errors(d_desc, d_tiles, static_cast<int>(tiles.size()), sc, cd, st);
    static const bool force_repack = std::getenv("EZQ_FORCE_REPACK") != nullptr;  // test aid: exercise k_repack
    if (force_repack) EZQ_CK(cudaMemsetAsync(sc.repack, 1, tot_cols, st));
    launch_repack(d_desc, d_tiles, static_cast<int>(tiles.size()), sc, cd, st);
    launch_tensor_totals(d_desc, n, sc, st);
    prof_end(p4, st, 4.0 * tot_elems);
    trace("qb: seqerr launched");
    int64_t tot_packed = 0;
    for (int i = 0; i < n; ++i) tot_packed += ezq_packed_size(hd[i].n, cfg->bits);
    p4 = prof_begin("pack", st);
    bool any_unfused = false;
    for (int i = 0; i < n; ++i) any_unfused |= hd[i].pack_fused == 0;
    if (any_unfused) launch_pack(d_desc, d_pblk_base, n, tot_pblk, sc, cd, st);
    prof_end(p4, st, 4.0 * tot_elems + static_cast<double>(tot_packed));
    {
        cudaError_t e = cudaGetLastError();
        if (e != cudaSuccess) {
            free_dout();
            return cuda_error(e, "phase-2 launch");
        }
    }
    EZQ_CK(cudaMemcpyAsync(hs.data(), d_stats, sizeof(TStats) * n, cudaMemcpyDeviceToHost, st));

    trace("qb: phase2 launched");
    // ---- results ----
    std::vector<std::unique_ptr<ezq_qweight>> res(n);
    cudaStream_t ost = st;  // stream of the output copies
    if (d2h && out_mem == EZQ_MEM_HOST) {
        cudaEvent_t ev;
        cudaEventCreateWithFlags(&ev, cudaEventDisableTiming);
        cudaEventRecord(ev, st);
        cudaStreamWaitEvent(d2h, ev, 0);
        cudaEventDestroy(ev);
        ost = d2h;
    }
    for (int i = 0; i < n; ++i) {
        res[i].reset(static_cast<ezq_qweight*>(std::calloc(1, sizeof(ezq_qweight))));
        ezq_qweight* q = res[i].get();
        q->rows = rows[i];
        q->cols = cols[i];
        q->bits = cfg->bits;
        q->mem = out_mem;
        q->owned = 1;
        q->packed_bytes = ezq_packed_size(hd[i].n, cfg->bits);
        if (out_mem == EZQ_MEM_HOST) {
            q->packed = static_cast<uint8_t*>(host_alloc(std::max<int64_t>(q->packed_bytes, 1)));
            q->scales = static_cast<float*>(host_alloc(sizeof(float) * cols[i]));
            q->outliers = hs[i].n_out > 0 ? static_cast<ezq_outlier*>(
                                                host_alloc(sizeof(ezq_outlier) * hs[i].n_out))
                                          : nullptr;
            cudaMemcpyAsync(q->packed, dout[i].packed, q->packed_bytes, cudaMemcpyDeviceToHost, ost);
            cudaMemcpyAsync(q->scales, dout[i].scales, sizeof(float) * cols[i],
                            cudaMemcpyDeviceToHost, ost);
            if (hs[i].n_out > 0)
                cudaMemcpyAsync(q->outliers, dout[i].outl, sizeof(ezq_outlier) * hs[i].n_out,
                                cudaMemcpyDeviceToHost, ost);
        } else {
            q->packed = dout[i].packed;
            q->scales = dout[i].scales;
            q->outliers = dout[i].outl;
        }
    }
    if (out_mem == EZQ_MEM_HOST && ost != st) {
        for (auto& o : dout) {  // freed after the deferred copies
            if (o.packed) cudaFreeAsync(o.packed, ost);
            if (o.scales) cudaFreeAsync(o.scales, ost);
            if (o.outl) cudaFreeAsync(o.outl, ost);
            o = Out{};
        }
    }
    trace("phase2 sync begin", n);
    cudaError_t se = cudaStreamSynchronize(st);
    trace("phase2 sync end", n);
    if (out_mem == EZQ_MEM_HOST) free_dout();
    auto drain = [&]() {  // deferred copies must land before their buffers go
        if (ost != st) cudaStreamSynchronize(ost);
    };
    if (se != cudaSuccess) {
        drain();
        for (auto& q : res) free_qweight_arrays(q.get()), std::free(q.release());
        return cuda_error(se, "phase-2 sync");
    }
    for (int i = 0; i < n; ++i) note_ties(hs[i].ties, hs[i].tie_fallback);
    for (int i = 0; i < n; ++i) {
        ezq_qweight* q = res[i].get();
        q->n_outliers = hs[i].n_out;
        q->mean = hs[i].mean;
        q->stddev = hs[i].stddev;
        q->sigma_n = cfg->sigma_n;
        q->has_errors = 1;
        q->rtn_error = hs[i].rtn_error;
        q->final_error = hs[i].final_error;
    }
    for (int i = 0; i < n; ++i) {
        int code = 0;
        std::string msg;
        if (hs[i].scale_zero) {
            code = EZQ_ERR_INVALID_ARGUMENT;
            msg = "scale must be finite and > 0, got " + fmt_double(0.0);
        } else if (hs[i].final_error > hs[i].rtn_error) {  // pipeline.cpp:107-108
            code = EZQ_ERR_INVARIANT;
            msg = "optimized error exceeds round-to-nearest error";
        }
        if (code) {
            drain();
            for (auto& q : res) {
                free_qweight_arrays(q.get());
                std::free(q.release());
            }
            if (failed) *failed = i;
            return set_error(code, msg);
        }
    }
    for (int i = 0; i < n; ++i) outs[i] = res[i].release();
    (void)eq;
    return clear_error();
}

// Host-resident inputs: tensors are processed in chunks of ~kChunkBytes
// whose H2D copies run on a second stream while the previous chunk computes
// (double-buffered device staging), so PCIe time hides behind K3.
int quantize_batch_host(const float* const* Ws, const int64_t* rows, const int64_t* cols, int n,
                        const ezq_config* cfg, int mode, int out_mem, void* user_stream,
                        ezq_qweight** outs, int* failed) {
    // Chunk sizes (overridable for tuning: EZQ_CHUNK_MB / EZQ_FIRST_MB).
    static const int64_t kChunkBytes =
        std::getenv("EZQ_CHUNK_MB") ? (std::atoll(std::getenv("EZQ_CHUNK_MB")) << 20) : (768ll << 20);
    std::vector<std::pair<int, int>> chunks;  // [first, last)
    int64_t max_bytes = 0;
    // The first chunk is small so compute starts after a short ingest; the
    // later ones are 768 MB (LLaMA-7B set host->host on B200: 384 MB chunks
    // 542 ms, 768 MB 489 ms, 1536 MB 498 ms; the pure 25.9 GB H2D copy takes
    // 467 ms, tools/h2d_ceiling.py).
    static const int64_t kFirstBytes = std::getenv("EZQ_FIRST_MB") ? (std::atoll(std::getenv("EZQ_FIRST_MB")) << 20)
                                                                    : (128ll << 20);
    // ... and so is the last: its compute and D2H are the exposed tail.
    static const int64_t kLastBytes = std::getenv("EZQ_LAST_MB") ? (std::atoll(std::getenv("EZQ_LAST_MB")) << 20)
                                                                  : (256ll << 20);
    int tail = n;
    for (int64_t b = 0; tail > 1;) {
        const int64_t tb = 4 * std::max<int64_t>(rows[tail - 1], 0) * std::max<int64_t>(cols[tail - 1], 0);
        if (b + tb > kLastBytes && tail < n) break;
        b += tb;
        --tail;
    }
    for (int i = 0; i < n;) {
        int j = i;
        int64_t bytes = 0;
        const int64_t cap = chunks.empty() ? std::min(kFirstBytes, kChunkBytes) : kChunkBytes;
        const int end = i < tail ? tail : n;
        while (j < end && (j == i || bytes + 4 * rows[j] * cols[j] <= cap)) {
            bytes += 4 * std::max<int64_t>(rows[j], 0) * std::max<int64_t>(cols[j], 0);
            ++j;
        }
        chunks.emplace_back(i, j);
        max_bytes = std::max(max_bytes, bytes);
        i = j;
    }
    if (chunks.size() < 2)
        return quantize_batch(Ws, rows, cols, n, cfg, mode, EZQ_MEM_HOST, out_mem, user_stream, outs,
                              failed);
    for (int i = 0; i < n; ++i) {
        outs[i] = nullptr;
        if (rows[i] <= 0 || cols[i] <= 0)  // same precedence as the one-shot path
            return quantize_batch(Ws, rows, cols, n, cfg, mode, EZQ_MEM_HOST, out_mem, user_stream,
                                  outs, failed);
    }
    int dev;
    if (int s = bind_device(&dev)) return s;
    cudaStream_t st = pick_stream(user_stream, dev);
    cudaStream_t cs = copy_stream(dev);
    float* buf[2] = {nullptr, nullptr};
    size_t buf_cap[2] = {0, 0};
    for (int k = 0; k < 2; ++k) {
        buf[k] = static_cast<float*>(block_get(max_bytes, st, &buf_cap[k]));
        if (!buf[k]) {
            if (k) block_put(buf[0], buf_cap[0], st);
            return cuda_error(cudaErrorMemoryAllocation, "chunk buffers");
        }
    }
    cudaEvent_t in_ready[2], done[2];
    for (int k = 0; k < 2; ++k) {
        cudaEventCreateWithFlags(&in_ready[k], cudaEventDisableTiming);
        cudaEventCreateWithFlags(&done[k], cudaEventDisableTiming);
    }
    EZQ_CK(cudaEventRecord(done[0], st));  // buffers free "now"
    EZQ_CK(cudaEventRecord(done[1], st));
    auto issue_copy = [&](size_t c) -> int {
        const int b = static_cast<int>(c % 2);
        EZQ_CK(cudaStreamWaitEvent(cs, done[b], 0));
        int64_t off = 0;
        for (int i = chunks[c].first; i < chunks[c].second; ++i) {
            const int64_t nb = 4 * rows[i] * cols[i];
            static const bool dma = std::getenv("EZQ_H2D_SM") == nullptr;
            if (dma)
                EZQ_CK(cudaMemcpyAsync(reinterpret_cast<char*>(buf[b]) + off, Ws[i], nb, cudaMemcpyHostToDevice, cs));
            else if (int e = ingest_h2d(reinterpret_cast<char*>(buf[b]) + off, Ws[i], nb, cs))
                return e;
            off += nb;
        }
        EZQ_CK(cudaEventRecord(in_ready[b], cs));
        return EZQ_OK;
    };
    trace("host batch start", static_cast<long long>(chunks.size()));
    int status = issue_copy(0);
    if (!status && chunks.size() > 1) status = issue_copy(1);
    for (size_t c = 0; c < chunks.size() && !status; ++c) {
        const int b = static_cast<int>(c % 2);
        const int i0 = chunks[c].first, i1 = chunks[c].second;
        std::vector<const float*> dW;
        int64_t off = 0;
        for (int i = i0; i < i1; ++i) {
            dW.push_back(reinterpret_cast<const float*>(reinterpret_cast<char*>(buf[b]) + off));
            off += 4 * rows[i] * cols[i];
        }
        if (cudaStreamWaitEvent(st, in_ready[b], 0) != cudaSuccess) {
            status = cuda_error(cudaGetLastError(), "chunk wait");
            break;
        }
        int sub_failed = -1;
        status = quantize_batch(dW.data(), rows + i0, cols + i0, i1 - i0, cfg, mode, EZQ_MEM_DEVICE,
                                out_mem, st, outs + i0, &sub_failed, d2h_stream(dev));
        if (status) {
            if (failed) *failed = sub_failed >= 0 ? i0 + sub_failed : -1;
            // translate device-relative bad indices is unnecessary: flat index is per tensor
            break;
        }
        cudaEventRecord(done[b], st);
        if (c + 2 < chunks.size()) status = issue_copy(c + 2);
    }
    trace("host batch drain");
    cudaStreamSynchronize(cs);
    cudaStreamSynchronize(d2h_stream(dev));  // deferred artifact copies
    trace("host batch end");
    block_put(buf[0], buf_cap[0], st);
    block_put(buf[1], buf_cap[1], st);
    for (int k = 0; k < 2; ++k) {
        cudaEventDestroy(in_ready[k]);
        cudaEventDestroy(done[k]);
    }
    if (status) {
        char msg[1024];
        int64_t idx;
        const int code = ezq_last_error(msg, sizeof msg, &idx);
        for (int i = 0; i < n; ++i) {
            ezq_qweight_free(outs[i]);
            outs[i] = nullptr;
        }
        return set_error(code ? code : status, msg, idx);
    }
    return clear_error();
}

}  // namespace ezq

using namespace ezq;

extern "C" {

int ezq_quantize_batch(const float* const* Ws, const int64_t* rows, const int64_t* cols, int n,
                       const ezq_config* cfg, int mode, int in_mem, int out_mem, void* stream,
                       ezq_qweight** outs, int* failed_index) {
    if (in_mem == EZQ_MEM_HOST && n > 1) {
        std::string msg;
        if (validate_config(cfg, &msg) == EZQ_OK)  // invalid configs take the one-shot path
            return quantize_batch_host(Ws, rows, cols, n, cfg, mode, out_mem, stream, outs,
                                       failed_index);
    }
    return quantize_batch(Ws, rows, cols, n, cfg, mode, in_mem, out_mem, stream, outs,
                          failed_index);
}

int ezq_sigma_sweep_batch(const float* const* Ws, const int64_t* rows, const int64_t* cols, int n,
                          const ezq_config* cfg, int in_mem, void* stream, const float* sigmas, int nsig,
                          int64_t* n_outliers, double* rtn_error, double* final_error, int* failed_index) {
    if (failed_index) *failed_index = -1;
    if (nsig < 0 || (nsig > 0 && (!sigmas || !n_outliers || !rtn_error || !final_error)))
        return set_error(EZQ_ERR_INVALID_ARGUMENT, "sigma sweep: bad sigma list or null output");
    if (n <= 0 || nsig == 0) return clear_error();
    std::vector<ezq_qweight*> q(static_cast<size_t>(n), nullptr);
    std::vector<TStats> saved(static_cast<size_t>(n));
    for (int k = 0; k < nsig; ++k) {
        ezq_config c = *cfg;
        c.sigma_n = sigmas[k];
        // device-resident inputs: the first point computes the stats, the
        // others reuse them (K1 once per sweep); host inputs stream per point
        const bool dev = in_mem == EZQ_MEM_DEVICE;
        const int s = dev ? quantize_batch(Ws, rows, cols, n, &c, EZQ_MODE_EASYQUANT, in_mem, EZQ_MEM_DEVICE, stream,
                                           q.data(), failed_index, nullptr, nullptr, k ? saved.data() : nullptr,
                                           k ? nullptr : saved.data())
                          : ezq_quantize_batch(Ws, rows, cols, n, &c, EZQ_MODE_EASYQUANT, in_mem, EZQ_MEM_DEVICE,
                                               stream, q.data(), failed_index);
        if (s != EZQ_OK) return s;
        for (int i = 0; i < n; ++i) {
            const int64_t o = static_cast<int64_t>(k) * n + i;
            n_outliers[o] = q[i]->n_outliers;
            rtn_error[o] = q[i]->has_errors ? q[i]->rtn_error : 0.0;
            final_error[o] = q[i]->has_errors ? q[i]->final_error : 0.0;
            ezq_qweight_free(q[i]);
            q[i] = nullptr;
        }
    }
    return clear_error();
}

int ezq_grid_oracle_batch(const float* const* Ws, const int64_t* rows, const int64_t* cols, int n,
                          const ezq_config* cfg, int grid_points, int in_mem, void* stream, double* best_scale,
                          double* best_error, int* failed_index) {
    if (grid_points < 2) return set_error(EZQ_ERR_INVALID_ARGUMENT, "grid_points must be >= 2");
    if (!best_scale || !best_error) return set_error(EZQ_ERR_INVALID_ARGUMENT, "null output");
    std::vector<ezq_qweight*> outs(static_cast<size_t>(std::max(n, 1)), nullptr);
    const GridReq g{grid_points, best_scale, best_error};
    return quantize_batch(Ws, rows, cols, n, cfg, EZQ_MODE_EASYQUANT, in_mem, EZQ_MEM_HOST, stream, outs.data(),
                          failed_index, nullptr, &g);
}

int ezq_quantize_tensor(const float* W, int64_t rows, int64_t cols, const ezq_config* cfg,
                        int mode, int in_mem, int out_mem, void* stream, ezq_qweight** out) {
    const float* ws[1] = {W};
    return quantize_batch(ws, &rows, &cols, 1, cfg, mode, in_mem, out_mem, stream, out, nullptr);
}

void ezq_qweight_free(ezq_qweight* q) {
    if (!q) return;
    free_qweight_arrays(q);
    std::free(q);
}

int ezq_qweight_to_host(const ezq_qweight* q, ezq_qweight** out) {
    *out = nullptr;
    ezq_qweight* h = static_cast<ezq_qweight*>(std::calloc(1, sizeof(ezq_qweight)));
    *h = *q;
    h->mem = EZQ_MEM_HOST;
    h->owned = 1;
    h->packed = static_cast<uint8_t*>(host_alloc(std::max<int64_t>(q->packed_bytes, 1)));
    h->scales = static_cast<float*>(host_alloc(sizeof(float) * std::max<int64_t>(q->cols, 1)));
    h->outliers = q->n_outliers ? static_cast<ezq_outlier*>(host_alloc(sizeof(ezq_outlier) * q->n_outliers))
                                : nullptr;
    const cudaMemcpyKind k = q->mem == EZQ_MEM_DEVICE ? cudaMemcpyDeviceToHost : cudaMemcpyHostToHost;
    cudaError_t e = cudaMemcpy(h->packed, q->packed, q->packed_bytes, k);
    if (e == cudaSuccess) e = cudaMemcpy(h->scales, q->scales, sizeof(float) * q->cols, k);
    if (e == cudaSuccess && q->n_outliers)
        e = cudaMemcpy(h->outliers, q->outliers, sizeof(ezq_outlier) * q->n_outliers, k);
    if (e != cudaSuccess) {
        ezq_qweight_free(h);
        return cuda_error(e, "ezq_qweight_to_host");
    }
    *out = h;
    return clear_error();
}

int ezq_qweight_wrap(int64_t rows, int64_t cols, int bits, const uint8_t* packed,
                     int64_t packed_bytes, const float* scales, int64_t n_scales,
                     const ezq_outlier* outliers, int64_t n_outliers, double mean, double stddev,
                     float sigma_n, int mem, ezq_qweight** out) {
    ezq_qweight* q = static_cast<ezq_qweight*>(std::calloc(1, sizeof(ezq_qweight)));
    q->rows = rows;
    q->cols = cols;
    q->bits = bits;
    q->mem = mem;
    q->owned = 0;
    q->packed = const_cast<uint8_t*>(packed);
    q->packed_bytes = packed_bytes;
    q->scales = const_cast<float*>(scales);
    q->reserved = static_cast<int32_t>(n_scales == cols ? 0 : 1);  // scale-count mismatch flag
    q->outliers = const_cast<ezq_outlier*>(outliers);
    q->n_outliers = n_outliers;
    q->mean = mean;
    q->stddev = stddev;
    q->sigma_n = sigma_n;
    *out = q;
    return clear_error();
}

// ---- tensor_stats (stats.cpp:27-108) ---------------------------------------
int ezq_tensor_stats(const float* W, int64_t rows, int64_t cols, int mem, void* stream,
                     ezq_stats* out) {
    std::memset(out, 0, sizeof(*out));
    const int64_t N = rows * cols;
    if (rows <= 0 || cols <= 0 || N <= 0) return clear_error();  // stats.cpp:51
    int dev;
    if (int s = bind_device(&dev)) return s;
    cudaStream_t st = pick_stream(stream, dev);
    TDesc hd;
    std::memset(&hd, 0, sizeof(hd));
    hd.rows = rows;
    hd.cols = cols;
    hd.n = N;
    hd.n_chunks = ceil_div(N, kStatsChunk);
    Arena ar;
    ar.reserve(sizeof(TStats));
    ar.reserve(sizeof(TDesc));
    ar.reserve(2 * sizeof(int64_t));
    for (int k = 0; k < 3; ++k) ar.reserve_n<double>(hd.n_chunks);
    for (int k = 0; k < 2; ++k) ar.reserve_n<float>(hd.n_chunks);
    if (mem == EZQ_MEM_HOST) ar.reserve(sizeof(float) * N);
    if (int s = ar.allocate(st)) return s;
    TStats* d_st = ar.take<TStats>(1);
    TDesc* d_td = ar.take<TDesc>(1);
    int64_t* d_cb = ar.take<int64_t>(2);
    Scratch sc{};
    sc.p_sum = ar.take<double>(hd.n_chunks);
    sc.p_max = ar.take<double>(hd.n_chunks);
    sc.p_dev = ar.take<double>(hd.n_chunks);
    sc.p_mn = ar.take<float>(hd.n_chunks);
    sc.p_mx = ar.take<float>(hd.n_chunks);
    if (mem == EZQ_MEM_HOST) {
        float* dW = ar.take<float>(N);
        EZQ_CK(cudaMemcpyAsync(dW, W, sizeof(float) * N, cudaMemcpyHostToDevice, st));
        hd.W = dW;
    } else {
        hd.W = W;
    }
    hd.st = d_st;
    std::vector<TStats> hs(1, fresh_stats());
    std::vector<TDesc> hdv(1, hd);
    std::vector<int64_t> cb = {0, hd.n_chunks};
    if (int s = upload(d_st, hs, st)) return s;
    if (int s = upload(d_td, hdv, st)) return s;
    if (int s = upload(d_cb, cb, st)) return s;
    launch_stats_pass1(d_td, d_cb, 1, hd.n_chunks, sc, st, (reinterpret_cast<uintptr_t>(hd.W) & 15) == 0);
    launch_stats_fin1(d_td, 1, sc, st);
    launch_stats_pass2(d_td, d_cb, 1, hd.n_chunks, sc, st, (reinterpret_cast<uintptr_t>(hd.W) & 15) == 0);
    launch_stats_fin2(d_td, 1, sc, 0.f, 0, st);
    EZQ_CK(cudaGetLastError());
    EZQ_CK(cudaMemcpyAsync(hs.data(), d_st, sizeof(TStats), cudaMemcpyDeviceToHost, st));
    EZQ_CK(cudaStreamSynchronize(st));
    out->mean = hs[0].mean;
    out->stddev = hs[0].stddev;
    out->max_abs = hs[0].max_abs;
    out->count = N;
    return clear_error();
}

// ---- detect_outliers (outliers.cpp:29-73) ----------------------------------
int ezq_detect_outliers(const float* W, int64_t rows, int64_t cols, const ezq_config* cfg,
                        int mem, void* stream, ezq_outlier** entries, int64_t* n, double* mean,
                        double* stddev) {
    *entries = nullptr;
    *n = 0;
    if (rows > UINT32_MAX || cols > UINT32_MAX)
        return set_error(EZQ_ERR_INVALID_ARGUMENT, "matrix dimensions exceed 32-bit coordinate range");
    const int64_t N = rows * cols;
    if (rows <= 0 || cols <= 0 || N <= 0) {
        *mean = 0.0;
        *stddev = 0.0;
        return clear_error();
    }
    int dev;
    if (int s = bind_device(&dev)) return s;
    cudaStream_t st = pick_stream(stream, dev);
    TDesc hd;
    std::memset(&hd, 0, sizeof(hd));
    hd.rows = rows;
    hd.cols = cols;
    hd.n = N;
    hd.n_chunks = ceil_div(N, kStatsChunk);
    hd.n_dblk = ceil_div(N, kDetectBlock);
    Arena ar;
    ar.reserve(sizeof(TStats));
    ar.reserve(sizeof(TDesc));
    ar.reserve(2 * sizeof(int64_t));
    ar.reserve(2 * sizeof(int64_t));
    for (int k = 0; k < 3; ++k) ar.reserve_n<double>(hd.n_chunks);
    for (int k = 0; k < 2; ++k) ar.reserve_n<float>(hd.n_chunks);
    for (int k = 0; k < 2; ++k) ar.reserve_n<long long>(hd.n_dblk);
    ar.reserve_n<int32_t>(hd.n_dblk * (kDetectBlock / kDetectSeg));
    if (mem == EZQ_MEM_HOST) ar.reserve(sizeof(float) * N);
    if (int s = ar.allocate(st)) return s;
    TStats* d_st = ar.take<TStats>(1);
    TDesc* d_td = ar.take<TDesc>(1);
    int64_t* d_cb = ar.take<int64_t>(2);
    int64_t* d_db = ar.take<int64_t>(2);
    Scratch sc{};
    sc.p_sum = ar.take<double>(hd.n_chunks);
    sc.p_max = ar.take<double>(hd.n_chunks);
    sc.p_dev = ar.take<double>(hd.n_chunks);
    sc.p_mn = ar.take<float>(hd.n_chunks);
    sc.p_mx = ar.take<float>(hd.n_chunks);
    sc.blk_count = ar.take<long long>(hd.n_dblk);
    sc.blk_offset = ar.take<long long>(hd.n_dblk);
    sc.seg_off = ar.take<int32_t>(hd.n_dblk * (kDetectBlock / kDetectSeg));
    if (mem == EZQ_MEM_HOST) {
        float* dW = ar.take<float>(N);
        EZQ_CK(cudaMemcpyAsync(dW, W, sizeof(float) * N, cudaMemcpyHostToDevice, st));
        hd.W = dW;
    } else {
        hd.W = W;
    }
    hd.st = d_st;
    std::vector<TStats> hs(1, fresh_stats());
    std::vector<TDesc> hdv(1, hd);
    std::vector<int64_t> cb = {0, hd.n_chunks}, db = {0, hd.n_dblk};
    if (int s = upload(d_st, hs, st)) return s;
    if (int s = upload(d_td, hdv, st)) return s;
    if (int s = upload(d_cb, cb, st)) return s;
    if (int s = upload(d_db, db, st)) return s;
    launch_stats_pass1(d_td, d_cb, 1, hd.n_chunks, sc, st, (reinterpret_cast<uintptr_t>(hd.W) & 15) == 0);
    launch_stats_fin1(d_td, 1, sc, st);
    launch_stats_pass2(d_td, d_cb, 1, hd.n_chunks, sc, st, (reinterpret_cast<uintptr_t>(hd.W) & 15) == 0);
    launch_stats_fin2(d_td, 1, sc, cfg->sigma_n, 1, st);
    launch_detect_count(d_td, d_db, 1, hd.n_dblk, sc, st);
    launch_detect_scan(d_td, 1, sc, st);
    EZQ_CK(cudaGetLastError());
    EZQ_CK(cudaMemcpyAsync(hs.data(), d_st, sizeof(TStats), cudaMemcpyDeviceToHost, st));
    EZQ_CK(cudaStreamSynchronize(st));
    *mean = hs[0].mean;
    *stddev = hs[0].stddev;
    const int64_t cnt = hs[0].n_out;
    if (cnt > 0) {
        ezq_outlier* d_e = nullptr;
        EZQ_CK(cudaMallocAsync(&d_e, sizeof(ezq_outlier) * cnt, st));
        hdv[0].outliers = d_e;
        if (int s = upload(d_td, hdv, st)) return s;
        launch_detect_write(d_td, d_db, 1, hd.n_dblk, sc, st);
        ezq_outlier* h = static_cast<ezq_outlier*>(std::malloc(sizeof(ezq_outlier) * cnt));
        EZQ_CK(cudaMemcpyAsync(h, d_e, sizeof(ezq_outlier) * cnt, cudaMemcpyDeviceToHost, st));
        cudaFreeAsync(d_e, st);
        EZQ_CK(cudaStreamSynchronize(st));
        *entries = h;
    }
    *n = cnt;
    return clear_error();
}

// ---- dequantize_tensor (pipeline.cpp:117-142) -------------------------------
int ezq_dequantize_tensor(const ezq_qweight* q, float* out, int out_mem, void* stream) {
    if (q->rows <= 0 || q->cols <= 0)
        return set_error(EZQ_ERR_IO_FORMAT, "quantized tensor has empty shape");
    if (q->reserved)  // wrap() saw n_scales != cols
        return set_error(EZQ_ERR_IO_FORMAT, "scale count does not match columns");
    const int64_t N = q->rows * q->cols;
    const int64_t need = ezq_packed_size(N, q->bits);
    if (q->packed_bytes < need)
        return set_error(EZQ_ERR_INVALID_ARGUMENT,
                         "packed buffer holds " + std::to_string(q->packed_bytes) + " bytes, need " +
                             std::to_string(need) + " for " + std::to_string(N) + " levels");
    int dev;
    if (int s = bind_device(&dev)) return s;
    cudaStream_t st = pick_stream(stream, dev);
    Arena ar;
    ar.reserve(2 * sizeof(unsigned long long));
    const bool hin = q->mem == EZQ_MEM_HOST;  // take() order below mirrors reserve()
    if (hin) {
        ar.reserve(need);
        ar.reserve(sizeof(float) * q->cols);
        ar.reserve(sizeof(ezq_outlier) * q->n_outliers);
    }
    if (out_mem == EZQ_MEM_HOST) ar.reserve(sizeof(float) * N);
    if (int s = ar.allocate(st)) return s;
    unsigned long long* d_bad = ar.take<unsigned long long>(2);
    const uint8_t* pk = q->packed;
    const float* sc = q->scales;
    const ezq_outlier* oe = q->outliers;
    if (hin) {
        uint8_t* a = ar.take<uint8_t>(need);
        float* b = ar.take<float>(q->cols);
        ezq_outlier* c = ar.take<ezq_outlier>(q->n_outliers);
        EZQ_CK(cudaMemcpyAsync(a, q->packed, need, cudaMemcpyHostToDevice, st));
        EZQ_CK(cudaMemcpyAsync(b, q->scales, sizeof(float) * q->cols, cudaMemcpyHostToDevice, st));
        if (q->n_outliers)
            EZQ_CK(cudaMemcpyAsync(c, q->outliers, sizeof(ezq_outlier) * q->n_outliers,
                                   cudaMemcpyHostToDevice, st));
        pk = a;
        sc = b;
        oe = c;
    }
    float* dst = out_mem == EZQ_MEM_HOST ? ar.take<float>(N) : out;
    EZQ_CK(cudaMemsetAsync(d_bad, 0xff, 2 * sizeof(unsigned long long), st));
    const int pd = prof_begin("dequant", st);
    launch_dequant(q->rows, q->cols, q->bits, pk, sc, dst, d_bad, st);
    launch_scatter(q->rows, q->cols, oe, q->n_outliers, dst, d_bad + 1, st);
    prof_end(pd, st, static_cast<double>(need) + 4.0 * q->cols + 4.0 * N + 16.0 * q->n_outliers);
    EZQ_CK(cudaGetLastError());
    unsigned long long hb[2];
    EZQ_CK(cudaMemcpyAsync(hb, d_bad, sizeof(hb), cudaMemcpyDeviceToHost, st));
    EZQ_CK(cudaStreamSynchronize(st));
    if (hb[0] != kNoBad) {
        uint8_t byte = 0;
        EZQ_CK(cudaMemcpy(&byte, pk + hb[0], 1, cudaMemcpyDeviceToHost));
        const int lmin = -(1 << (q->bits - 1)) + 1;
        const int span = (1 << (q->bits - 1)) - lmin;
        return set_error(EZQ_ERR_INVALID_ARGUMENT,
                         "packed byte " + std::to_string(byte) + " exceeds level span " +
                             std::to_string(span),
                         static_cast<int64_t>(hb[0]));
    }
    if (hb[1] != kNoBad) {
        ezq_outlier e;
        EZQ_CK(cudaMemcpy(&e, oe + hb[1], sizeof(e), cudaMemcpyDeviceToHost));
        return set_error(EZQ_ERR_INVALID_ARGUMENT,
                         "outlier coordinate (" + std::to_string(e.row) + ", " +
                             std::to_string(e.col) + ") outside " + std::to_string(q->rows) + "x" +
                             std::to_string(q->cols),
                         static_cast<int64_t>(hb[1]));
    }
    if (out_mem == EZQ_MEM_HOST) {
        EZQ_CK(cudaMemcpyAsync(out, dst, sizeof(float) * N, cudaMemcpyDeviceToHost, st));
        EZQ_CK(cudaStreamSynchronize(st));
    }
    return clear_error();
}

// ---- reconstruction_error (rtn.cpp:34-77) -----------------------------------
int ezq_reconstruction_error(const float* a, const float* b, int64_t rows, int64_t cols,
                             const uint32_t* skip_rows, const uint32_t* skip_cols, int64_t n_skip,
                             int mem, void* stream, double* out) {
    *out = 0.0;
    // Column lists in entry order (outlier_rows_by_column, outliers.cpp:75-87).
    std::vector<int64_t> off;
    std::vector<uint32_t> srows;
    if (skip_rows && n_skip > 0) {
        std::vector<int64_t> cnt(static_cast<size_t>(cols) + 1, 0);
        for (int64_t i = 0; i < n_skip; ++i) {
            if (skip_cols[i] >= static_cast<uint64_t>(cols))
                return set_error(EZQ_ERR_INVALID_ARGUMENT,
                                 "outlier column " + std::to_string(skip_cols[i]) +
                                     " out of range for " + std::to_string(cols) + " columns");
            ++cnt[skip_cols[i] + 1];
        }
        for (int64_t c = 0; c < cols; ++c) cnt[c + 1] += cnt[c];
        off = cnt;
        srows.resize(n_skip);
        std::vector<int64_t> pos(cnt.begin(), cnt.end() - 1);
        for (int64_t i = 0; i < n_skip; ++i) srows[pos[skip_cols[i]]++] = skip_rows[i];
    }
    if (rows <= 0 || cols <= 0) return clear_error();
    int dev;
    if (int s = bind_device(&dev)) return s;
    cudaStream_t st = pick_stream(stream, dev);
    const int64_t N = rows * cols;
    Arena ar;
    ar.reserve(sizeof(double) * cols);
    ar.reserve(sizeof(int64_t) * off.size());
    ar.reserve(sizeof(uint32_t) * srows.size());
    if (mem == EZQ_MEM_HOST) {
        ar.reserve(sizeof(float) * N);
        ar.reserve(sizeof(float) * N);
    }
    if (int s = ar.allocate(st)) return s;
    double* d_col = ar.take<double>(cols);
    int64_t* d_off = off.empty() ? nullptr : ar.take<int64_t>(off.size());
    uint32_t* d_rows = srows.empty() ? nullptr : ar.take<uint32_t>(srows.size());
    const float *da = a, *db = b;
    if (mem == EZQ_MEM_HOST) {
        float* x = ar.take<float>(N);
        float* y = ar.take<float>(N);
        EZQ_CK(cudaMemcpyAsync(x, a, sizeof(float) * N, cudaMemcpyHostToDevice, st));
        EZQ_CK(cudaMemcpyAsync(y, b, sizeof(float) * N, cudaMemcpyHostToDevice, st));
        da = x;
        db = y;
    }
    if (d_off) {
        if (int s = upload(d_off, off, st)) return s;
        if (int s = upload(d_rows, srows, st)) return s;
    }
    launch_recon_error(da, db, rows, cols, d_off, d_rows, d_col, st);
    EZQ_CK(cudaGetLastError());
    std::vector<double> col(cols);
    EZQ_CK(cudaMemcpyAsync(col.data(), d_col, sizeof(double) * cols, cudaMemcpyDeviceToHost, st));
    EZQ_CK(cudaStreamSynchronize(st));
    double total = 0.0;
    for (double v : col) total += v;  // column-ordered merge (rtn.cpp:74-75)
    *out = total;
    return clear_error();
}

}  // extern "C"
