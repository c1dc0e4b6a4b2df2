// Host/device-shared descriptors and launchers of every kernel family.
//
// Kernel map (DESIGN.md §3 gives the roofline and algorithmic bytes of each):
//   K1  stats_pass1/2 + finalize   tensor mean/sigma, bit-exact chunk order
//   K2  detect_count/scan/write    n-sigma mask -> flat-ordered COO
//   K3  qrange                     per-column q_range Adam loop, strip in SMEM
//   K3b seq_errors                 reference-order per-column errors, scales
//   K4  pack                       exact final levels -> nibbles/bytes
//   K5  dequant + scatter          dense restore with outliers
//   K6  gemv                       fused dequant + outlier GEMV (k_gemv.cu)
//   Kc  channel kernels            sequential single-channel API (k_channel.cu)
//
// Every kernel works on a *batch* of tensors (the whole-model driver groups
// independent weight matrices into shared launches); a single tensor is a
// batch of one.
#pragma once

#include <cstdint>
#include <cuda_runtime.h>

#include "../../include/ezquant_c.h"
#include "ezq_device.cuh"

namespace ezq {

constexpr int kDetectBlock = 16384;  // elements per detect CTA (256 thr x 64)
constexpr int kDetectSeg = 2048;     // elements per detect warp (contiguous)
constexpr int kPackPerThread = 16;   // elements per pack/dequant thread
constexpr int kPackThreads = 256;
constexpr int64_t kPackBlock = (int64_t)kPackPerThread * kPackThreads;

// Per-tensor state in device memory.
struct TStats {
    double sum;     // pass-1 merged sum
    double max_abs;
    double mean;
    double stddev;
    double thr;     // double(sigma_n) * stddev; +inf when masking is off
    double ss;      // pass-2 merged squared deviations
    float mn, mx;
    int32_t constant;  // mn == mx shortcut (stats.cpp:77-83)
    int32_t mask;      // 1 when outliers are isolated (not Rtn, stddev > 0)
    unsigned long long bad_index;  // first non-finite flat index (~0 = none)
    long long n_out;               // outlier count (K2)
    double rtn_error;              // tensor totals, column-ordered sums
    double final_error;
    int32_t scale_zero;            // a column scale rounded to 0.0f (error)
    int32_t ties;                  // near-tie columns re-evaluated in reference order (k_resolve_ties)
    int32_t tie_fallback;          // ... of which ran the whole reference loop (slots overflowed)
    int32_t pad;
    // Exact float form of the outlier predicate (outliers.cpp:23):
    // |double(v) - mean| >= thr  <=>  v <= olo || v >= ohi  (finite v).
    float olo, ohi;
};

// One tensor of a batch (device pointers).
struct TDesc {
    const float* W;  // row-major rows x cols
    int64_t rows, cols, n;
    TStats* st;
    int64_t chunk_base;  // first global stats chunk
    int64_t n_chunks;
    int64_t dblk_base;   // first global detect block
    int64_t n_dblk;
    int64_t pblk_base;   // first global pack block
    int64_t col_base;    // first global column (per-column arrays)
    // outputs (device)
    uint8_t* packed;
    float* scales;
    ezq_outlier* outliers;
    int32_t pack_fused;  // K3b writes the packed codes (k != 4 or even cols); K4 skips the tensor
    int32_t pad_;
};

// Batch-wide scratch (device pointers into one arena).
struct Scratch {
    // K1
    double* p_sum;
    double* p_max;
    float* p_mn;
    float* p_mx;
    double* p_dev;
    // K2
    long long* blk_count;
    long long* blk_offset;
    int32_t* seg_off;  // [block][kDetectBlock / kDetectSeg]: outliers of the block's earlier segments
    // per-column (global column index)
    double* s_rtn;    // initial scale per column (snapped / float(s0))
    double* s_fin;    // scale chosen by K3 per column
    double* err_rtn;  // reference-order error at s_rtn
    double* err_fin;  // reference-order error at s_fin
    double* inv;      // 1 / double(final float scale), for K4
    float* invf;      // float(inv), K4's certified fp32 level
    uint8_t* repack;  // 1: K3b packed at s_fin but stored s_rtn (re-packed by k_repack)
    // Selection near-ties (K3s loop -> k_resolve_ties): per
    // column the count of candidate scales whose exact errors lie within the
    // reference's sequential-sum rounding of the best (0 = certified), with
    // kTieFixed for a fixed-step comparison; kTieMax slots of candidate scale
    // and approximate full error, in step order.
    int32_t* tie_n;
    double* tie_s;
    double* tie_e;
};
constexpr int kTieMax = 32;  // candidate slots per column (a bit mask in k_resolve_ties)
constexpr int kTieFixed = 1 << 20;

struct CfgDev {
    int bits, lmin, lmax, mode;  // mode: EZQ_MODE_*
    int steps, select, fixed_at, pad;
    float sigma_n, guard;
    float guard_sat;  // K3 saturating-FFMA level guard (level_guard_sat)
    float sat_b;      // RN32(-lmin / span)
    int tie_cap;      // candidate slots used per column (<= kTieMax; 0 = no near-tie resolution)
    AdamConsts adam;
    const double* bc1;  // [steps+1], index t
    const double* bc2;
    const double* rbc1;  // RN(1 / bc1[t]), RN(1 / bc2[t])
    const double* rbc2;
};

// ---- K3 work decomposition -------------------------------------------------
struct K3Group {
    int32_t tensor;
    int32_t col0;
    int32_t ncols;
    int32_t row0;  // K3s row piece: first row (0 for the streaming K3)
};

struct K3Launch {
    int L, W;          // lanes per column, warps per team
    int teams;         // columns per CTA (CB)
    int threads;       // CTA size
    int64_t rows;      // common row count of the launch
    int rpad;          // rows padded to a multiple of 4*L*W
    int rstride;       // floats between column strips in SMEM (rpad + 4)
    size_t smem;       // dynamic SMEM bytes
    bool global_strip; // strip too large for SMEM: stage in global scratch
};

// ---- launchers (defined in the .cu files; all asynchronous on `st`) -------
// `aligned`: every tensor base is 16-byte aligned (enables the cp.async path).
void launch_stats_pass1(const TDesc* td, const int64_t* chunk_base, int ntens,
                        int64_t total_chunks, Scratch sc, cudaStream_t st, bool aligned);
void launch_stats_fin1(const TDesc* td, int ntens, Scratch sc, cudaStream_t st);
void launch_stats_pass2(const TDesc* td, const int64_t* chunk_base, int ntens,
                        int64_t total_chunks, Scratch sc, cudaStream_t st, bool aligned);
void launch_stats_rethreshold(const TDesc* td, int ntens, float sigma_n, int mask_mode, cudaStream_t st);
void launch_stats_fin2(const TDesc* td, int ntens, Scratch sc, float sigma_n, int mask_mode,
                       cudaStream_t st);
void launch_detect_count(const TDesc* td, const int64_t* dblk_base, int ntens,
                         int64_t total_blocks, Scratch sc, cudaStream_t st);
void launch_detect_scan(const TDesc* td, int ntens, Scratch sc, cudaStream_t st);
void launch_detect_write(const TDesc* td, const int64_t* dblk_base, int ntens,
                         int64_t total_blocks, Scratch sc, cudaStream_t st);

K3Launch plan_k3(int64_t rows, int64_t total_cols_hint, int num_sms, int max_smem);
size_t k3_smem(const K3Launch& kl, int teams);
size_t k3_small_smem(const K3Launch& kl, int teams);
void set_k3_width(K3Launch& kl, int teams);
void launch_k3(const K3Launch& kl, const TDesc* td, const K3Group* groups, int ngroups,
               Scratch sc, CfgDev cfg, float* gstrip, int grid, cudaStream_t st);
// K3s (k_qsort.cu): sorted-column q_range loop. Columns longer than
// kK3sPieceRows are sorted in k3s_pieces(rows) independent row pieces whose
// counts and sums add. A sort kernel writes per-piece tables into `work`, a
// loop kernel reads them; groups are processed in waves that fit work_bytes.
constexpr int64_t kK3sPieceRows = 8192;
constexpr int kK3sMaxPieces = 8;
int k3s_pieces(int64_t rows);            // 0: not supported (use the streaming K3)
int64_t k3s_piece_rows(int64_t rows);    // rows of a (full) piece
int k3s_npad(int64_t rows);
bool k3s_supported(int bits);
int k3s_cpb(int64_t piece_rows);         // columns per sort CTA (group width)
size_t k3s_slot_bytes(int64_t piece_rows);  // table + info bytes per column piece
// groups: for every column group, `pieces` consecutive entries (row0 = 0,
// piece_rows, 2 piece_rows, ...).
// grid_points > 0: run the brute-force grid oracle on the tables instead of
// the Adam loop (best grid scale / error per column into s_fin / err_fin).
void launch_k3_sorted(int64_t rows, int cpb, const TDesc* td, const K3Group* groups, int ngroups, Scratch sc,
                      CfgDev cfg, void* work, size_t work_bytes, cudaStream_t st, int grid_points = 0);
void launch_seq_errors(const TDesc* td, const int2* tiles, int ntiles, Scratch sc, CfgDev cfg,
                       cudaStream_t st);
// Re-evaluates the K3s loop's uncertified near-tie columns in reference order
// (sc.tie_*), fixing s_fin before K3b. Streaming-K3 columns carry tie_n = 0.
void launch_resolve_ties(const TDesc* td, const int2* tiles, int ntiles, Scratch sc, CfgDev cfg, cudaStream_t st);
// Re-packs the (rare) fused-pack columns whose stored scale is s_rtn.
void launch_repack(const TDesc* td, const int2* tiles, int ntiles, Scratch sc, CfgDev cfg, cudaStream_t st);
void launch_tensor_totals(const TDesc* td, int ntens, Scratch sc, cudaStream_t st);
void launch_pack(const TDesc* td, const int64_t* pblk_base, int ntens, int64_t total_blocks,
                 Scratch sc, CfgDev cfg, cudaStream_t st);

// K5: dense restore of one tensor; bad_index receives the first flat index of
// an out-of-span byte (k != 4) or the first out-of-bounds outlier entry.
void launch_dequant(int64_t rows, int64_t cols, int bits, const uint8_t* packed,
                    const float* scales, float* out, unsigned long long* bad_byte,
                    cudaStream_t st);
void launch_scatter(int64_t rows, int64_t cols, const ezq_outlier* e, int64_t n, float* out,
                    unsigned long long* bad_entry, cudaStream_t st);

// Kc: sequential single-channel kernels.
void launch_channel_eval(const float* x, int64_t n, const double* scales, int nscales,
                         CfgDev cfg, double* err, double* grad, cudaStream_t st);
void launch_optimize_channels(const float* x, const int64_t* offsets, int nch, CfgDev cfg,
                              int keep_trace, double* out, double* trace, cudaStream_t st);
void launch_recon_error(const float* a, const float* b, int64_t rows, int64_t cols,
                        const int64_t* skip_off, const uint32_t* skip_rows, double* col_sum,
                        cudaStream_t st);
void launch_quantize_channel(const float* x, int64_t n, double scale, CfgDev cfg,
                             int16_t* levels, cudaStream_t st);

// Instrumentation: kernels launched by this process.
void count_launch(int n = 1);
// Instrumentation: near-tie columns resolved (ezq_tie_stats).
void note_ties(int64_t resolved, int64_t fallback);
// Host (page-locked) -> device copy by SM loads (k_ingest), DMA fallback.
int ingest_h2d(void* dst, const void* src, size_t bytes, cudaStream_t st);
// Optional per-family device timing (ezq_profile_enable): returns a token to
// pass to prof_end, or -1 when profiling is off.
int prof_begin(const char* family, cudaStream_t st);
void prof_end(int token, cudaStream_t st, double work);

}  // namespace ezq
