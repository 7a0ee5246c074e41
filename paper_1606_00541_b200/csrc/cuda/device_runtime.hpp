#pragma once
// Device-side objects behind the C-ABI handles: a prepared triangle (DeviceTri),
// an L+U preconditioner with optional RAS gather/scatter (DevicePrecond) and a
// CSR operator (DeviceSpmv). All are immutable after construction and safe for
// concurrent use from several streams (per-stream workspaces).

#include <cuda_runtime.h>

#include <map>
#include <memory>
#include <mutex>
#include <stdexcept>
#include <string>
#include <vector>

#include "tri_plan.hpp"

namespace hec::dev {

[[noreturn]] void cuda_fail(cudaError_t e, const char* what, const char* file, int line);
#define HEC_CUDA(x)                                                   \
    do {                                                              \
        cudaError_t e_ = (x);                                         \
        if (e_ != cudaSuccess) ::hec::dev::cuda_fail(e_, #x, __FILE__, __LINE__); \
    } while (0)

// Throws std::runtime_error unless a CUDA device is usable.
void require_device();

template <class T>
struct DevBuf {
    T* p = nullptr;
    std::size_t count = 0;
    DevBuf() = default;
    explicit DevBuf(std::size_t n) { alloc(n); }
    DevBuf(const DevBuf&) = delete;
    DevBuf& operator=(const DevBuf&) = delete;
    DevBuf(DevBuf&& o) noexcept : p(o.p), count(o.count) { o.p = nullptr; o.count = 0; }
    DevBuf& operator=(DevBuf&& o) noexcept {
        if (this != &o) { release(); p = o.p; count = o.count; o.p = nullptr; o.count = 0; }
        return *this;
    }
    ~DevBuf() { release(); }
    void alloc(std::size_t n) {
        release();
        count = n;
        if (n) HEC_CUDA(cudaMalloc(reinterpret_cast<void**>(&p), n * sizeof(T)));
    }
    void upload(const T* src, std::size_t n) {
        alloc(n);
        if (n) HEC_CUDA(cudaMemcpy(p, src, n * sizeof(T), cudaMemcpyHostToDevice));
    }
    void upload(const std::vector<T>& v) { upload(v.data(), v.size()); }
    void release() {
        if (p) cudaFree(p);
        p = nullptr;
        count = 0;
    }
};

struct TriOptions {
    int strategy = 0;  // 0 auto, 1 levels, 2 pipeline
    int ctas = 0;      // 0 = number of SMs
    int threads = 0;   // solver threads per CTA (128 | 256), 0 = auto
};

struct TriStats {
    int n = 0, nlev = 0, strategy = 0, ctas = 0, threads = 0, chunks = 0, slots = 0;
    int layout = -1, group = 0, groups = 0, rpl = 0, width = 0, ring = 0, halo_ring = 0;
    long long nnz = 0, device_bytes = 0, wave_len = 0;
    double alg_bytes = 0.0, predicted_us = 0.0;
};

class DeviceTri {
public:
    // mirror: build the wave layout as the exact mirror of another one (the L of
    // an ILU pair) when valid (plan::WaveMirror), else the layout of its own
    // cmirror: likewise for the column layout (tri_plan.hpp COLUMNS)
    DeviceTri(const plan::TriSource& src, const TriOptions& opt, const plan::WaveMirror* mirror = nullptr,
              const plan::ColMirror* cmirror = nullptr);
    ~DeviceTri();
    DeviceTri(const DeviceTri&) = delete;
    DeviceTri& operator=(const DeviceTri&) = delete;

    // xs[o] = solution; out[oidx] = solution where oidx >= 0 (if out != null).
    void solve(const double* b, double* xs, double* out, cudaStream_t st,
               unsigned long long* trace = nullptr);
    // The two halves of solve(): bp[r] = b[bidx[r]] (bp holds n + 2 doubles), then
    // the solve from the reordered right-hand side.
    void permute(const double* b, double* bp, cudaStream_t st) const;
    void solve_ordered(const double* bp, double* xs, double* out, cudaStream_t st,
                       unsigned long long* trace = nullptr);
    // The solve alone: x in *wave order* (xw[wave position]; the solution order for
    // the level strategy), then permute_out gives xs[o] = xw[wpos[o]].
    void solve_wave(const double* bp, double* xw, double* out, cudaStream_t st,
                    unsigned long long* trace = nullptr);
    void permute_out(const double* xw, double* xs, cudaStream_t st) const;
    // The permutations restricted to the solution indices [o0, o1) (o0 a multiple
    // of 4), for host copies sliced to overlap them: bp[wpos[o]] = b[o] and
    // xs[o] = xw[wpos[o]]. Only for wave layouts whose positions are the n rows.
    bool sliceable() const { return strategy_ == 2 && !cols_ && wave_len_ == n_ && !h_wpos_.empty(); }
    void scatter_in(const double* b, double* bp, int o0, int o1, cudaStream_t st) const;
    void permute_out_range(const double* xw, double* xs, int o0, int o1, cudaStream_t st) const;
    // host copies of the maps: bidx (reordered input) and wpos (solution index ->
    // output position; empty = identity)
    const std::vector<int>& host_bidx() const { return h_bidx_; }
    const std::vector<int>& host_wpos() const { return h_wpos_; }
    // this layout's chunk structure, for mirroring (false for level launches)
    bool mirror_info(plan::WaveMirror& m) const;
    // the column layout's tiling, for mirroring (false for any other layout)
    bool col_mirror_info(plan::ColMirror& m) const;
    bool mirrored() const { return mirrored_; }
    // entries of the wave-ordered vectors (bp holds wave_len() + 2, xw wave_len())
    long long wave_len() const { return wave_len_; }
    // chunk -> CTA map of the pipeline layout (empty for LEVELS)
    const std::vector<int>& cta_chunk0() const { return p_cta0_host_; }
    // Synchronous host-vector convenience (pinned or pageable).
    void solve_host(const double* b, double* x);
    const TriStats& stats() const { return stats_; }
    int n() const { return n_; }
    // drops the workspace of a stream the caller is about to destroy (kept as the spare)
    void release_workspace(cudaStream_t st);
    int launches_per_solve() const;

private:
    struct Workspace {
        DevBuf<uint32_t> counters;            // ticket, finished CTAs, mailbox epoch
        DevBuf<unsigned long long> mailbox;   // cross-CTA values, 2 epoch-tagged words each
        DevBuf<double> bp;                    // right-hand side in reordered-row order
        DevBuf<double> xw;                    // solution in wave order
        // LEVELS: the argument block and the captured graph of the level launches
        DevBuf<unsigned char> largs;
        cudaGraphExec_t levels = nullptr;
        ~Workspace() {
            if (levels) cudaGraphExecDestroy(levels);
        }
    };
    Workspace& workspace(cudaStream_t st);
    std::unique_ptr<Workspace> make_workspace() const;
    void run_levels(const double* b, bool ordered, double* xs, double* out, cudaStream_t st);

    int n_ = 0;
    int strategy_ = 2;
    TriStats stats_;
    // LEVELS
    std::vector<int> level_starts_;
    std::vector<int> long_starts_;  // per level, into l_long_rows_
    DevBuf<int> l_long_rows_;
    int l_long_min_ = 0;
    DevBuf<int> l_starts_;  // level_starts_ on the device, for the persistent level kernel
    bool l_persist_ = false;  // HEC_LEVELS_PERSIST: one cooperative launch instead of per-level launches
    DevBuf<int> l_bidx_, l_xidx_, l_oidx_, l_ell_dep_, l_tail_rp_, l_tail_dep_;
    DevBuf<double> l_ell_val_, l_diag_, l_tail_val_;
    int l_width_ = 0, l_ld_ = 0;
    bool has_out_ = false;
    // WAVE (persistent wavefront kernel)
    DevBuf<unsigned char> p_blob_;
    DevBuf<int> p_spans_, p_cta0_, p_bidx_, p_wpos_;
    std::vector<int> h_bidx_, h_wpos_;
    int p_ctas_ = 0, p_inflight_ = 0, p_ring_ = 0, p_ring_off_ = 0, p_buf_off_ = 0, p_buf_bytes_ = 0;
    int p_smem_ = 0, p_warps_ = 0, p_lead_ = 1, spin_ns_ = 0, p_rpl_ = 1, p_halo_ring_ = 32, p_role_threads_ = 224;
    unsigned long long watchdog_ns_ = 10000000000ULL;  // 10 s: a solve is milliseconds
    int clock_khz_ = 2000000;                          // SM clock (cycles per ms), for the watchdog
    void* p_kernel_ = nullptr;
    void* p_kernel_trace_ = nullptr;
    long long p_exports_ = 0;
    std::vector<int> p_cta0_host_, h_chunk_r0_;
    bool mirrored_ = false;
    long long wave_len_ = 0;
    // COLUMNS (k_cols, 7-point grids)
    bool cols_ = false;
    plan::ColMirror c_info_;
    DevBuf<unsigned char> c_blocks_;
    DevBuf<int> c_cta_;
    int c_block_bytes_ = 0, c_ring_ = 0, c_warps_ = 0;
    bool c_unit_ = false;
    void build_columns(const plan::ColLayout& C);
    void launch_cols(const double* bp, double* xw, cudaStream_t st, unsigned long long* trace);

    std::mutex mu_;
    std::map<cudaStream_t, std::unique_ptr<Workspace>> ws_;
    std::unique_ptr<Workspace> spare_;  // taken by the first stream (no allocation, capture-safe)
    // host-call staging
    std::mutex h_mu_;
    DevBuf<double> h_b_, h_x_;
    cudaStream_t h_stream_ = nullptr;
};

class DevicePrecond {
public:
    // l/u sources carry no maps; they are attached here from gather/owned.
    DevicePrecond(int n, int n_ext, const int* gather, const char* owned, plan::TriSource l,
                  plan::TriSource u, const TriOptions& opt);
    // Local form (one RAS subdomain of a distributed vector): the input has n_in
    // entries and row k of the factors reads r[gather[k]]; the output has n_out
    // entries and row k writes x[out_index[k]] unless out_index[k] < 0.
    DevicePrecond(int n_in, int n_out, int n_ext, const int* gather, const int* out_index, plan::TriSource l,
                  plan::TriSource u, const TriOptions& opt);
    void apply(const double* r, double* x, cudaStream_t st);
    void apply_host(const double* r, double* x);
    // The handle's own stream (created on first use) with the lock that
    // serialises host-path users of it; workspaces stay bound to this stream.
    cudaStream_t host_stream(std::unique_lock<std::mutex>& lock);
    int launches_per_apply() const;
    const DeviceTri& lower() const { return *l_; }
    const DeviceTri& upper() const { return *u_; }
    int n() const { return n_; }
    int n_out() const { return n_out_; }

private:
    struct Workspace {
        DevBuf<double> bl, yw, bu, xw;  // L input (reordered), L output (wave), U input, U output
    };
    int n_ = 0, n_out_ = 0, n_ext_ = 0;
    bool identity_ = true;
    std::unique_ptr<DeviceTri> l_, u_;
    DevBuf<int> lu_map_;  // U input position -> L output position (the two permutations composed)
    void compose();
    void build_upper(const plan::TriSource& u, const TriOptions& opt);
    std::mutex mu_;
    std::map<cudaStream_t, std::unique_ptr<Workspace>> ws_;
    std::mutex h_mu_;
    DevBuf<double> h_r_, h_x_;
    cudaStream_t h_stream_ = nullptr;
    // apply_host with the copies sliced: host->device slices on h_in_, the
    // permutation of each slice on h_stream_ behind it, device->host on h_out_
    static constexpr int kMaxSlices = 8;
    cudaStream_t h_in_ = nullptr, h_out_ = nullptr;
    cudaEvent_t ev_in_[kMaxSlices] = {}, ev_out_[kMaxSlices] = {};
    int host_slices() const;
    void apply_middle(const double* bl, double* xw, Workspace& w, cudaStream_t st);
    Workspace& workspace(cudaStream_t st);

public:
    ~DevicePrecond();
};

// Device HEC SpMV (spmv_hec.cu): column-major ELL slots + CSR remainder.
class DeviceSpmv {
public:
    // From CSR: split like hec_from_csr(a, false, automatic), padding skipped
    // (bitwise spmv_csr, proj/src/csr.cpp:43-57).
    DeviceSpmv(int n_rows, int n_cols, const int* rp, const int* ci, const double* v);
    // From a reference HecMatrix (bitwise spmv_hec, proj/src/hec.cpp:88-108).
    DeviceSpmv(int n_rows, int n_cols, int width, const int* ell_cols, const double* ell_vals, const int* csr_rp,
               const int* csr_ci, const double* csr_v);
    void run(const double* x, double* y, cudaStream_t st) const;
    // y = b - A x (fused residual)
    void residual(const double* b, const double* x, double* y, cudaStream_t st) const;
    void run_host(const double* x, double* y);
    int n_rows() const { return n_rows_; }
    int n_cols() const { return n_cols_; }
    long long nnz() const { return nnz_; }
    int ell_width() const { return w_; }
    // algorithmic bytes of one product: 12 nnz + 4 (n+1) + 16 n
    double alg_bytes() const { return 12.0 * nnz_ + 4.0 * (n_rows_ + 1) + 16.0 * n_rows_; }

private:
    void upload(int w, const std::vector<int>& col, const std::vector<double>& val, const std::vector<int>& rp,
                const std::vector<int>& ci, const std::vector<double>& v);
    void launch(const double* x, const double* b, double* y, cudaStream_t st) const;
    int n_rows_ = 0, n_cols_ = 0, w_ = 0, ld_ = 0;
    bool has_rem_ = false;
    long long nnz_ = 0;
    DevBuf<int> ell_col_, rem_rp_, rem_ci_;
    DevBuf<double> ell_val_, rem_v_;
    std::mutex mu_;
    DevBuf<double> h_x_, h_y_;
};

// One-shot products with host vectors (the drop-in hec::spmv_csr / spmv_hec).
std::vector<double> spmv_csr_device(int n_rows, int n_cols, const int* rp, const int* ci, const double* v,
                                    const double* x);
std::vector<double> spmv_hec_device(int n_rows, int n_cols, int width, const int* ell_cols, const double* ell_vals,
                                    const int* csr_rp, const int* csr_ci, const double* csr_v, const double* x);

}  // namespace hec::dev
