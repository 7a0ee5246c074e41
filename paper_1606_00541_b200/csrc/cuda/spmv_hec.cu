// Device HEC SpMV: y = A x (and the fused residual y = b - A x) over the
// hybrid ELL + CSR layout (reference proj/src/hec.cpp:88-108 spmv_hec and
// proj/src/csr.cpp:43-57 spmv_csr).
//
// Layout in HBM (DeviceSpmv):
//   ell_col[w][ld] int32, ell_val[w][ld] f64   column-major, ld = round_up(n, 64)
//       so every slot column starts 256-byte aligned; slot k of row i at k*ld+i.
//       A column index < 0 marks a slot the kernel skips (padding of a layout
//       built from CSR); padding of a reference HecMatrix keeps its column
//       (min(i, n_cols-1)) and value 0 and is multiplied like the reference does.
//   rem_rp[ld+1], rem_ci, rem_v                 the CSR remainder (row order).
//
// Kernel: one warp per 64 consecutive rows, two rows per lane. The ELL slots
// are read with 8-byte (int2) / 16-byte (double2) streaming loads -- a warp
// reads 256 + 512 contiguous bytes per slot --, x through the read-only path.
// The remainder entries of the warp's 64 rows are one contiguous range; the
// warp stages it through shared memory in coalesced 128-entry tiles and each
// lane consumes its rows' entries in storage order. Every row is therefore
// accumulated exactly like the reference loop (ELL slots 0..w-1, then the CSR
// entries in order; separate multiply and add, no FMA): bitwise equal.

#include "device_runtime.hpp"

#include <algorithm>
#include <cstring>

namespace hec::dev {

namespace {

constexpr int kSpmvThreads = 256;
constexpr int kTile = 128;  // remainder entries staged per warp and tile

struct SpmvArgs {
    int n, w, ld, has_rem;
    const int* ell_col;
    const double* ell_val;
    const int* rem_rp;
    const int* rem_ci;
    const double* rem_v;
    const double* x;
    const double* b;  // residual form: y = b - A x
    double* y;
};

template <bool RESID>
__global__ void __launch_bounds__(kSpmvThreads) k_spmv_hec(SpmvArgs a) {
    __shared__ int s_ci[kSpmvThreads / 32][kTile];
    __shared__ double s_v[kSpmvThreads / 32][kTile];
    const int lane = threadIdx.x & 31, wb = threadIdx.x >> 5;
    const long long nwarps = static_cast<long long>(gridDim.x) * (kSpmvThreads / 32);
    const double* __restrict__ x = a.x;
    for (long long t = static_cast<long long>(blockIdx.x) * (kSpmvThreads / 32) + wb; t * 64 < a.n; t += nwarps) {
        const int i0 = static_cast<int>(t * 64) + 2 * lane;  // < ld: the padded columns are readable
        double acc0 = 0.0, acc1 = 0.0;
#pragma unroll 4
        for (int k = 0; k < a.w; ++k) {
            const size_t s = static_cast<size_t>(k) * a.ld + i0;
            const int2 c = __ldcs(reinterpret_cast<const int2*>(a.ell_col + s));
            const double2 v = __ldcs(reinterpret_cast<const double2*>(a.ell_val + s));
            if (c.x >= 0) acc0 = __dadd_rn(acc0, __dmul_rn(v.x, __ldg(x + c.x)));
            if (c.y >= 0) acc1 = __dadd_rn(acc1, __dmul_rn(v.y, __ldg(x + c.y)));
        }
        if (a.has_rem) {  // warp-uniform
            const int r0 = a.rem_rp[i0], r1 = a.rem_rp[i0 + 1], r2 = a.rem_rp[i0 + 2];
            const int e0 = __shfl_sync(0xffffffffu, r0, 0), e1 = __shfl_sync(0xffffffffu, r2, 31);
            for (int tb = e0; tb < e1; tb += kTile) {
#pragma unroll
                for (int u = 0; u < kTile / 32; ++u) {
                    const int e = tb + u * 32 + lane;
                    if (e < e1) {
                        s_ci[wb][u * 32 + lane] = __ldcs(a.rem_ci + e);
                        s_v[wb][u * 32 + lane] = __ldcs(a.rem_v + e);
                    }
                }
                __syncwarp();
                const int te = tb + kTile;
                for (int e = max(r0, tb); e < min(r1, te); ++e)
                    acc0 = __dadd_rn(acc0, __dmul_rn(s_v[wb][e - tb], __ldg(x + s_ci[wb][e - tb])));
                for (int e = max(r1, tb); e < min(r2, te); ++e)
                    acc1 = __dadd_rn(acc1, __dmul_rn(s_v[wb][e - tb], __ldg(x + s_ci[wb][e - tb])));
                __syncwarp();
            }
        }
        if (i0 < a.n) a.y[i0] = RESID ? __dsub_rn(a.b[i0], acc0) : acc0;
        if (i0 + 1 < a.n) a.y[i0 + 1] = RESID ? __dsub_rn(a.b[i0 + 1], acc1) : acc1;
    }
}

int grid_for(int n) {
    static int sms = 0;
    if (!sms) {
        int dev = 0;
        HEC_CUDA(cudaGetDevice(&dev));
        HEC_CUDA(cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev));
    }
    const long long tiles = (static_cast<long long>(n) + 63) / 64;
    const long long blocks = (tiles + kSpmvThreads / 32 - 1) / (kSpmvThreads / 32);
    return static_cast<int>(std::max<long long>(1, std::min<long long>(blocks, 16LL * sms)));  // 16 x 148 resident
}

inline int round_up(int v, int m) { return (v + m - 1) / m * m; }

// The reference's automatic ELL width (hec.cpp:11-24): the median row length,
// clamped to [0, max].
int median_width(const std::vector<int>& cnt) {
    if (cnt.empty()) return 0;
    std::vector<int> s = cnt;
    auto mid = s.begin() + s.size() / 2;
    std::nth_element(s.begin(), mid, s.end());
    return std::clamp(*mid, 0, *std::max_element(cnt.begin(), cnt.end()));
}

}  // namespace

void DeviceSpmv::upload(int w, const std::vector<int>& col, const std::vector<double>& val,
                        const std::vector<int>& rp, const std::vector<int>& ci, const std::vector<double>& v) {
    w_ = w;
    ell_col_.upload(col);
    ell_val_.upload(val);
    has_rem_ = !ci.empty();
    rem_rp_.upload(rp);
    if (has_rem_) {
        rem_ci_.upload(ci);
        rem_v_.upload(v);
    }
}

// From CSR (the layout GMRES multiplies with): reference hec_from_csr(a, false,
// automatic) split -- the first min(w, cnt_i) entries of each row go to ELL
// slots, the rest to the remainder -- with the padding slots marked -1, so each
// row sums exactly the CSR row in storage order: bitwise spmv_csr.
DeviceSpmv::DeviceSpmv(int n_rows, int n_cols, const int* rp, const int* ci, const double* v)
    : n_rows_(n_rows), n_cols_(n_cols) {
    require_device();
    if (n_rows < 0 || n_cols < 0) throw std::invalid_argument("hec_spmv_create: negative dimension");
    nnz_ = n_rows > 0 ? rp[n_rows] : 0;
    ld_ = round_up(std::max(n_rows, 1), 64);
    std::vector<int> cnt(n_rows);
    for (int i = 0; i < n_rows; ++i) {
        cnt[i] = rp[i + 1] - rp[i];
        if (cnt[i] < 0) throw std::invalid_argument("hec_spmv_create: row offsets not monotone");
    }
    const int w = median_width(cnt);
    std::vector<int> col(static_cast<size_t>(w) * ld_, -1);
    std::vector<double> val(static_cast<size_t>(w) * ld_, 0.0);
    std::vector<int> rrp(static_cast<size_t>(ld_) + 1, 0);
    for (int i = 0; i < n_rows; ++i) rrp[i + 1] = rrp[i] + std::max(0, cnt[i] - w);
    for (int i = n_rows; i < ld_; ++i) rrp[i + 1] = rrp[i];
    std::vector<int> rci(static_cast<size_t>(rrp[ld_]));
    std::vector<double> rv(rci.size());
#pragma omp parallel for schedule(static)
    for (int i = 0; i < n_rows; ++i) {
        const int in_ell = std::min(w, cnt[i]);
        for (int k = 0; k < in_ell; ++k) {
            const int c = ci[rp[i] + k];
            if (c < 0 || c >= n_cols) continue;  // checked below (serially, with the message)
            col[static_cast<size_t>(k) * ld_ + i] = c;
            val[static_cast<size_t>(k) * ld_ + i] = v[rp[i] + k];
        }
        int d = rrp[i];
        for (int e = rp[i] + in_ell; e < rp[i + 1]; ++e, ++d) {
            rci[d] = ci[e];
            rv[d] = v[e];
        }
    }
    for (long long e = 0; e < nnz_; ++e)
        if (ci[e] < 0 || ci[e] >= n_cols) throw std::invalid_argument("hec_spmv_create: column out of range");
    upload(w, col, val, rrp, rci, rv);
}

// From a reference HecMatrix (hec.hpp:13-46): ELL slots as stored (padding
// included: the reference multiplies it, hec.cpp:99-102), then the CSR part.
DeviceSpmv::DeviceSpmv(int n_rows, int n_cols, int width, const int* ell_cols, const double* ell_vals,
                       const int* csr_rp, const int* csr_ci, const double* csr_v)
    : n_rows_(n_rows), n_cols_(n_cols) {
    require_device();
    if (n_rows < 0 || n_cols < 0 || width < 0) throw std::invalid_argument("hec_spmv_create_hec: negative size");
    ld_ = round_up(std::max(n_rows, 1), 64);
    std::vector<int> col(static_cast<size_t>(width) * ld_, -1);
    std::vector<double> val(static_cast<size_t>(width) * ld_, 0.0);
    for (int k = 0; k < width; ++k) {
        const size_t src = static_cast<size_t>(k) * n_rows, dst = static_cast<size_t>(k) * ld_;
        for (int i = 0; i < n_rows; ++i)
            if (ell_cols[src + i] < 0 || ell_cols[src + i] >= n_cols)
                throw std::invalid_argument("hec_spmv_create_hec: ELL column out of range");
        if (n_rows) {
            std::memcpy(col.data() + dst, ell_cols + src, sizeof(int) * n_rows);
            std::memcpy(val.data() + dst, ell_vals + src, sizeof(double) * n_rows);
        }
    }
    std::vector<int> rrp(static_cast<size_t>(ld_) + 1);
    for (int i = 0; i <= n_rows; ++i) rrp[i] = csr_rp[i];
    for (int i = n_rows; i < ld_; ++i) rrp[i + 1] = rrp[i];
    const int nr = rrp[n_rows];
    for (int e = 0; e < nr; ++e)
        if (csr_ci[e] < 0 || csr_ci[e] >= n_cols) throw std::invalid_argument("hec_spmv_create_hec: column out of range");
    nnz_ = nr;
    for (size_t s = 0; s < static_cast<size_t>(width) * n_rows; ++s) nnz_ += ell_vals[s] != 0.0;
    upload(width, col, val, rrp, std::vector<int>(csr_ci, csr_ci + nr), std::vector<double>(csr_v, csr_v + nr));
}

void DeviceSpmv::launch(const double* x, const double* b, double* y, cudaStream_t st) const {
    if (n_rows_ == 0) return;
    SpmvArgs a{};
    a.n = n_rows_;
    a.w = w_;
    a.ld = ld_;
    a.has_rem = has_rem_ ? 1 : 0;
    a.ell_col = ell_col_.p;
    a.ell_val = ell_val_.p;
    a.rem_rp = rem_rp_.p;
    a.rem_ci = rem_ci_.p;
    a.rem_v = rem_v_.p;
    a.x = x;
    a.b = b;
    a.y = y;
    if (b)
        k_spmv_hec<true><<<grid_for(n_rows_), kSpmvThreads, 0, st>>>(a);
    else
        k_spmv_hec<false><<<grid_for(n_rows_), kSpmvThreads, 0, st>>>(a);
    HEC_CUDA(cudaGetLastError());
}

void DeviceSpmv::run(const double* x, double* y, cudaStream_t st) const { launch(x, nullptr, y, st); }

void DeviceSpmv::residual(const double* b, const double* x, double* y, cudaStream_t st) const {
    launch(x, b, y, st);
}

void DeviceSpmv::run_host(const double* x, double* y) {
    std::lock_guard<std::mutex> g(mu_);
    if (h_x_.count < static_cast<std::size_t>(std::max(n_cols_, 1))) h_x_.alloc(std::max(n_cols_, 1));
    if (h_y_.count < static_cast<std::size_t>(std::max(n_rows_, 1))) h_y_.alloc(std::max(n_rows_, 1));
    HEC_CUDA(cudaMemcpy(h_x_.p, x, sizeof(double) * n_cols_, cudaMemcpyHostToDevice));
    run(h_x_.p, h_y_.p, nullptr);
    HEC_CUDA(cudaMemcpy(y, h_y_.p, sizeof(double) * n_rows_, cudaMemcpyDeviceToHost));
}

std::vector<double> spmv_csr_device(int n_rows, int n_cols, const int* rp, const int* ci, const double* v,
                                    const double* x) {
    DeviceSpmv a(n_rows, n_cols, rp, ci, v);
    std::vector<double> y(static_cast<size_t>(n_rows));
    a.run_host(x, y.data());
    return y;
}

std::vector<double> spmv_hec_device(int n_rows, int n_cols, int width, const int* ell_cols, const double* ell_vals,
                                    const int* csr_rp, const int* csr_ci, const double* csr_v, const double* x) {
    DeviceSpmv a(n_rows, n_cols, width, ell_cols, ell_vals, csr_rp, csr_ci, csr_v);
    std::vector<double> y(static_cast<size_t>(n_rows));
    a.run_host(x, y.data());
    return y;
}

}  // namespace hec::dev
