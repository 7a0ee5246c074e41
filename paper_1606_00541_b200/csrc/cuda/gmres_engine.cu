// Restarted right-preconditioned GMRES(m) on one GPU or on several (RAS: one
// subdomain per rank), zero initial guess.
//
// Control flow, tolerances, the lucky-breakdown / stall logic, the Givens
// rotations, the back substitution and every reported quantity follow the
// reference proj/src/gmres.cpp:28-137 line for line (host arithmetic, same
// order). The n-length work runs on the GPU:
//
//   w = A M^-1 v_j      halo exchange of v_j (RAS), local ILU apply (the
//                       persistent k_wave triangular solves), halo exchange of
//                       z, HEC SpMV of the owned rows
//   orthogonalisation   classical Gram-Schmidt with one re-orthogonalisation
//                       (CGS2) instead of the reference's modified Gram-Schmidt
//                       (gmres.cpp:72-77): the j+1 dots of a pass are one fused
//                       multi-vector kernel and ONE all-reduce, so an iteration
//                       costs two all-reduces (pass 1: V^T w; pass 2: V^T w' and
//                       ||w'||^2) instead of j+2. h = h1 + h2 and
//                       ||w''||^2 = ||w'||^2 - ||h2||^2 (V orthonormal).
//                       In exact arithmetic CGS2 and MGS produce the same
//                       Hessenberg matrix; rounding differs, so iteration counts
//                       are compared within +-1.
//   restart             x += M^-1 (V y), r = b - A x (fused residual SpMV).
//
// Dots are deterministic: per-thread sums in a fixed element order, fixed
// block trees, and a fixed-order final sum by the last block (then the
// all-reduce across ranks).

#include <cuda_runtime.h>

#include <algorithm>
#include <chrono>
#include <cmath>
#include <cstdint>
#include <cstdio>
#include <cstdlib>
#include <vector>

#include "comm.hpp"
#include "device_runtime.hpp"
#include "gmres_engine.hpp"
#include "ptx.cuh"

namespace hec::dev {

namespace {

constexpr int kT = 256;       // threads per block
constexpr int kKG = 32;       // basis vectors per fused pass
constexpr int kMaxOut = kKG + 1;

// Block-reduces acc[0..kc) and, with_norm, acc[kKG] (as output kc) to
// partials[k * grid + block]; the last block to finish sums partials[k * grid +
// 0..grid) in a fixed order into out[k]. Fixed shapes: run-to-run reproducible.
template <int KG>
__device__ __forceinline__ void reduce_out(double (&acc)[KG + 1], int kc, int with_norm, double* partials,
                                           unsigned* counter, double* out) {
    __shared__ double sw[KG + 1][kT / 32];
    __shared__ bool last;
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5, nwarps = blockDim.x >> 5;  // blockDim <= kT
    const int cnt = kc + (with_norm ? 1 : 0);
#pragma unroll
    for (int k = 0; k < (KG + 1); ++k) {
        const bool use = k < kc || (k == KG && with_norm);
        if (use) {
            double v = acc[k];
            for (int o = 16; o > 0; o >>= 1) v = __dadd_rn(v, __shfl_down_sync(0xffffffffu, v, o));
            if (lane == 0) sw[k < kc ? k : kc][warp] = v;
        }
    }
    __syncthreads();
    if (threadIdx.x < cnt) {
        double s = 0.0;
        for (int q = 0; q < nwarps; ++q) s = __dadd_rn(s, sw[threadIdx.x][q]);
        partials[static_cast<size_t>(threadIdx.x) * gridDim.x + blockIdx.x] = s;
    }
    __threadfence();
    __syncthreads();
    if (threadIdx.x == 0) last = atomicAdd(counter, 1u) == gridDim.x - 1;
    __syncthreads();
    if (!last) return;
    __threadfence();
    for (int k = warp; k < cnt; k += nwarps) {  // one warp per output, fixed order
        double s = 0.0;
        for (unsigned b = lane; b < gridDim.x; b += 32)
            s = __dadd_rn(s, __ldcg(&partials[static_cast<size_t>(k) * gridDim.x + b]));
        for (int o = 16; o > 0; o >>= 1) s = __dadd_rn(s, __shfl_down_sync(0xffffffffu, s, o));
        if (lane == 0) out[k] = s;
    }
    if (threadIdx.x == 0) *counter = 0;
}

// Multi-vector kernel (the Gram-Schmidt passes, the basis combination and the
// norms): every block streams row tiles of kc basis columns (and w) into shared
// memory with TMA bulk copies, double-buffered on mbarriers, so the memory
// system always has two tiles per SM in flight while the threads work from
// shared memory (one row per thread):
//   w_out = (w_in - sum_{k<kc} c_k V_k) / s      if w_out (w_in null: 0.0;
//            k in order; s per scale_mode: 0 none, 1 scale_val, 2 the CGS2 norm
//            sqrt(max(0, c[kc] - sum_k c_k^2)) written to *s_out)
//   out[k] = V_k . u (k < kc), out[kc] = u . u   if dots (u = w_out, or w_in
//            when nothing is written; the norm only if with_norm)
constexpr int kTile = 256;  // rows per tile = threads per block (at most; 128 for wide passes)
struct MvArgs {
    int n, kc;
    size_t ldv;
    const double* V;
    const double* c;
    const double* w_in;
    double* w_out;
    int scale_mode;
    double scale_val;
    double* s_out;
    int dots, with_norm;
    double* partials;
    unsigned* counter;
    double* out;
};

// Called by the 32 lanes of warp 0: lane 0 arms the stage's mbarrier with the
// tile's byte count, then every lane issues the bulk copies of its columns (a
// single thread issuing ~30 copies back to back would pace the stream).
__device__ __forceinline__ void mv_issue(const MvArgs& a, int tile, double* stage, uint64_t* bar, int lane) {
    const int rows = blockDim.x;
    const int r0 = tile * rows;
    const int m = min(rows, a.n - r0);
    const uint32_t bytes = static_cast<uint32_t>(((m + 1) & ~1) * 8);  // 16-byte multiple (columns are padded)
    const int nw = a.w_in ? 1 : 0;
    if (lane == 0) mbar_expect_tx(bar, bytes * static_cast<uint32_t>(a.kc + nw));
    __syncwarp();
    for (int k = lane; k < a.kc + nw; k += 32)
        bulk_g2s(stage + k * rows, k < a.kc ? a.V + k * a.ldv + r0 : a.w_in + r0, bytes, bar);
}

// KG: the widest pass this instantiation takes (its accumulators live in
// registers: 8 / 16 / 32 columns leave room for 4 / 3 / 2 blocks per SM)
template <int KG>
__global__ void __launch_bounds__(kTile, KG <= 8 ? 4 : (KG <= 16 ? 3 : 2)) k_mv(MvArgs a) {
    extern __shared__ __align__(128) double mv_smem[];
    __shared__ uint64_t bar[2];
    __shared__ double sc[(KG + 1)];
    __shared__ double s_scale;
    const int tid = threadIdx.x, rows = blockDim.x;
    const int ntiles = (a.n + rows - 1) / rows;
    const int per_stage = (a.kc + 1) * rows;
    if (tid < a.kc && a.c) sc[tid] = a.c[tid];
    if (tid == 0) {
        double s = 1.0;
        if (a.scale_mode == 1) s = a.scale_val;
        if (a.scale_mode == 2) {
            double h2 = 0.0;
            for (int k = 0; k < a.kc; ++k) h2 = __dadd_rn(h2, __dmul_rn(a.c[k], a.c[k]));
            s = __dsqrt_rn(fmax(__dsub_rn(a.c[a.kc], h2), 0.0));
            if (blockIdx.x == 0) *a.s_out = s;
            if (!(s > 0.0)) s = 1.0;  // breakdown: the column is never used (gmres.cpp:79-83)
        }
        s_scale = s;
        mbar_init(&bar[0], 1);
        mbar_init(&bar[1], 1);
        asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    }
    __syncthreads();
    if (tid < 32)
        for (int q = 0; q < 2; ++q) {
            const int tile = blockIdx.x + q * gridDim.x;
            if (tile < ntiles) mv_issue(a, tile, mv_smem + q * per_stage, &bar[q], tid);
        }
    const double s = s_scale;
    double acc[(KG + 1)];
#pragma unroll
    for (int k = 0; k < (KG + 1); ++k) acc[k] = 0.0;
    for (int it = 0, tile = blockIdx.x; tile < ntiles; ++it, tile += gridDim.x) {
        const int q = it & 1;
        const double* st = mv_smem + q * per_stage;
        mbar_wait(&bar[q], (it >> 1) & 1);
        const int i = tile * rows + tid;
        if (i < a.n) {
            double u = a.w_in ? st[a.kc * rows + tid] : 0.0;
            if (a.w_out) {
#pragma unroll
                for (int k = 0; k < KG; ++k)
                    if (k < a.kc) u = __dsub_rn(u, __dmul_rn(sc[k], st[k * rows + tid]));
                if (a.scale_mode) u = __ddiv_rn(u, s);
                a.w_out[i] = u;
            }
            if (a.dots) {
#pragma unroll
                for (int k = 0; k < KG; ++k)
                    if (k < a.kc) acc[k] = __dadd_rn(acc[k], __dmul_rn(st[k * rows + tid], u));
                acc[KG] = __dadd_rn(acc[KG], __dmul_rn(u, u));
            }
        }
        __syncthreads();  // every thread is done with this stage
        if (tid < 32) {
            const int next = tile + 2 * gridDim.x;
            if (next < ntiles) {
                asm volatile("fence.proxy.async.shared::cta;" ::: "memory");  // generic reads before async writes
                mv_issue(a, next, mv_smem + q * per_stage, &bar[q], tid);
            }
        }
    }
    if (a.dots) reduce_out<KG>(acc, a.kc, a.with_norm, a.partials, a.counter, a.out);
}

__global__ void k_add_v(int n, double* x, const double* d) {
    for (int i = blockIdx.x * blockDim.x + threadIdx.x; i < n; i += gridDim.x * blockDim.x)
        x[i] = __dadd_rn(x[i], d[i]);
}

// send[i] = v[idx[i]] (halo pack)
__global__ void k_pack(int m, const int* __restrict__ idx, const double* v, double* send) {
    for (int i = blockIdx.x * blockDim.x + threadIdx.x; i < m; i += gridDim.x * blockDim.x) send[i] = v[idx[i]];
}

struct PinnedHost {
    double* p = nullptr;
    explicit PinnedHost(std::size_t n) { HEC_CUDA(cudaMallocHost(&p, sizeof(double) * std::max<std::size_t>(n, 1))); }
    ~PinnedHost() {
        if (p) cudaFreeHost(p);
    }
    PinnedHost(const PinnedHost&) = delete;
    PinnedHost& operator=(const PinnedHost&) = delete;
};

struct EventPair {
    cudaEvent_t e[2] = {};
    EventPair() {
        for (auto& x : e) HEC_CUDA(cudaEventCreateWithFlags(&x, cudaEventDisableTiming));
    }
    ~EventPair() {
        for (auto& x : e)
            if (x) cudaEventDestroy(x);
    }
    cudaEvent_t operator[](int k) const { return e[k]; }
    EventPair(const EventPair&) = delete;
    EventPair& operator=(const EventPair&) = delete;
};

int sm_count() {
    int dev = 0, sms = 0;
    HEC_CUDA(cudaGetDevice(&dev));
    HEC_CUDA(cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev));
    return sms;
}

}  // namespace

void halo_exchange(const DistSystem& S, double* vloc, double* sendbuf, cudaStream_t st) {
    if (!S.comm || S.comm->world() == 1) return;
    if (S.n_send) {
        const int vb = 256;
        k_pack<<<std::max(1, std::min(4 * sm_count(), (S.n_send + vb - 1) / vb)), vb, 0, st>>>(S.n_send, S.send_idx,
                                                                                             vloc, sendbuf);
        HEC_CUDA(cudaGetLastError());
    }
    S.comm->exchange(sendbuf, S.send_off, vloc + S.n_own, S.recv_off, st);
}

namespace {
// HEC_GMRES_PROFILE=1: CUDA-event times of the phases of every inner iteration
// (apply + SpMV with its exchanges, CGS2 pass 1, pass 2, normalisation), summed
// and printed to stderr at the end of the solve (diagnostics; adds event syncs).
struct PhaseProfile {
    bool on = std::getenv("HEC_GMRES_PROFILE") != nullptr;
    cudaEvent_t ev[5] = {};
    bool marked[5] = {};
    double ms[4] = {};
    int iters = 0;
    PhaseProfile() {
        if (on)
            for (auto& e : ev) cudaEventCreate(&e);
    }
    ~PhaseProfile() {
        if (!on) return;
        std::fprintf(stderr, "[hec gmres] %d iterations, ms per iteration: apply+spmv %.3f  pass1 %.3f  pass2 %.3f  "
                             "normalise %.3f\n", iters, ms[0] / std::max(iters, 1), ms[1] / std::max(iters, 1),
                     ms[2] / std::max(iters, 1), ms[3] / std::max(iters, 1));
        for (auto& e : ev) cudaEventDestroy(e);
    }
    void mark(cudaStream_t st, int k) {
        if (!on) return;
        cudaEventRecord(ev[k], st);
        marked[k] = true;
    }
    void collect() {
        if (!on || !marked[4]) return;
        for (int k = 0; k < 4; ++k) {
            float t = 0.f;
            cudaEventElapsedTime(&t, ev[k], ev[k + 1]);
            ms[k] += t;
        }
        ++iters;
        for (bool& m : marked) m = false;
    }
};
}  // namespace

GmresOutcome gmres_dist(DistSystem& S, const double* b_own, double* x_own, const GmresParams& cfg,
                        cudaStream_t st) {
    PhaseProfile prof;
    if (cfg.restart < 1) throw std::invalid_argument("gmres: restart must be >= 1");
    if (cfg.max_iters < 0) throw std::invalid_argument("gmres: max_iters must be >= 0");
    if (cfg.rel_tol < 0.0 || cfg.abs_tol < 0.0) throw std::invalid_argument("gmres: tolerances must be >= 0");
    if (!S.A || S.A->n_rows() != S.n_own || S.A->n_cols() != S.n_loc)
        throw std::invalid_argument("gmres: operator size mismatch");
    if (S.M && (S.M->n() != S.n_loc || S.M->n_out() != S.n_own))
        throw std::invalid_argument("gmres: preconditioner size mismatch");
    NullComm none;
    Comm& comm = S.comm ? *S.comm : none;

    const auto t0 = std::chrono::steady_clock::now();
    const int n = S.n_own;
    const int mr = cfg.restart;
    GmresOutcome out;
    const int grid = std::max(1, std::min(4 * sm_count(), (n + kT - 1) / kT));
    const int sms = sm_count();
    const size_t ldv = static_cast<size_t>((std::max(S.n_loc, 1) + 31) / 32 * 32);  // 256-byte aligned columns

    DevBuf<double> V(static_cast<size_t>(mr + 1) * ldv), w(ldv), zloc(ldv), xloc(ldv), xc(ldv), r(ldv), b(ldv);
    DevBuf<double> hb(2 * static_cast<size_t>(mr) + 8), yv(static_cast<size_t>(mr) + 1);
    DevBuf<double> partials(static_cast<size_t>(kMaxOut) * 16 * sms), sendbuf(std::max(S.n_send, 1));
    DevBuf<unsigned> counter(1);
    HEC_CUDA(cudaMemsetAsync(counter.p, 0, sizeof(unsigned), st));
    HEC_CUDA(cudaMemsetAsync(xloc.p, 0, sizeof(double) * ldv, st));
    HEC_CUDA(cudaMemcpyAsync(b.p, b_own, sizeof(double) * n, cudaMemcpyDeviceToDevice, st));
    double* hb1 = hb.p;            // pass-1 dots (j+1)
    double* hb2 = hb.p + mr + 2;   // pass-2 dots (j+1), ||w'||^2, ||w''||
    // pinned host staging for the per-iteration Hessenberg column and the other
    // small host round trips: a copy into pageable memory goes through the
    // driver's staging buffer, synchronously (measured: 256^3 solves of 1.34 to
    // 2.04 s for the same 1.28 s of device phases)
    const size_t hstride = 2 * static_cast<size_t>(mr) + 8;
    PinnedHost hpin(2 * hstride + (mr + 1) + 1);
    double* const hh2 = hpin.p;  // two slots: column j read while column j+1 runs
    double* const ny = hpin.p + 2 * hstride;
    double* const s2p = ny + mr + 1;
    EventPair ev_col;

    auto halo = [&](double* vloc) {  // fill vloc[n_own ..) from the owners
        if (comm.world() == 1) return;
        out.launches += S.n_send ? 1 : 0;
        halo_exchange(S, vloc, sendbuf.p, st);
    };
    auto apply_op = [&](double* vloc, double* dst) {  // dst = A M^-1 v (own rows)
        halo(vloc);
        if (S.M) {
            S.M->apply(vloc, zloc.p, st);
            out.launches += S.M->launches_per_apply();
            halo(zloc.p);
            S.A->run(zloc.p, dst, st);
        } else {
            S.A->run(vloc, dst, st);
        }
        ++out.launches;
    };
    // one multi-vector pass (k_mv): grid sized by the shared memory its tiles need
    static bool mv_attr = false;
    if (!mv_attr) {
        for (auto k : {k_mv<8>, k_mv<16>, k_mv<kKG>}) {
            HEC_CUDA(cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                          2 * kMaxOut * kTile * static_cast<int>(sizeof(double))));
            // several blocks per SM need the whole carve-out as shared memory
            HEC_CUDA(cudaFuncSetAttribute(k, cudaFuncAttributePreferredSharedMemoryCarveout,
                                          cudaSharedmemCarveoutMaxShared));
        }
        mv_attr = true;
    }
    auto mv = [&](int kc, const double* Vb, const double* c, const double* w_in, double* w_out, int scale_mode,
                  double scale_val, double* s_out, int dots, int with_norm, double* outp) {
        MvArgs m{};
        m.n = n;
        m.kc = kc;
        m.ldv = ldv;
        m.V = Vb;
        m.c = c;
        m.w_in = w_in;
        m.w_out = w_out;
        m.scale_mode = scale_mode;
        m.scale_val = scale_val;
        m.s_out = s_out;
        m.dots = dots;
        m.with_norm = with_norm;
        m.partials = partials.p;
        m.counter = counter.p;
        m.out = outp;
        // tiles of 256 rows, 128 when the pass is wide: at least three blocks (six
        // tiles in flight) per SM
        const int rows = (kc + 1) * kTile * 16 <= 72 * 1024 ? kTile : kTile / 2;
        const int smem = 2 * (kc + 1) * rows * static_cast<int>(sizeof(double));
        void (*kern)(MvArgs) = kc <= 8 ? k_mv<8> : (kc <= 16 ? k_mv<16> : k_mv<kKG>);
        int per_sm = 0;  // resident blocks (registers, shared memory): one wave of persistent blocks
        HEC_CUDA(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, kern, rows, smem));
        const int ntiles = (n + rows - 1) / rows;
        const int g = std::max(1, std::min(ntiles, std::max(per_sm, 1) * sms));
        kern<<<g, rows, smem, st>>>(m);
        HEC_CUDA(cudaGetLastError());
        ++out.launches;
    };
    auto norm = [&](const double* v) {  // sqrt(sum over ranks of v . v)
        mv(0, nullptr, nullptr, v, nullptr, 0, 1.0, nullptr, 1, 1, hb.p);
        comm.allreduce_sum(hb.p, 1, st);
        HEC_CUDA(cudaMemcpyAsync(s2p, hb.p, sizeof(double), cudaMemcpyDeviceToHost, st));
        HEC_CUDA(cudaStreamSynchronize(st));
        return std::sqrt(*s2p);
    };

    const double bnorm = norm(b.p);
    if (prof.on)
        std::fprintf(stderr, "[hec gmres] setup (buffers, first norm) %.3f ms\n",
                     std::chrono::duration<double, std::milli>(std::chrono::steady_clock::now() - t0).count());
    const double threshold = std::max(cfg.rel_tol * bnorm, cfg.abs_tol);
    std::vector<double> h(static_cast<size_t>(mr + 1) * mr, 0.0), cs(mr), sn(mr), g(mr + 1), y(mr);
    HEC_CUDA(cudaMemcpyAsync(r.p, b.p, sizeof(double) * n, cudaMemcpyDeviceToDevice, st));
    double rnorm = bnorm;
    bool stalled = false;

    while (true) {
        if (rnorm <= threshold) {
            out.converged = true;
            break;
        }
        if (out.iterations >= cfg.max_iters || stalled) break;
        // v_0 = r / rnorm (gmres.cpp:62)
        mv(0, nullptr, nullptr, r.p, V.p, 1, rnorm, nullptr, 0, 0, nullptr);
        std::fill(g.begin(), g.end(), 0.0);
        g[0] = rnorm;

        // Column jj of the Arnoldi process: apply, the Gram-Schmidt passes, and
        // the copy of its Hessenberg entries into host slot jj & 1 (event ev_col).
        auto launch_col = [&](int jj) {
            double* vj = V.p + jj * ldv;
            prof.mark(st, 0);
            apply_op(vj, w.p);
            prof.mark(st, 1);
            const int kc = jj + 1;
            if (kc <= kKG) {
                // CGS2 pass 1: h1 = V^T w
                mv(kc, V.p, nullptr, w.p, nullptr, 0, 1.0, nullptr, 1, 0, hb1);
                prof.mark(st, 2);
                comm.allreduce_sum(hb1, kc, st);
                // pass 2: w' = w - V h1; h2 = V^T w', ||w'||^2
                mv(kc, V.p, hb1, w.p, w.p, 0, 1.0, nullptr, 1, 1, hb2);
                prof.mark(st, 3);
                comm.allreduce_sum(hb2, kc + 1, st);
                // v_{jj+1} = (w' - V h2) / ||w''||
                mv(kc, V.p, hb2, w.p, V.p + (jj + 1) * ldv, 2, 1.0, hb2 + kc + 1, 0, 0, nullptr);
                prof.mark(st, 4);
            } else {
                // more basis vectors than one fused pass holds: modified Gram-Schmidt,
                // one vector at a time (each step still one dot + one all-reduce)
                for (int i = 0; i < kc; ++i) {
                    mv(1, V.p + i * ldv, nullptr, w.p, nullptr, 0, 1.0, nullptr, 1, 0, hb1 + i);
                    comm.allreduce_sum(hb1 + i, 1, st);
                    mv(1, V.p + i * ldv, hb1 + i, w.p, w.p, 0, 1.0, nullptr, i + 1 == kc, 1, hb2 + kc - 1);
                }
                comm.allreduce_sum(hb2 + kc, 1, st);
                HEC_CUDA(cudaMemsetAsync(hb2, 0, sizeof(double) * kc, st));
                mv(0, nullptr, hb2 + kc, w.p, V.p + (jj + 1) * ldv, 2, 1.0, hb2 + kc + 1, 0, 0, nullptr);
            }
            HEC_CUDA(cudaMemcpyAsync(hh2 + (jj & 1) * hstride, hb.p, sizeof(double) * (2 * mr + 8),
                                     cudaMemcpyDeviceToHost, st));
            HEC_CUDA(cudaEventRecord(ev_col[jj & 1], st));
        };
        // The next column only needs v_{j+1}, which the device produces itself, so
        // it is queued before the host reads column j's entries: the host's Givens
        // work and its wake-up latency hide behind a column of device work. If the
        // cycle stops at column j (convergence or breakdown), the queued column is
        // discarded (it touches neither h, g nor V[:, <= j+1]).
        const bool ahead = !prof.on;  // the phase profile wants one column at a time
        int j = 0;
        bool lucky = false;
        if (j < mr && out.iterations < cfg.max_iters) launch_col(0);
        while (j < mr && out.iterations < cfg.max_iters) {
            const int kc = j + 1;
            if (ahead && j + 1 < mr && out.iterations + 1 < cfg.max_iters) launch_col(j + 1);
            HEC_CUDA(cudaEventSynchronize(ev_col[j & 1]));
            const double* hh = hh2 + (j & 1) * hstride;
            prof.collect();
            for (int i = 0; i <= j; ++i) h[i + j * (mr + 1)] = hh[i] + hh[mr + 2 + i];
            const double hjj1 = hh[mr + 2 + kc + 1];
            h[(j + 1) + j * (mr + 1)] = hjj1;
            if (!(hjj1 > 1e-300)) lucky = true;

            // Givens rotations (gmres.cpp:85-104)
            for (int i = 0; i < j; ++i) {
                const double hi = h[i + j * (mr + 1)];
                const double hi1 = h[(i + 1) + j * (mr + 1)];
                h[i + j * (mr + 1)] = cs[i] * hi + sn[i] * hi1;
                h[(i + 1) + j * (mr + 1)] = -sn[i] * hi + cs[i] * hi1;
            }
            const double hjj = h[j + j * (mr + 1)];
            const double denom = std::hypot(hjj, hjj1);
            if (denom > 0.0) {
                cs[j] = hjj / denom;
                sn[j] = hjj1 / denom;
            } else {
                cs[j] = 1.0;
                sn[j] = 0.0;
            }
            h[j + j * (mr + 1)] = denom;
            h[(j + 1) + j * (mr + 1)] = 0.0;
            const double gj = g[j];
            g[j] = cs[j] * gj;
            g[j + 1] = -sn[j] * gj;

            ++out.iterations;
            ++j;
            const double est = std::fabs(g[j]);
            out.inner_residuals.push_back(est);
            if (est <= threshold || lucky) break;
            if (!ahead && j < mr && out.iterations < cfg.max_iters) launch_col(j);
        }

        // back substitution (gmres.cpp:113-119), x += M^-1 (V y), r = b - A x
        for (int i = j - 1; i >= 0; --i) {
            double s = g[i];
            for (int t = i + 1; t < j; ++t) s -= h[i + t * (mr + 1)] * y[t];
            y[i] = s / h[i + i * (mr + 1)];
        }
        // xc = sum_i y_i V_i from 0.0 in i order (gmres.cpp:121-122) as 0 - sum (-y_i) V_i (exact negation)
        for (int i = 0; i < j; ++i) ny[i] = -y[i];
        HEC_CUDA(cudaMemcpyAsync(yv.p, ny, sizeof(double) * std::max(j, 1), cudaMemcpyHostToDevice, st));
        HEC_CUDA(cudaStreamSynchronize(st));  // ny is reused next cycle
        for (int k0 = 0; k0 < std::max(j, 1); k0 += kKG)  // groups of at most kKG columns, k order kept
            mv(std::min(kKG, j - k0), V.p + k0 * ldv, yv.p + k0, k0 ? xc.p : nullptr, xc.p, 0, 1.0, nullptr, 0, 0,
               nullptr);
        if (S.M) {
            halo(xc.p);
            S.M->apply(xc.p, zloc.p, st);
            out.launches += S.M->launches_per_apply();
            k_add_v<<<grid, kT, 0, st>>>(n, xloc.p, zloc.p);
        } else {
            k_add_v<<<grid, kT, 0, st>>>(n, xloc.p, xc.p);
        }
        ++out.launches;
        halo(xloc.p);
        S.A->residual(b.p, xloc.p, r.p, st);
        ++out.launches;
        const double rn = norm(r.p);
        if (lucky && rn > threshold) stalled = true;
        rnorm = rn;
    }
    out.final_relative_residual = bnorm > 0.0 ? rnorm / bnorm : rnorm;
    HEC_CUDA(cudaMemcpyAsync(x_own, xloc.p, sizeof(double) * n, cudaMemcpyDeviceToDevice, st));
    HEC_CUDA(cudaStreamSynchronize(st));
    HEC_CUDA(cudaGetLastError());
    out.allreduces = comm.allreduces;
    out.exchanges = comm.exchanges;
    out.solve_seconds = std::chrono::duration<double>(std::chrono::steady_clock::now() - t0).count();
    return out;
}

// Single GPU: hec::gmres / hec_gmres_solve (one rank, no halo).
GmresOutcome gmres_device(const DeviceSpmv& A, DevicePrecond* M, const double* b_host, const GmresParams& cfg,
                          double* x_host) {
    if (A.n_rows() != A.n_cols()) throw std::invalid_argument("gmres: matrix must be square");
    if (M && M->n() != A.n_rows()) throw std::invalid_argument("gmres: preconditioner size mismatch");
    const int n = A.n_rows();
    DistSystem S;
    S.n_own = S.n_loc = n;
    S.A = &A;
    S.M = M;
    // one long-lived stream per preconditioner (its workspaces stay bound to it)
    std::unique_lock<std::mutex> lock;
    cudaStream_t st = nullptr;
    cudaStream_t own = nullptr;
    if (M) {
        st = M->host_stream(lock);
    } else {
        HEC_CUDA(cudaStreamCreateWithFlags(&own, cudaStreamNonBlocking));
        st = own;
    }
    struct Guard {
        cudaStream_t s;
        ~Guard() {
            if (s) cudaStreamDestroy(s);
        }
    } guard{own};
    DevBuf<double> b(std::max(n, 1)), x(std::max(n, 1));
    HEC_CUDA(cudaMemcpyAsync(b.p, b_host, sizeof(double) * n, cudaMemcpyHostToDevice, st));
    GmresOutcome o = gmres_dist(S, b.p, x.p, cfg, st);
    HEC_CUDA(cudaMemcpyAsync(x_host, x.p, sizeof(double) * n, cudaMemcpyDeviceToHost, st));
    HEC_CUDA(cudaStreamSynchronize(st));
    o.solve_seconds = o.solve_seconds;  // measured inside gmres_dist (excludes the two copies)
    return o;
}

}  // namespace hec::dev
