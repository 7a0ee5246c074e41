// Device runtime: construction of the B200 layouts, per-stream workspaces and
// launches for DeviceTri / DevicePrecond / DeviceSpmv.

#include "device_runtime.hpp"

#include <algorithm>
#include <cstdio>
#include <cstdlib>
#include <cstring>

#include "tri_kernels.cuh"

namespace hec::dev {

void cuda_fail(cudaError_t e, const char* what, const char* file, int line) {
    throw std::runtime_error(std::string("CUDA error ") + cudaGetErrorName(e) + " (" + cudaGetErrorString(e) +
                             ") at " + file + ":" + std::to_string(line) + ": " + what);
}

void require_device() {
    int count = 0;
    const cudaError_t e = cudaGetDeviceCount(&count);
    if (e != cudaSuccess || count == 0) {
        cudaGetLastError();
        throw std::runtime_error(
            "hecsolve-b200: no CUDA device available (the B200 path has no CPU fallback)");
    }
}

namespace {

int sm_count() {
    int dev = 0, sms = 0;
    HEC_CUDA(cudaGetDevice(&dev));
    HEC_CUDA(cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev));
    return sms;
}

int smem_optin() {
    int dev = 0, v = 0;
    HEC_CUDA(cudaGetDevice(&dev));
    HEC_CUDA(cudaDeviceGetAttribute(&v, cudaDevAttrMaxSharedMemoryPerBlockOptin, dev));
    return v;
}

inline int rup(int v, int m) { return (v + m - 1) / m * m; }

}  // namespace

// ------------------------------------------------------------ DeviceTri ----
DeviceTri::DeviceTri(const plan::TriSource& src, const TriOptions& opt, const plan::WaveMirror* mirror,
                     const plan::ColMirror* cmirror) {
    require_device();
    plan::validate(src);
    n_ = src.n;
    has_out_ = src.out_map != nullptr;
    stats_.n = src.n;
    stats_.nlev = src.nlev;
    long long nnz = 0;
    if (src.n > 0) nnz = src.csr_rp[src.n];
    for (long long k = 0; k < static_cast<long long>(src.ell_width) * src.n; ++k)
        if (src.ell_cols[k] != static_cast<int>(k % src.n)) ++nnz;
    stats_.nnz = nnz;
    stats_.alg_bytes = 12.0 * static_cast<double>(nnz) + 20.0 * src.n;

    strategy_ = opt.strategy == 1 ? 1 : 2;
    if (strategy_ == 2 && n_ > 0) {
        plan::WaveConfig cfg;
        cfg.ctas = opt.ctas > 0 ? std::min(opt.ctas, sm_count()) : sm_count();  // one resident CTA per SM
        // solver-shape knobs (default: chosen by the planner from the rows per CTA
        // level): HEC_WAVE_G warps per chunk, HEC_WAVE_K groups, HEC_WAVE_RPL rows per lane
        if (const char* e = std::getenv("HEC_WAVE_G")) {
            cfg.group = std::atoi(e);
            if (const char* k = std::getenv("HEC_WAVE_K")) cfg.groups = std::atoi(k);
            if (const char* r = std::getenv("HEC_WAVE_RPL")) cfg.rpl = std::atoi(r);
            if (!wave_kernel(1, cfg.group, cfg.groups, cfg.rpl, false))
                throw std::invalid_argument("HEC_WAVE_G/K/RPL: no kernel for this solver shape");
        }
        if (const char* e = std::getenv("HEC_WAVE_SLABS")) cfg.pencils = std::atoi(e) == 0;  // layout knob
        auto pow2 = [](int v) { return v > 0 && (v & (v - 1)) == 0; };
        if (const char* e = std::getenv("HEC_WAVE_RING")) {  // x-ring entries (power of two >= 1024)
            cfg.ring = std::atoi(e);
            if (!pow2(cfg.ring) || cfg.ring < 1024) throw std::invalid_argument("HEC_WAVE_RING: power of two >= 1024");
        }
        if (const char* e = std::getenv("HEC_WAVE_INFLIGHT")) {  // descriptor slots (power of two, 4..32)
            cfg.inflight = std::atoi(e);
            if (!pow2(cfg.inflight) || cfg.inflight < 4 || cfg.inflight > 32)
                throw std::invalid_argument("HEC_WAVE_INFLIGHT: power of two in [4, 32]");
        }
        if (const char* e = std::getenv("HEC_WAVE_HALO_MAX")) {  // staged-halo ring cap (power of two)
            cfg.halo_ring_max = std::atoi(e);
            if (!pow2(cfg.halo_ring_max) || cfg.ring + 1 + cfg.halo_ring_max > 65536)
                throw std::invalid_argument("HEC_WAVE_HALO_MAX: power of two with ring + 1 + halo <= 65536");
        }
        if (const char* e = std::getenv("HEC_WAVE_SPIN_NS")) spin_ns_ = std::max(0, std::atoi(e));  // poll back-off
        {
            int dev = 0;
            HEC_CUDA(cudaGetDevice(&dev));
            HEC_CUDA(cudaDeviceGetAttribute(&clock_khz_, cudaDevAttrClockRate, dev));
            clock_khz_ = std::max(clock_khz_, 1000000);  // the boost clock may exceed the reported rate: be generous
        }
        if (const char* e = std::getenv("HEC_WAVE_WATCHDOG_MS"))
            watchdog_ns_ = 1000000ULL * static_cast<unsigned long long>(std::max(1, std::atoi(e)));
        const int budget = smem_optin() - 1024;  // static shared + slack
        cfg.smem_bytes = budget;
        cfg.ctrl_bytes = kWaveCtrlBytes;
        // 7-point grid factors: the column-state kernel (HEC_WAVE_COLUMNS=1; experimental, off by default)
        const char* ce = std::getenv("HEC_WAVE_COLUMNS");
        if (ce && std::atoi(ce) != 0 && cfg.pencils && !mirror && !std::getenv("HEC_WAVE_G")) {
            plan::ColConfig cc;
            cc.ctas = cfg.ctas;
            cc.smem_bytes = budget;
            if (const char* e = std::getenv("HEC_COLS_WARPS")) cc.warps = std::atoi(e);
            if (const char* e = std::getenv("HEC_COLS_RPL")) cc.rpl = std::atoi(e);
            if (const char* e = std::getenv("HEC_COLS_RING")) cc.ring_max = std::min(plan::kColEdgeLevels - 2, std::max(3, std::atoi(e)));
            auto try_cols = [&](const plan::ColMirror* cm) {
                cc.mirror = cm;
                try {
                    build_columns(plan::build_columns(src, cc));
                } catch (const std::invalid_argument& e) {
                    if (std::getenv("HEC_DEBUG"))
                        std::fprintf(stderr, "[hec] no column layout%s: %s\n", cm ? " (mirror)" : "", e.what());
                }
            };
            if (cmirror) try_cols(cmirror);  // U of an ILU pair: L's slots reversed
            if (!cols_) try_cols(nullptr);
        }
        plan::WaveLayout P;
        bool ok = !cols_;
        if (ok) try {
            if (mirror) {
                cfg.mirror = mirror;
                try {
                    P = plan::build_wave(src, cfg);  // U as the mirror of L (no gather pass between them)
                } catch (const std::invalid_argument& e) {
                    if (std::getenv("HEC_DEBUG")) std::fprintf(stderr, "[hec] no mirrored layout: %s\n", e.what());
                    cfg.mirror = nullptr;
                }
            }
            if (!cfg.mirror) P = plan::build_wave(src, cfg);
        } catch (const std::invalid_argument& e) {
            ok = false;  // row order the wave layout cannot schedule: level launches
            if (std::getenv("HEC_DEBUG")) std::fprintf(stderr, "[hec] no wave layout: %s\n", e.what());
        }
        if (cols_) {
            stats_.strategy = strategy_;
            return;
        }
        p_ring_ = ok ? P.ring : cfg.ring;
        p_ring_off_ = kWaveCtrlBytes;
        p_halo_ring_ = ok ? P.halo_ring : 32;
        p_buf_off_ = ok ? P.buf_off : 0;
        p_buf_bytes_ = ok ? P.buf_bytes : 0;
        if (ok) {
            p_warps_ = P.warps;
            p_inflight_ = P.inflight;
            p_lead_ = P.lead;
            if (std::getenv("HEC_DEBUG"))
                std::fprintf(stderr, "[hec] wave n=%d chunks=%d ctas=%d warps=%d (%dx%d) rpl=%d W=%d ring=%d H=%d NS=%d %s grid=%dx%d max_region=%d "
                             "buf=%d exports=%lld deps ring=%lld global=%lld halo=%lld halo_values=%lld\n", P.n,
                             P.chunks, P.ctas, P.warps, P.group, P.groups, P.rpl, P.max_width, P.ring, P.halo_ring,
                             P.inflight, P.pencils ? "pencils" : (P.strips ? "strips" : "slabs"), P.grid_nx,
                             P.grid_ny, P.max_region, p_buf_bytes_, P.exports, P.ring_deps, P.global_deps,
                             P.halo_deps, P.halo_values);
            p_smem_ = p_buf_off_ + p_buf_bytes_;
            p_ctas_ = P.ctas;
            p_rpl_ = P.rpl;
            p_kernel_ = wave_kernel(P.max_width, P.group, P.groups, p_rpl_, false);
            p_kernel_trace_ = wave_kernel(P.max_width, P.group, P.groups, p_rpl_, true);
            if (!p_kernel_ || !p_kernel_trace_) throw std::runtime_error("hec: no wave kernel for this layout");
            HEC_CUDA(cudaFuncSetAttribute(p_kernel_, cudaFuncAttributeMaxDynamicSharedMemorySize, p_smem_));
            HEC_CUDA(cudaFuncSetAttribute(p_kernel_trace_, cudaFuncAttributeMaxDynamicSharedMemorySize, p_smem_));
            p_exports_ = P.exports;
            p_blob_.upload(P.blob);
            p_spans_.upload(P.span);
            p_bidx_.upload(P.bidx);
            p_cta0_.upload(P.cta_chunk0);
            p_cta0_host_ = P.cta_chunk0;
            h_chunk_r0_ = P.chunk_r0;
            mirrored_ = P.mirrored;
            wave_len_ = n_;
            p_wpos_.upload(P.wpos);
            h_wpos_ = P.wpos;
            h_bidx_ = P.bidx;
            stats_.ctas = p_ctas_;
            p_role_threads_ = wave_role_threads(P.group, P.groups, P.rpl);
            stats_.threads = p_role_threads_ + 32 * p_warps_;
            if (!p_kernel_) throw std::invalid_argument("hec_tri_create: no wave kernel for this width");
            stats_.chunks = P.chunks;
            stats_.slots = p_inflight_;
            stats_.layout = P.mirrored ? 3 : (P.pencils ? 1 : (P.strips ? 2 : 0));
            spare_ = make_workspace();
            stats_.group = P.group;
            stats_.groups = P.groups;
            stats_.rpl = P.rpl;
            stats_.width = P.max_width;
            stats_.ring = P.ring;
            stats_.halo_ring = P.halo_ring;
            stats_.device_bytes = static_cast<long long>(P.blob.size() + 4 * P.span.size() + 4 * P.cta_chunk0.size() +
                                                         4 * P.bidx.size() + 16 * P.exports);
        } else {
            strategy_ = 1;  // a chunk too large for shared memory: level launches
        }
    }
    if (strategy_ == 1 && n_ > 0) {
        int long_min = plan::kLongRowMin;
        if (const char* e = std::getenv("HEC_LEVELS_LONG")) long_min = std::max(0, std::atoi(e));  // 0: no warp rows
        plan::LevelLayout L = plan::build_levels(src, long_min);
        long_starts_ = L.long_starts;
        l_long_min_ = L.long_min;
        if (!L.long_rows.empty()) l_long_rows_.upload(L.long_rows);
        level_starts_ = L.level_starts;
        if (const char* e = std::getenv("HEC_LEVELS_PERSIST")) l_persist_ = std::atoi(e) != 0;
        if (l_persist_) l_starts_.upload(L.level_starts);
        l_width_ = L.width;
        l_ld_ = L.ld;
        l_bidx_.upload(L.bidx);
        h_bidx_ = L.bidx;
        h_wpos_.clear();  // level launches write x in solution order
        l_xidx_.upload(L.xidx);
        if (has_out_) l_oidx_.upload(L.oidx);
        l_ell_dep_.upload(L.ell_dep);
        l_ell_val_.upload(L.ell_val);
        l_diag_.upload(L.diag);
        l_tail_rp_.upload(L.tail_rp);
        l_tail_dep_.upload(L.tail_dep);
        l_tail_val_.upload(L.tail_val);
        stats_.device_bytes = static_cast<long long>(
            4 * (L.bidx.size() + L.xidx.size() + L.oidx.size() + L.ell_dep.size() + L.tail_rp.size() +
                 L.tail_dep.size() + L.long_rows.size()) +
            8 * (L.ell_val.size() + L.diag.size() + L.tail_val.size()));
        stats_.threads = 256;
        wave_len_ = n_;
        spare_ = make_workspace();
    }
    stats_.wave_len = wave_len_;
    stats_.strategy = strategy_;
}

void DeviceTri::build_columns(const plan::ColLayout& C) {
    void* k = cols_kernel(C.warps, C.rpl, C.unit, false, C.order);
    void* kt = cols_kernel(C.warps, C.rpl, C.unit, true, C.order);
    if (!k || !kt) throw std::invalid_argument("columns: no kernel for this warp count");
    const int smem = plan::kColCtrlBytes + C.ring * (C.block_bytes + 8 * C.lanes);
    HEC_CUDA(cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, smem));
    HEC_CUDA(cudaFuncSetAttribute(kt, cudaFuncAttributeMaxDynamicSharedMemorySize, smem));
    cols_ = true;
    c_info_ = C.mirror_info();
    c_blocks_.upload(C.blocks);
    c_cta_.upload(C.cta);
    c_block_bytes_ = C.block_bytes;
    c_ring_ = C.ring;
    c_warps_ = C.warps;
    c_unit_ = C.unit;
    p_kernel_ = k;
    p_kernel_trace_ = kt;
    p_smem_ = smem;
    p_ctas_ = C.ctas;
    p_warps_ = C.warps;
    p_exports_ = C.mailboxes;
    mirrored_ = C.mirrored;
    wave_len_ = C.slots;
    // the permute pass writes bp in the order the kernel reads it: a mirrored
    // layout reads slot s from bp[S-1-s]
    h_bidx_ = C.bidx;
    if (mirrored_) std::reverse(h_bidx_.begin(), h_bidx_.end());
    p_bidx_.upload(h_bidx_);
    h_wpos_ = C.wpos;
    p_wpos_.upload(h_wpos_);
    p_cta0_host_.resize(C.ctas + 1);  // level-block range of each CTA (diagnostics)
    for (int c = 0; c < C.ctas; ++c) p_cta0_host_[c] = C.cta[4 * c + 3];
    p_cta0_host_[C.ctas] = static_cast<int>(C.total_levels);
    stats_.ctas = C.ctas;
    stats_.threads = 32 * (C.warps + 1);
    stats_.chunks = static_cast<int>(C.total_levels);
    stats_.slots = C.ring;
    stats_.layout = C.mirrored ? 5 : 4;
    stats_.group = C.warps;
    stats_.groups = 1;
    stats_.rpl = C.rpl;
    stats_.width = 3;
    stats_.ring = C.ring;
    stats_.halo_ring = 0;
    stats_.wave_len = C.slots;
    stats_.device_bytes = static_cast<long long>(C.blocks.size() + 4 * C.cta.size() + 4 * C.bidx.size() +
                                                 4 * C.wpos.size() + 16 * C.mailboxes);
    if (std::getenv("HEC_DEBUG"))
        std::fprintf(stderr, "[hec] columns n=%d grid=%dx%dx%d tiles=%dx%d warps=%dx%d rpl=%d ctas=%d slots=%lld levels=%lld "
                     "ring=%d block=%d unit=%d mirrored=%d order=%d,%d,%d\n", C.n, C.nx, C.ny, C.nz, C.PX, C.PY, C.WX,
                     C.WY, C.rpl, C.ctas, C.slots, C.total_levels, C.ring, C.block_bytes, C.unit ? 1 : 0, C.mirrored ? 1 : 0,
                     C.order & 3, (C.order >> 2) & 3, (C.order >> 4) & 3);
    spare_ = make_workspace();
}

bool DeviceTri::col_mirror_info(plan::ColMirror& m) const {
    if (!cols_) return false;
    m = c_info_;
    return true;
}

void DeviceTri::launch_cols(const double* bp, double* xw, cudaStream_t st, unsigned long long* trace) {
    Workspace& w = workspace(st);
    ColArgs a{};
    a.blocks = c_blocks_.p;
    a.cta = reinterpret_cast<const int4*>(c_cta_.p);
    a.bp = bp;
    a.xw = xw;
    a.mbox = w.mailbox.p;
    a.counters = w.counters.p;
    a.slots = wave_len_;
    a.ctas = p_ctas_;
    a.nx = c_info_.nx;
    a.ny = c_info_.ny;
    a.nz = c_info_.nz;
    a.WX = c_info_.WX;
    a.WY = c_info_.WY;
    a.PX = c_info_.PX;
    a.PY = c_info_.PY;
    a.ox = c_info_.ox;
    a.oy = c_info_.oy;
    a.mbox_top0 = static_cast<long long>(p_ctas_) * (4 * c_info_.rpl * a.WY) * a.nz;
    a.block_bytes = c_block_bytes_;
    a.ring = c_ring_;
    a.bp_reversed = mirrored_ ? 1 : 0;
    a.watchdog_cycles = watchdog_ns_ / 1000000ULL * static_cast<unsigned long long>(clock_khz_);
    a.order = c_info_.order;
    a.trace = trace;
    void* args[] = {&a};
    HEC_CUDA(cudaLaunchCooperativeKernel(trace ? p_kernel_trace_ : p_kernel_, dim3(p_ctas_), dim3(32 * (c_warps_ + 1)),
                                         args, p_smem_, st));
}

DeviceTri::~DeviceTri() {
    if (h_stream_) cudaStreamDestroy(h_stream_);
}

bool DeviceTri::mirror_info(plan::WaveMirror& m) const {
    if (strategy_ != 2 || h_chunk_r0_.empty() || h_wpos_.empty()) return false;
    m.ctas = p_ctas_;
    m.cta_chunk0 = p_cta0_host_.data();
    m.chunk_r0 = h_chunk_r0_.data();
    m.wpos = h_wpos_.data();
    return true;
}

int DeviceTri::launches_per_solve() const {
    if (n_ == 0) return 0;
    // levels: the argument kernel + one kernel per level (one graph launch); wave: permute-in + wave + permute-out
    return strategy_ == 1 ? static_cast<int>(level_starts_.size()) : 3;
}

// Mailboxes, counters and scratch of the solves enqueued on one stream (so solves
// on different streams may run concurrently). The handle is created with one
// spare, which the first stream it is used on takes without allocating or
// synchronising -- so a fresh stream may go straight into CUDA-graph capture.
// Any further stream allocates (not allowed while that stream is capturing).
std::unique_ptr<DeviceTri::Workspace> DeviceTri::make_workspace() const {
    auto w = std::make_unique<Workspace>();
    if (strategy_ == 1) {  // level launches: the argument block; the graph is captured on first use
        w->largs.alloc(sizeof(LevelArgs));
        return w;
    }
    w->counters.alloc(3);  // ticket, CTAs finished, mailbox epoch (advanced by the kernel itself)
    const uint32_t init[3] = {0u, 0u, 1u};
    HEC_CUDA(cudaMemcpy(w->counters.p, init, sizeof(init), cudaMemcpyHostToDevice));
    w->mailbox.alloc(2 * static_cast<std::size_t>(std::max<long long>(p_exports_, 1)));
    w->bp.alloc(static_cast<std::size_t>(std::max<long long>(wave_len_, 1)) + 2);
    w->xw.alloc(static_cast<std::size_t>(std::max<long long>(wave_len_, 1)));
    HEC_CUDA(cudaMemset(w->mailbox.p, 0, sizeof(unsigned long long) * w->mailbox.count));  // epoch 0: empty
    HEC_CUDA(cudaDeviceSynchronize());
    return w;
}

DeviceTri::Workspace& DeviceTri::workspace(cudaStream_t st) {
    std::lock_guard<std::mutex> g(mu_);
    auto& w = ws_[st];
    if (!w) {
        if (spare_) {
            w = std::move(spare_);
        } else {
            cudaStreamCaptureStatus cs = cudaStreamCaptureStatusNone;
            HEC_CUDA(cudaStreamIsCapturing(st, &cs));
            if (cs != cudaStreamCaptureStatusNone)
                throw std::runtime_error("hec: first solve of this handle on a stream that is being captured; "
                                         "run one solve on that stream before capturing");
            w = make_workspace();
        }
    }
    return *w;
}

void DeviceTri::release_workspace(cudaStream_t st) {
    std::lock_guard<std::mutex> g(mu_);
    auto it = ws_.find(st);
    if (it == ws_.end()) return;
    if (!spare_) spare_ = std::move(it->second);  // keep one for the next stream
    ws_.erase(it);
}

void DeviceTri::permute(const double* b, double* bp, cudaStream_t st) const {
    if (n_ == 0) return;
    permute_in(b, strategy_ == 1 ? l_bidx_.p : p_bidx_.p, bp, strategy_ == 1 ? n_ : static_cast<int>(wave_len_), st);
    HEC_CUDA(cudaGetLastError());
}

void DeviceTri::solve(const double* b, double* xs, double* out, cudaStream_t st, unsigned long long* trace) {
    if (n_ == 0) return;
    if (strategy_ == 1) {
        run_levels(b, false, xs, out, st);  // the level kernels gather b themselves
        return;
    }
    Workspace& w = workspace(st);
    permute(b, w.bp.p, st);
    solve_ordered(w.bp.p, xs, out, st, trace);
}
void DeviceTri::permute_out(const double* xw, double* xs, cudaStream_t st) const {
    if (n_ == 0 || !xs) return;
    if (strategy_ == 1) {  // level launches already write the solution order
        if (xw != xs) HEC_CUDA(cudaMemcpyAsync(xs, xw, sizeof(double) * n_, cudaMemcpyDeviceToDevice, st));
        return;
    }
    permute_in(xw, p_wpos_.p, xs, n_, st);  // xs[o] = xw[wpos[o]]: coalesced writes
    HEC_CUDA(cudaGetLastError());
}

void DeviceTri::scatter_in(const double* b, double* bp, int o0, int o1, cudaStream_t st) const {
    if (o1 <= o0) return;
    scatter_rows(b + o0, p_wpos_.p + o0, bp, o1 - o0, st);
    HEC_CUDA(cudaGetLastError());
}

void DeviceTri::permute_out_range(const double* xw, double* xs, int o0, int o1, cudaStream_t st) const {
    if (o1 <= o0) return;
    permute_in(xw, p_wpos_.p + o0, xs + o0, o1 - o0, st);
    HEC_CUDA(cudaGetLastError());
}

void DeviceTri::run_levels(const double* b, bool ordered, double* xs, double* out, cudaStream_t st) {
    {
        LevelArgs a{};
        a.b = b;
        a.b_ordered = ordered ? 1 : 0;
        a.xs = xs;
        a.out = has_out_ ? out : nullptr;
        a.bidx = l_bidx_.p;
        a.xidx = l_xidx_.p;
        a.oidx = l_oidx_.p;
        a.ell_dep = l_ell_dep_.p;
        a.ell_val = l_ell_val_.p;
        a.diag = l_diag_.p;
        a.tail_rp = l_tail_rp_.p;
        a.tail_dep = l_tail_dep_.p;
        a.tail_val = l_tail_val_.p;
        a.long_rows = l_long_rows_.p;
        a.long_min = l_long_min_;
        a.width = l_width_;
        a.ld = l_ld_;
        Workspace& w = workspace(st);
        LevelArgs* dev = reinterpret_cast<LevelArgs*>(w.largs.p);
        const int nlev = static_cast<int>(level_starts_.size()) - 1;
        if (l_persist_) {
            set_level_args(a, dev, st);
            launch_levels_persist(dev, l_starts_.p, nlev, st);
            HEC_CUDA(cudaGetLastError());
            return;
        }
        if (!w.levels) {  // capture the level launches once, on a private stream
            cudaStream_t cs = nullptr;
            HEC_CUDA(cudaStreamCreateWithFlags(&cs, cudaStreamNonBlocking));
            cudaGraph_t graph = nullptr;
            HEC_CUDA(cudaStreamBeginCapture(cs, cudaStreamCaptureModeThreadLocal));
            launch_levels(dev, level_starts_.data(), long_starts_.data(), nlev, cs);
            HEC_CUDA(cudaStreamEndCapture(cs, &graph));
            HEC_CUDA(cudaGraphInstantiate(&w.levels, graph, 0));
            cudaGraphDestroy(graph);
            cudaStreamDestroy(cs);
        }
        set_level_args(a, dev, st);
        HEC_CUDA(cudaGetLastError());
        HEC_CUDA(cudaGraphLaunch(w.levels, st));
    }
}

void DeviceTri::solve_ordered(const double* bp, double* xs, double* out, cudaStream_t st, unsigned long long* trace) {
    if (n_ == 0) return;
    if (strategy_ == 1) {
        run_levels(bp, true, xs, out, st);
        return;
    }
    Workspace& w = workspace(st);
    solve_wave(bp, w.xw.p, out, st, trace);
    permute_out(w.xw.p, xs, st);
}
void DeviceTri::solve_wave(const double* bp, double* xw, double* out, cudaStream_t st, unsigned long long* trace) {
    if (n_ == 0) return;
    if (strategy_ == 1) {
        run_levels(bp, true, xw, out, st);
        return;
    }
    if (cols_) {
        launch_cols(bp, xw, st, trace);
        return;
    }
    Workspace& w = workspace(st);
    WaveArgs a{};
    a.blobs = p_blob_.p;
    a.spans = reinterpret_cast<const int4*>(p_spans_.p);
    a.cta_chunk0 = p_cta0_.p;
    a.bp = bp;
    a.xs = xw;
    a.out = has_out_ ? out : nullptr;
    a.mbox = w.mailbox.p;
    a.counters = w.counters.p;
    a.ctas = p_ctas_;
    a.inflight = p_inflight_;
    a.inflight_log2 = __builtin_ctz(static_cast<unsigned>(p_inflight_));
    a.lead = p_lead_;
    a.ring = p_ring_;
    a.halo_ring = p_halo_ring_;
    a.ring_off = p_ring_off_;
    a.buf_off = p_buf_off_;
    a.buf_bytes = p_buf_bytes_;
    a.spin_ns = spin_ns_;
    a.watchdog_cycles = watchdog_ns_ / 1000000ULL * static_cast<unsigned long long>(clock_khz_);  // ms * kHz
    a.trace = trace;
    void* args[] = {&a};
    // cooperative: every CTA resident at once (CTAs wait on each other's rows)
    HEC_CUDA(cudaLaunchCooperativeKernel(trace ? p_kernel_trace_ : p_kernel_, dim3(p_ctas_),
                                         dim3(p_role_threads_ + 32 * p_warps_), args, p_smem_, st));
}

void DeviceTri::solve_host(const double* b, double* x) {
    if (n_ == 0) return;
    std::lock_guard<std::mutex> g(h_mu_);  // serialises host-path callers of this handle
    if (!h_stream_) HEC_CUDA(cudaStreamCreateWithFlags(&h_stream_, cudaStreamNonBlocking));
    if (h_b_.count < static_cast<std::size_t>(n_)) {
        h_b_.alloc(n_);
        h_x_.alloc(n_);
    }
    const std::size_t bytes = sizeof(double) * n_;
    HEC_CUDA(cudaMemcpyAsync(h_b_.p, b, bytes, cudaMemcpyHostToDevice, h_stream_));
    solve(h_b_.p, h_x_.p, nullptr, h_stream_);
    HEC_CUDA(cudaMemcpyAsync(x, h_x_.p, bytes, cudaMemcpyDeviceToHost, h_stream_));
    HEC_CUDA(cudaStreamSynchronize(h_stream_));
}

// -------------------------------------------------------- DevicePrecond ----
DevicePrecond::DevicePrecond(int n_in, int n_out, int n_ext, const int* gather, const int* out_index,
                             plan::TriSource l, plan::TriSource u, const TriOptions& opt)
    : n_(n_in), n_out_(n_out), n_ext_(n_ext) {
    require_device();
    identity_ = false;
    if (n_in < 0 || n_out < 0 || n_ext < 0) throw std::invalid_argument("hec_precond_create_local: negative size");
    if (l.n != n_ext || u.n != n_ext) throw std::invalid_argument("hec_precond_create_local: factor size mismatch");
    if (n_ext > 0 && (!gather || !out_index)) throw std::invalid_argument("hec_precond_create_local: missing map");
    std::vector<int> hits(static_cast<std::size_t>(n_out), 0);
    for (int k = 0; k < n_ext; ++k) {
        if (gather[k] < 0 || gather[k] >= n_in)
            throw std::invalid_argument("hec_precond_create_local: gather out of range");
        if (out_index[k] >= n_out) throw std::invalid_argument("hec_precond_create_local: output index out of range");
        if (out_index[k] >= 0 && ++hits[out_index[k]] > 1)
            throw std::invalid_argument("hec_precond_create_local: output row written twice");
    }
    // identity maps (one subdomain holding the whole vector): the square form
    identity_ = n_in == n_out && n_ext == n_in;
    for (int k = 0; identity_ && k < n_ext; ++k) identity_ = gather[k] == k && out_index[k] == k;
    if (!identity_) {
        l.b_map = gather;
        u.out_map = out_index;
    }
    l_ = std::make_unique<DeviceTri>(l, opt);
    build_upper(u, opt);
}

DevicePrecond::DevicePrecond(int n, int n_ext, const int* gather, const char* owned, plan::TriSource l,
                             plan::TriSource u, const TriOptions& opt)
    : n_(n), n_out_(n), n_ext_(n_ext) {
    require_device();
    identity_ = gather == nullptr;
    if (identity_ && n_ext != n) throw std::invalid_argument("hec_precond_create: identity map needs n_ext == n");
    if (!identity_ && n_ext == n && owned) {  // one block covering every row in order: the square form
        bool id = true;
        for (int k = 0; id && k < n; ++k) id = gather[k] == k && owned[k];
        identity_ = id;
    }
    if (l.n != n_ext || u.n != n_ext) throw std::invalid_argument("hec_precond_create: factor size mismatch");
    std::vector<int> out_map;
    if (!identity_) {
        for (int k = 0; k < n_ext; ++k)
            if (gather[k] < 0 || gather[k] >= n) throw std::invalid_argument("hec_precond_create: gather out of range");
        out_map.resize(n_ext);
        std::vector<int> hits(n, 0);
        for (int k = 0; k < n_ext; ++k) {
            out_map[k] = owned[k] ? gather[k] : -1;
            if (owned[k]) ++hits[gather[k]];
        }
        for (int g = 0; g < n; ++g)
            if (hits[g] != 1) throw std::invalid_argument("hec_precond_create: every row must be owned exactly once");
        l.b_map = gather;           // L reads r[gather[o]]
        u.out_map = out_map.data(); // U scatters owned rows into x
    }
    l_ = std::make_unique<DeviceTri>(l, opt);
    build_upper(u, opt);
}

// U as the mirror of L's wave layout when that is valid (its right-hand side is
// then L's wave-ordered output read backwards, chunk by chunk: no pass between
// the solves); otherwise its own layout plus the composed gather.
void DevicePrecond::build_upper(const plan::TriSource& u, const TriOptions& opt) {
    plan::WaveMirror m;
    plan::ColMirror cm;
    const bool no = std::getenv("HEC_NO_MIRROR") != nullptr;
    if (!no && l_->col_mirror_info(cm))
        u_ = std::make_unique<DeviceTri>(u, opt, nullptr, &cm);
    else
        u_ = std::make_unique<DeviceTri>(u, opt, (!no && l_->mirror_info(m)) ? &m : nullptr);
    if (!u_->mirrored()) compose();
}

DevicePrecond::~DevicePrecond() {
    if (h_stream_) cudaStreamDestroy(h_stream_);
    if (h_in_) cudaStreamDestroy(h_in_);
    if (h_out_) cudaStreamDestroy(h_out_);
    for (int k = 0; k < kMaxSlices; ++k) {
        if (ev_in_[k]) cudaEventDestroy(ev_in_[k]);
        if (ev_out_[k]) cudaEventDestroy(ev_out_[k]);
    }
}

DevicePrecond::Workspace& DevicePrecond::workspace(cudaStream_t st) {
    std::lock_guard<std::mutex> g(mu_);
    auto& w = ws_[st];
    if (!w) {
        w = std::make_unique<Workspace>();
        const std::size_t ll = static_cast<std::size_t>(std::max<long long>(l_->wave_len(), 1));
        const std::size_t lu = static_cast<std::size_t>(std::max<long long>(u_->wave_len(), 1));
        // k_wave inputs: bulk copies of b read up to one element past the last row
        w->bl.alloc(ll + 2);
        w->yw.alloc(ll + 2);  // also U's input when U mirrors L
        w->bu.alloc(lu + 2);
        w->xw.alloc(lu);
    }
    return *w;
}

void DevicePrecond::apply(const double* r, double* x, cudaStream_t st) {
    if (n_ext_ == 0) return;
    Workspace& w = workspace(st);
    // L from r gathered into its row order, its output left in wave order; U's
    // right-hand side is gathered straight from there through the composed map
    // (no pass through the solution order in between)
    l_->permute(r, w.bl.p, st);
    if (identity_) {
        apply_middle(w.bl.p, w.xw.p, w, st);
        u_->permute_out(w.xw.p, x, st);
        return;
    }
    l_->solve_wave(w.bl.p, w.yw.p, nullptr, st);
    const double* bu = w.yw.p;  // mirrored U: L's output as it lies
    if (!u_->mirrored()) {
        permute_in(w.yw.p, lu_map_.p, w.bu.p, static_cast<int>(u_->wave_len()), st);
        HEC_CUDA(cudaGetLastError());
        bu = w.bu.p;
    }
    u_->solve_wave(bu, w.xw.p, x, st);  // owned rows scattered into x by the kernel
}

// L from its reordered input, then U, output left in U's wave order (square form)
void DevicePrecond::apply_middle(const double* bl, double* xw, Workspace& w, cudaStream_t st) {
    l_->solve_wave(bl, w.yw.p, nullptr, st);
    const double* bu = w.yw.p;  // mirrored U: L's output as it lies
    if (!u_->mirrored()) {
        permute_in(w.yw.p, lu_map_.p, w.bu.p, static_cast<int>(u_->wave_len()), st);
        HEC_CUDA(cudaGetLastError());
        bu = w.bu.p;
    }
    u_->solve_wave(bu, xw, nullptr, st);
}

// slices of at least 2^20 rows (a few microseconds of permutation each), at most 8
int DevicePrecond::host_slices() const {
    if (!identity_ || n_ != n_out_ || !l_->sliceable() || !u_->sliceable()) return 1;
    if (std::getenv("HEC_HOST_SLICES")) return std::max(1, std::min(kMaxSlices, std::atoi(std::getenv("HEC_HOST_SLICES"))));
    return std::max(1, std::min(kMaxSlices, n_ >> 20));
}
void DevicePrecond::compose() {
    const std::vector<int>& bu = u_->host_bidx();
    const std::vector<int>& wl = l_->host_wpos();
    std::vector<int> m(bu.size());
    for (std::size_t p = 0; p < bu.size(); ++p) m[p] = wl.empty() ? bu[p] : wl[bu[p]];
    lu_map_.upload(m);
}

cudaStream_t DevicePrecond::host_stream(std::unique_lock<std::mutex>& lock) {
    lock = std::unique_lock<std::mutex>(h_mu_);
    if (!h_stream_) HEC_CUDA(cudaStreamCreateWithFlags(&h_stream_, cudaStreamNonBlocking));
    return h_stream_;
}

int DevicePrecond::launches_per_apply() const {
    if (n_ext_ == 0) return 0;
    return l_->launches_per_solve() + u_->launches_per_solve() - (identity_ ? 1 : 2) - (u_->mirrored() ? 1 : 0);
}

void DevicePrecond::apply_host(const double* r, double* x) {
    if (n_ == 0 && n_out_ == 0) return;
    std::lock_guard<std::mutex> g(h_mu_);
    if (!h_stream_) HEC_CUDA(cudaStreamCreateWithFlags(&h_stream_, cudaStreamNonBlocking));
    if (h_r_.count < static_cast<std::size_t>(std::max(n_, 1))) h_r_.alloc(std::max(n_, 1));
    if (h_x_.count < static_cast<std::size_t>(std::max(n_out_, 1))) h_x_.alloc(std::max(n_out_, 1));
    const int S = host_slices();
    if (S <= 1) {
        HEC_CUDA(cudaMemcpyAsync(h_r_.p, r, sizeof(double) * n_, cudaMemcpyHostToDevice, h_stream_));
        apply(h_r_.p, h_x_.p, h_stream_);
        HEC_CUDA(cudaMemcpyAsync(x, h_x_.p, sizeof(double) * n_out_, cudaMemcpyDeviceToHost, h_stream_));
        HEC_CUDA(cudaStreamSynchronize(h_stream_));
        return;
    }
    // the copies dominate (2 x 8n bytes over PCIe against ~1 ms of solves at 256^3):
    // each input slice is permuted while the next one is in flight, and each
    // output slice is copied back while the next one is permuted
    if (!h_in_) {
        HEC_CUDA(cudaStreamCreateWithFlags(&h_in_, cudaStreamNonBlocking));
        HEC_CUDA(cudaStreamCreateWithFlags(&h_out_, cudaStreamNonBlocking));
        for (int k = 0; k < kMaxSlices; ++k) {
            HEC_CUDA(cudaEventCreateWithFlags(&ev_in_[k], cudaEventDisableTiming));
            HEC_CUDA(cudaEventCreateWithFlags(&ev_out_[k], cudaEventDisableTiming));
        }
    }
    Workspace& w = workspace(h_stream_);
    const int step = ((n_ + S - 1) / S + 3) & ~3;  // slice starts stay 16-byte aligned
    for (int k = 0; k < S; ++k) {
        const int o0 = std::min(n_, k * step), o1 = std::min(n_, o0 + step);
        HEC_CUDA(cudaMemcpyAsync(h_r_.p + o0, r + o0, sizeof(double) * (o1 - o0), cudaMemcpyHostToDevice, h_in_));
        HEC_CUDA(cudaEventRecord(ev_in_[k], h_in_));
        HEC_CUDA(cudaStreamWaitEvent(h_stream_, ev_in_[k], 0));
        l_->scatter_in(h_r_.p, w.bl.p, o0, o1, h_stream_);
    }
    apply_middle(w.bl.p, w.xw.p, w, h_stream_);
    for (int k = 0; k < S; ++k) {
        const int o0 = std::min(n_, k * step), o1 = std::min(n_, o0 + step);
        u_->permute_out_range(w.xw.p, h_x_.p, o0, o1, h_stream_);
        HEC_CUDA(cudaEventRecord(ev_out_[k], h_stream_));
        HEC_CUDA(cudaStreamWaitEvent(h_out_, ev_out_[k], 0));
        HEC_CUDA(cudaMemcpyAsync(x + o0, h_x_.p + o0, sizeof(double) * (o1 - o0), cudaMemcpyDeviceToHost, h_out_));
    }
    HEC_CUDA(cudaStreamSynchronize(h_out_));
}

}  // namespace hec::dev
