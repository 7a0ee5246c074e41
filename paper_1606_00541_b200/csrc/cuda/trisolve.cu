// B200 (sm_100a) triangular-solve kernels on the HEC layouts of tri_plan.hpp.
//
// Reference semantics: hec::solve, proj/src/triangular.cpp:90-135 (Algorithm 2
// of arXiv 1606.00541). Per row: acc = b; acc -= v * x[dep] in stored order;
// x = acc / diag. Every product and difference is rounded separately
// (__dmul_rn/__dsub_rn: no FMA contraction, like the reference's mulsd/subsd)
// and the division is the IEEE-correct __ddiv_rn, so results are bitwise equal
// to the reference for any schedule.
//
// Two strategies:
//  * k_level_rows   one launch per level, thread per reordered row (baseline;
//                   the reference's level barrier becomes a kernel boundary).
//  * k_wave         persistent wavefront, one CTA per SM (tri_plan.hpp). CTA c
//                   owns a contiguous block of lower-frame rows, each solver
//                   warp a fixed slice of it. Warp roles: 0 = producer (byte-
//                   ring allocation + cp.async.bulk of chunk blobs into shared
//                   memory), 1..kWaveWaiters = waiters (cp.async gather of b,
//                   polling of the epoch-tagged mailboxes that carry values
//                   from lower CTAs), the rest = solvers. The reference's
//                   per-level barrier becomes dataflow: a warp starts its part
//                   of level k as soon as the warps it reads from finished
//                   level k-1 (shared-memory progress counters) and the
//                   foreign values are staged; no grid or CTA barrier.

#include <cuda_runtime.h>

#include <algorithm>
#include <cstdint>

#include "tri_kernels.cuh"
#include "tri_plan.hpp"

namespace hec::dev {

// ------------------------------------------------------------------ PTX ----
__device__ __forceinline__ uint32_t smem_u32(const void* p) {
    return static_cast<uint32_t>(__cvta_generic_to_shared(p));
}
__device__ __forceinline__ void mbar_init(uint64_t* bar, uint32_t count) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(bar)), "r"(count) : "memory");
}
__device__ __forceinline__ void mbar_arrive(uint64_t* bar) {
    asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(smem_u32(bar)) : "memory");
}
__device__ __forceinline__ void mbar_expect_tx(uint64_t* bar, uint32_t bytes) {
    asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(bar)), "r"(bytes)
                 : "memory");
}
__device__ __forceinline__ bool mbar_try_wait(uint64_t* bar, uint32_t parity) {
    uint32_t ok;
    asm volatile(
        "{\n\t.reg .pred p;\n\t"
        "mbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2;\n\t"
        "selp.u32 %0, 1, 0, p;\n\t}"
        : "=r"(ok)
        : "r"(smem_u32(bar)), "r"(parity)
        : "memory");
    return ok != 0;
}
__device__ __forceinline__ void mbar_wait(uint64_t* bar, uint32_t parity) {
    while (!mbar_try_wait(bar, parity)) {
    }
}
__device__ __forceinline__ void bulk_g2s(void* dst, const void* src, uint32_t bytes, uint64_t* bar) {
    asm volatile(
        "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(
            smem_u32(dst)),
        "l"(src), "r"(bytes), "r"(smem_u32(bar))
        : "memory");
}
__device__ __forceinline__ void cp_async8(void* dst, const void* src) {
    asm volatile("cp.async.ca.shared.global [%0], [%1], 8;" ::"r"(smem_u32(dst)), "l"(src) : "memory");
}
__device__ __forceinline__ void cp_async_arrive(uint64_t* bar) {
    asm volatile("cp.async.mbarrier.arrive.noinc.shared::cta.b64 [%0];" ::"r"(smem_u32(bar)) : "memory");
}
__device__ __forceinline__ unsigned long long ld_relaxed_u64(const unsigned long long* p) {
    unsigned long long v;
    asm volatile("ld.relaxed.gpu.global.b64 %0, [%1];" : "=l"(v) : "l"(p) : "memory");
    return v;
}
__device__ __forceinline__ void st_relaxed_u64(unsigned long long* p, unsigned long long v) {
    asm volatile("st.relaxed.gpu.global.b64 [%0], %1;" ::"l"(p), "l"(v) : "memory");
}
__device__ __forceinline__ void named_bar_sync(int id, int count) {
    asm volatile("bar.sync %0, %1;" ::"r"(id), "r"(count) : "memory");
}
__device__ __forceinline__ uint64_t gtimer() {
    uint64_t t;
    asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
    return t;
}

// IEEE row update, never contracted into an FMA.
__device__ __forceinline__ double sub_prod(double acc, double v, double x) {
    return __dsub_rn(acc, __dmul_rn(v, x));
}

// -------------------------------------------------------------- LEVELS ----
__global__ void k_level_rows(LevelArgs a, int r0, int r1) {
    const int r = r0 + blockIdx.x * blockDim.x + threadIdx.x;
    if (r >= r1) return;
    double acc = a.b[a.b_ordered ? r : a.bidx[r]];
    for (int k = 0; k < a.width; ++k) {
        const size_t slot = static_cast<size_t>(k) * a.ld + r;
        const int d = a.ell_dep[slot];
        if (d >= 0) acc = sub_prod(acc, a.ell_val[slot], a.xs[d]);
    }
    for (int t = a.tail_rp[r]; t < a.tail_rp[r + 1]; ++t) acc = sub_prod(acc, a.tail_val[t], a.xs[a.tail_dep[t]]);
    const double x = __ddiv_rn(acc, a.diag[r]);
    a.xs[a.xidx[r]] = x;
    if (a.out) {
        const int o = a.oidx[r];
        if (o >= 0) a.out[o] = x;
    }
}

void launch_levels(const LevelArgs& a, const int* level_starts_host, int nlev, cudaStream_t st) {
    for (int k = 0; k < nlev; ++k) {
        const int r0 = level_starts_host[k], r1 = level_starts_host[k + 1];
        const int m = r1 - r0;
        const int tpb = m >= 256 ? 256 : (m >= 128 ? 128 : 64);
        k_level_rows<<<(m + tpb - 1) / tpb, tpb, 0, st>>>(a, r0, r1);
    }
}

// ------------------------------------------------------------------ WAVE ----
using plan::WaveHeader;

__device__ __forceinline__ uint32_t ld_relaxed_u32(const uint32_t* p) {
    uint32_t v;
    asm volatile("ld.relaxed.gpu.global.u32 %0, [%1];" : "=r"(v) : "l"(p) : "memory");
    return v;
}
__device__ __forceinline__ uint32_t ld_volatile_u32(const uint32_t* p) {
    uint32_t v;
    asm volatile("ld.volatile.shared.u32 %0, [%1];" : "=r"(v) : "r"(smem_u32(p)) : "memory");
    return v;
}
__device__ __forceinline__ void st_volatile_u32(uint32_t* p, uint32_t v) {
    asm volatile("st.volatile.shared.u32 [%0], %1;" ::"r"(smem_u32(p)), "r"(v) : "memory");
}
__device__ __forceinline__ uint2 ld_volatile_v2(const uint2* p) {
    uint2 v;
    asm volatile("ld.volatile.shared.v2.u32 {%0, %1}, [%2];" : "=r"(v.x), "=r"(v.y) : "r"(smem_u32(p)) : "memory");
    return v;
}
__device__ __forceinline__ void st_volatile_v2(uint2* p, uint32_t x, uint32_t y) {
    asm volatile("st.volatile.shared.v2.u32 [%0], {%1, %2};" ::"r"(smem_u32(p)), "r"(x), "r"(y) : "memory");
}
__device__ __forceinline__ double lds_f64(uint32_t addr) {
    double v;
    asm volatile("ld.shared.f64 %0, [%1];" : "=d"(v) : "r"(addr));
    return v;
}
__device__ __forceinline__ void cp_async_commit() { asm volatile("cp.async.commit_group;" ::: "memory"); }
__device__ __forceinline__ void cp_async_wait_all() { asm volatile("cp.async.wait_all;" ::: "memory"); }
__device__ __forceinline__ ulonglong2 ld_relaxed_v2(const unsigned long long* p) {
    ulonglong2 v;
    asm volatile("ld.relaxed.gpu.global.v2.u64 {%0, %1}, [%2];" : "=l"(v.x), "=l"(v.y) : "l"(p) : "memory");
    return v;
}
__device__ __forceinline__ void st_relaxed_v2(unsigned long long* p, unsigned long long lo, unsigned long long hi) {
    asm volatile("st.relaxed.gpu.global.v2.u64 [%0], {%1, %2};" ::"l"(p), "l"(lo), "l"(hi) : "memory");
}

// Mailbox words carry 32 value bits and the solve's epoch each, so one
// 8-byte single-copy-atomic word never mixes two solves.
__device__ __forceinline__ bool mail_ok(ulonglong2 v, uint32_t ep) {
    return static_cast<uint32_t>(v.x >> 32) == ep && static_cast<uint32_t>(v.y >> 32) == ep;
}
__device__ __forceinline__ double mail_value(ulonglong2 v) {
    return __longlong_as_double(static_cast<long long>((v.y << 32) | (v.x & 0xffffffffULL)));
}
__device__ __forceinline__ void mail_store(unsigned long long* box, double x, uint32_t ep) {
    const unsigned long long bits = static_cast<unsigned long long>(__double_as_longlong(x));
    const unsigned long long tag = static_cast<unsigned long long>(ep) << 32;
    st_relaxed_v2(box, (bits & 0xffffffffULL) | tag, (bits >> 32) | tag);
}

// x = a / d, correctly rounded, with y = RN(1/d) computed off the critical
// path: q = RN(a y), r = a - d q (exact), q' = RN(q + r y) is RN(a/d) while a
// and q' stay clear of the under/overflow ranges (Markstein; the same tail as
// the CUDA __ddiv_rn fast path, fed a correctly rounded reciprocal). Outside
// the guard -- zeros, huge/tiny operands, Inf/NaN -- the IEEE division runs.
// tools/markstein_check.c sweeps the identity on the host.
__device__ __noinline__ double div_slow(double a, double d) { return __ddiv_rn(a, d); }
__device__ __forceinline__ double div_rn(double a, double d, double y) {
    const double q = __dmul_rn(a, y);
    const double r = __fma_rn(-d, q, a);
    const double q1 = __fma_rn(r, y, q);
    const double aa = fabs(a), aq = fabs(q1);
    if (__builtin_expect(aa > 0x1p-900 && aa < 0x1p900 && aq > 0x1p-900 && aq < 0x1p900, 1)) return q1;
    return div_slow(a, d);
}

// Dependency value (see tri_plan.hpp): ring / zero slot / staged halo live in
// shared memory at ring_s + 8 d (d <= R) or hb_s + 8 d (d > R); d < 0 is x[-d-1].
__device__ __forceinline__ uint32_t dep_addr(int d, int R, uint32_t ring_s, uint32_t hb_s) {
    return (d <= R ? ring_s : hb_s) + 8u * static_cast<uint32_t>(d);
}
__device__ __forceinline__ double dep_value(int d, int R, uint32_t ring_s, uint32_t hb_s, const double* xs) {
    return d >= 0 ? lds_f64(dep_addr(d, R, ring_s, hb_s)) : __ldcg(xs + (-d - 1));
}

// acc -= v[u] * x[dep[u]] for the W sliced-ELL slots of row t (padding slots
// hold 0 * 0.0, which leaves acc bitwise unchanged), products formed first,
// then the subtractions in slot order (reference triangular.cpp:118-122).
template <int W>
__device__ __forceinline__ double accumulate(double acc, const int* dep, const double* val, int mp, int t, int R,
                                             uint32_t ring_s, uint32_t hb_s, const double* xs, bool global) {
    double p[W];
#pragma unroll
    for (int u = 0; u < W; ++u) {
        const int d = dep[u * mp + t];
        double xv;
        if (global) xv = dep_value(d, R, ring_s, hb_s, xs);
        else xv = lds_f64(dep_addr(d, R, ring_s, hb_s));
        p[u] = __dmul_rn(val[u * mp + t], xv);
    }
#pragma unroll
    for (int u = 0; u < W; ++u) acc = __dsub_rn(acc, p[u]);
    return acc;
}

// Shared-memory control block (kWaveCtrlBytes): prog[32] | hready[32] (+pad)
// | roff[32] | bar_full[32] | bar_empty[32] | (unused) | boff[32] | ticket.
// roff = region start (producer), boff = blob start.
template <int W, int NW, int RPL, bool TRACE>
__global__ void __launch_bounds__(kWaveRoleThreads + 32 * NW, 1) k_wave(WaveArgs a) {
    constexpr int kSeg = plan::kWaveHeaderBytes;
    constexpr int kDiag = kSeg + (8 * NW + 15) / 16 * 16;  // seg table rounded to 16 bytes (tri_plan.hpp)
    extern __shared__ __align__(128) unsigned char smem[];
    uint32_t* prog = reinterpret_cast<uint32_t*>(smem);
    uint32_t* hready = reinterpret_cast<uint32_t*>(smem + 128);
    uint32_t* roff = reinterpret_cast<uint32_t*>(smem + 384);
    uint64_t* bar_full = reinterpret_cast<uint64_t*>(smem + 512);
    uint64_t* bar_empty = bar_full + 32;
    uint32_t* boff = reinterpret_cast<uint32_t*>(smem + 1280);
    int* s_cta = reinterpret_cast<int*>(smem + 1408);
    __shared__ uint32_t s_epoch;
    double* ring = reinterpret_cast<double*>(smem + a.ring_off);
    unsigned char* buf = smem + a.buf_off;
    const int NS = a.inflight, LG = a.inflight_log2;
    const int R = a.ring;

    const int tid = threadIdx.x;
    const int warp = tid >> 5, lane = tid & 31;
    if (tid < 128) prog[tid] = 0u;  // prog, slot, roff
    if (tid == 0) {
        *s_cta = static_cast<int>(atomicAdd(&a.counters[0], 1u));
        s_epoch = ld_relaxed_u32(&a.counters[2]);
        for (int s = 0; s < NS; ++s) {
            mbar_init(&bar_full[s], 1);
            mbar_init(&bar_empty[s], NW);
        }
        asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
        ring[R] = 0.0;  // the slot padding entries point at
    }
    __syncthreads();
    const int c = *s_cta;
    const int c0 = a.cta_chunk0[c];
    const int nch = a.cta_chunk0[c + 1] - c0;
    auto tr = [&](int j, int k) -> unsigned long long& { return a.trace[static_cast<size_t>(c0 + j) * 64 + k]; };

    if (warp == 0) {
        // ------------- producer: byte-ring allocation + bulk copy of chunk blobs -------------
        int head = 0, oldest = 0;
        int4 sp_a = make_int4(0, 0, 0, 0), sp_b = make_int4(0, 0, 0, 0);
        for (int j = 0; j < nch; ++j) {
            if ((j & 31) == 0) {
                const int g = j + lane;
                sp_a = g < nch ? a.spans[2 * (c0 + g)] : make_int4(0, 0, 0, 0);
                sp_b = g < nch ? a.spans[2 * (c0 + g) + 1] : make_int4(0, 0, 0, 0);
            }
            const int off16 = __shfl_sync(0xffffffffu, sp_a.x, j & 31);
            const int bytes = __shfl_sync(0xffffffffu, sp_a.y, j & 31);
            const int need = __shfl_sync(0xffffffffu, sp_a.z, j & 31);
            const int r0 = __shfl_sync(0xffffffffu, sp_a.w, j & 31);
            const int bbytes = __shfl_sync(0xffffffffu, sp_b.x, j & 31);
            const int bcopy = __shfl_sync(0xffffffffu, sp_b.y, j & 31);
            const int s = j & (NS - 1);
            if (j >= NS) {
                mbar_wait(&bar_empty[s], ((j >> LG) - 1) & 1);
                oldest = max(oldest, j - NS + 1);
            }
            int pos;
            for (;;) {
                if (oldest == j) {  // nothing in flight: restart at the front
                    pos = 0;
                    break;
                }
                // live region starts at the oldest chunk's region (its b area)
                const int tail = static_cast<int>(roff[oldest & (NS - 1)]);
                if (head >= tail) {
                    if (head + need <= a.buf_bytes) { pos = head; break; }
                    if (need < tail) { pos = 0; break; }
                } else if (head + need < tail) {
                    pos = head;
                    break;
                }
                mbar_wait(&bar_empty[oldest & (NS - 1)], (oldest >> LG) & 1);
                ++oldest;
            }
            if (lane == 0) {
                roff[s] = static_cast<uint32_t>(pos);
                boff[s] = static_cast<uint32_t>(pos + bbytes);
                if (TRACE) tr(j, 0) = gtimer();
                mbar_expect_tx(&bar_full[s], static_cast<uint32_t>(bytes + bcopy));
                bulk_g2s(buf + pos + bbytes, a.blobs + static_cast<size_t>(off16) * 16, static_cast<uint32_t>(bytes),
                         &bar_full[s]);
                bulk_g2s(buf + pos, a.bp + (r0 & ~1), static_cast<uint32_t>(bcopy), &bar_full[s]);
            }
            __syncwarp();
            head = pos + need;
        }
    } else if (warp <= kWaveWaiters) {
        // ------------- waiters (round robin over chunks): stage the values this
        // chunk reads from lower CTAs, then publish it -------------
        const uint32_t ep = s_epoch;
        for (int j = warp - 1; j < nch; j += kWaveWaiters) {
            const int s = j & (NS - 1);
            mbar_wait(&bar_full[s], (j >> LG) & 1);
            unsigned char* blob = buf + boff[s];  // region = [b][blob][staged halo]
            const int4 hb1 = *reinterpret_cast<const int4*>(blob + 16);  // nhalo, halo, tptr, bytes
            if (TRACE && lane == 0) tr(j, 1) = gtimer();
            const int nhalo = hb1.x;
            if (nhalo) {
                const int* hid = reinterpret_cast<const int*>(blob + hb1.y);
                double* hst = reinterpret_cast<double*>(blob + hb1.w);
                for (int t0 = 0; t0 < nhalo; t0 += 32 * 8) {
                    ulonglong2 v[8];
                    int id[8];
                    unsigned miss = 0;
#pragma unroll
                    for (int u = 0; u < 8; ++u) {  // 8 loads in flight per lane
                        const int t = t0 + u * 32 + lane;
                        id[u] = t < nhalo ? hid[t] : -1;
                        if (id[u] >= 0) {
                            v[u] = ld_relaxed_v2(a.mbox + 2 * static_cast<size_t>(id[u]));
                            miss |= 1u << u;
                        }
                    }
                    // re-read every value not produced yet, all in flight, until complete
                    for (;;) {
#pragma unroll
                        for (int u = 0; u < 8; ++u)
                            if ((miss >> u) & 1u) {
                                if (mail_ok(v[u], ep)) {
                                    hst[t0 + u * 32 + lane] = mail_value(v[u]);
                                    miss &= ~(1u << u);
                                }
                            }
                        if (!__any_sync(0xffffffffu, miss != 0)) break;
#pragma unroll
                        for (int u = 0; u < 8; ++u)
                            if ((miss >> u) & 1u) v[u] = ld_relaxed_v2(a.mbox + 2 * static_cast<size_t>(id[u]));
                    }
                }
            }
            if (TRACE && lane == 0) tr(j, 2) = gtimer();
            __syncwarp();
            asm volatile("fence.acq_rel.cta;" ::: "memory");
            if (lane == 0) {
                st_volatile_u32(&hready[s], static_cast<uint32_t>(j + 1));
                if (TRACE) tr(j, 3) = gtimer();
            }
        }
    } else {
        // ------------- solvers: warp w owns a fixed slice of the CTA's rows -------------
        const int w = warp - 1 - kWaveWaiters;
        const uint32_t ep = s_epoch;
        const uint32_t ring_s = smem_u32(ring);
        const int L = a.lead;
        double* const xs = a.xs;
        double* const outv = a.out;
        unsigned long long* const mbox = a.mbox;
        double pend_x[RPL];
        int pend_xi[RPL], pend_o[RPL];
#pragma unroll
        for (int k = 0; k < RPL; ++k) {
            pend_x[k] = 0.0;
            pend_xi[k] = pend_o[k] = -1;
        }
        // TRACE: SM-clock breakdown of one chunk for solver warps 0 and 5 (trace words 48..63)
        const int cw = (w == 5) ? 56 : -1;
        long long c_top = 0;
#define HEC_STAMP(K, DEP)                                                        \
    if (TRACE && cw >= 0 && lane == 0) {                                           \
        asm volatile("" ::"r"(static_cast<int>(DEP)) : "memory");                 \
        tr(j, cw + (K)) = static_cast<unsigned long long>(clock64() - c_top);      \
    }
        for (int j = 0; j < nch; ++j) {
            const int s = j & (NS - 1);
            if (TRACE) c_top = clock64();
            mbar_wait(&bar_full[s], (j >> LG) & 1);  // blob and b landed
            HEC_STAMP(0, 0)
            if (TRACE && lane == 0) tr(j, 8 + 3 * w) = gtimer();
            const unsigned char* blob = buf + boff[s];
            const int4 h0 = *reinterpret_cast<const int4*>(blob);  // m, mp, q0, flags
            const uint2 sg = *reinterpret_cast<const uint2*>(blob + kSeg + 8 * w);
            const int t0 = static_cast<int>(sg.x & 0xffffu), t1 = static_cast<int>(sg.x >> 16);
            HEC_STAMP(1, t0 + h0.x)
            if (h0.w & 16)  // values from lower CTAs staged by the waiters
                while (ld_volatile_u32(&hready[s]) != static_cast<uint32_t>(j + 1)) {
                    if (a.spin_ns) __nanosleep(a.spin_ns);
                }
            // the warps this segment reads from must have finished chunk j-1, and every
            // warp chunk j-lead (no warp runs further ahead: ring safety, tri_plan.hpp)
            if (NW > 1 && lane < NW) {
                const uint32_t need = ((sg.y >> lane) & 1u) ? static_cast<uint32_t>(j)
                                                            : static_cast<uint32_t>(max(0, j - L + 1));
                while (ld_volatile_u32(&prog[lane]) < need) {
                    if (a.spin_ns) __nanosleep(a.spin_ns);
                }
            }
            __syncwarp();
            if (TRACE && lane == 0) tr(j, 9 + 3 * w) = gtimer();
            HEC_STAMP(2, 0)
            if (t1 > t0) {
                const int mp = h0.y, q0 = h0.z, flags = h0.w;
                const double* dg = reinterpret_cast<const double*>(blob + kDiag);
                const double* val = dg + mp;
                const int* dep = reinterpret_cast<const int*>(val + W * mp);
                const int* xidx = dep + W * mp;
                const int* exl = xidx + mp;
                const double* bst = reinterpret_cast<const double*>(blob) - ((h0.x + 4) & ~3) + ((flags >> 5) & 1);
                const double* hb = reinterpret_cast<const double*>(blob + reinterpret_cast<const int*>(blob)[7]) - (R + 1);
                // RPL rows per lane (the layout splits chunks so a warp never has more than
                // 32 * RPL rows), processed together for instruction-level parallelism
                bool act[RPL];
                int tt[RPL], ee[RPL];
                double xx[RPL];
#pragma unroll
                for (int k = 0; k < RPL; ++k) {
                    act[k] = t0 + lane + 32 * k < t1;
                    tt[k] = act[k] ? t0 + lane + 32 * k : t0;
                }
                if ((flags & 9) == 0) {
                    // fast path: every dependency in shared memory, no tail
                    int dd[RPL][W];
                    double vv[RPL][W], xv[RPL][W], dv[RPL], acc[RPL];
                    // row groups past the segment end are skipped (warp-uniform test)
#pragma unroll
                    for (int k = 0; k < RPL; ++k) {
                        if (k > 0 && t0 + 32 * k >= t1) break;
                        dv[k] = dg[tt[k]];
                        acc[k] = bst[tt[k]];
                        ee[k] = exl[tt[k]];
#pragma unroll
                        for (int u = 0; u < W; ++u) {
                            dd[k][u] = dep[u * mp + tt[k]];
                            vv[k][u] = val[u * mp + tt[k]];
                        }
                    }
#pragma unroll
                    for (int k = 0; k < RPL; ++k) {
                        if (k > 0 && t0 + 32 * k >= t1) break;
#pragma unroll
                        for (int u = 0; u < W; ++u) xv[k][u] = (dd[k][u] <= R ? ring : hb)[dd[k][u]];
                    }
                    HEC_STAMP(3, dd[0][0])
                    HEC_STAMP(4, static_cast<int>(xv[0][0]))
#pragma unroll
                    for (int k = 0; k < RPL; ++k) {
                        if (k > 0 && t0 + 32 * k >= t1) {
                            xx[k] = 0.0;
                            ee[k] = -1;
                            continue;
                        }
                        const double y = __drcp_rn(dv[k]);  // off the critical path
#pragma unroll
                        for (int u = 0; u < W; ++u) acc[k] = __dsub_rn(acc[k], __dmul_rn(vv[k][u], xv[k][u]));
                        xx[k] = div_rn(acc[k], dv[k], y);
                    }
                    HEC_STAMP(6, static_cast<int>(xx[0]))
                } else {
                    const uint32_t ring_s = smem_u32(ring), hb_s = smem_u32(hb);
#pragma unroll
                    for (int k = 0; k < RPL; ++k) {
                        const int t = tt[k];
                        const double dv = dg[t];
                        ee[k] = exl[t];
                        const double y = __drcp_rn(dv);
                        double acc = bst[t];
#pragma unroll
                        for (int u = 0; u < W; ++u)
                            acc = __dsub_rn(acc, __dmul_rn(val[u * mp + t], dep_value(dep[u * mp + t], R, ring_s, hb_s, xs)));
                        if (flags & 1) {  // CSR tail beyond the sliced-ELL width, storage order
                            const int* tptr = reinterpret_cast<const int*>(blob + reinterpret_cast<const int*>(blob)[6]);
                            const int mt = (mp + 4) & ~3;  // round_up(mp + 1, 4)
                            const int ntl = tptr[mp];
                            const double* tval = reinterpret_cast<const double*>(tptr + mt);
                            const int* tdep = reinterpret_cast<const int*>(tval + ((ntl + 1) & ~1));
                            for (int e = tptr[t]; e < tptr[t + 1]; ++e)
                                acc = __dsub_rn(acc, __dmul_rn(tval[e], dep_value(tdep[e], R, ring_s, hb_s, xs)));
                        }
                        xx[k] = div_rn(acc, dv, y);
                    }
                }
#pragma unroll
                for (int k = 0; k < RPL; ++k) {
                    // consumers in other CTAs are on the critical path: feed them first
                    if (act[k] && ee[k] >= 0) mail_store(mbox + 2 * static_cast<size_t>(ee[k]), xx[k], ep);
                    if (act[k]) ring[(q0 + tt[k]) & (R - 1)] = xx[k];
                    pend_x[k] = xx[k];
                    pend_xi[k] = act[k] ? xidx[tt[k]] : -1;
                    pend_o[k] = (act[k] && (flags & 2)) ? exl[mp + tt[k]] : -1;
                }
            }
            __syncwarp();
            if (NW > 1) asm volatile("fence.acq_rel.cta;" ::: "memory");  // ring rows -> other warps
            if (lane == 0) {
                if (NW > 1) st_volatile_u32(&prog[w], static_cast<uint32_t>(j + 1));
                mbar_arrive(&bar_empty[s]);
                if (TRACE) tr(j, 10 + 3 * w) = gtimer();
            }
            HEC_STAMP(7, 0)
            // the scattered stores of x leave the critical path: they are issued after
            // the warp published its rows (only the own CTA reads x back, and only rows
            // of chunks <= j-2, whose stores precede a later publication)
#pragma unroll
            for (int k = 0; k < RPL; ++k)
                if (pend_xi[k] >= 0) {
                    xs[pend_xi[k]] = pend_x[k];
                    if (pend_o[k] >= 0) outv[pend_o[k]] = pend_x[k];
                    pend_xi[k] = -1;
                }
        }
    }

#undef HEC_STAMP
    __syncthreads();
    if (tid == 0) {
        __threadfence();
        const uint32_t finished = atomicAdd(&a.counters[1], 1u);
        if (finished == static_cast<uint32_t>(a.ctas) - 1) {
            // last CTA out: re-arm the tickets and advance the mailbox epoch for the
            // next launch on this stream (never 0: 0 marks a mailbox never written)
            a.counters[0] = 0;
            a.counters[1] = 0;
            a.counters[2] = s_epoch == 0xffffffffu ? 1u : s_epoch + 1u;
            __threadfence();
        }
    }
}

__global__ void k_permute_in(const double* __restrict__ b, const int* __restrict__ bidx, double* __restrict__ bp,
                             int n) {
    for (int r = blockIdx.x * blockDim.x + threadIdx.x; r < n; r += gridDim.x * blockDim.x) bp[r] = __ldg(b + bidx[r]);
}

void permute_in(const double* b, const int* bidx, double* bp, int n, cudaStream_t st) {
    if (n <= 0) return;
    int dev = 0, sms = 148;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
    const int blocks = std::min((n + 255) / 256, sms * 8);
    k_permute_in<<<blocks, 256, 0, st>>>(b, bidx, bp, n);
}

// solver layouts: 16 warps x 1 row per lane, or 1 warp x RPL rows per lane
#define HEC_WAVE_INST3(WD, NWW, RP)                                \
    template __global__ void k_wave<WD, NWW, RP, false>(WaveArgs); \
    template __global__ void k_wave<WD, NWW, RP, true>(WaveArgs);
#define HEC_WAVE_INST(WD) HEC_WAVE_INST3(WD, 16, 1) HEC_WAVE_INST3(WD, 1, 2) HEC_WAVE_INST3(WD, 1, 4) \
    HEC_WAVE_INST3(WD, 1, 8)
HEC_WAVE_INST(1) HEC_WAVE_INST(2) HEC_WAVE_INST(3) HEC_WAVE_INST(4) HEC_WAVE_INST(5) HEC_WAVE_INST(6)
HEC_WAVE_INST(7) HEC_WAVE_INST(8) HEC_WAVE_INST(10) HEC_WAVE_INST(13) HEC_WAVE_INST(16)
#undef HEC_WAVE_INST
#undef HEC_WAVE_INST3

void* wave_kernel(int width, int warps, int rpl, bool trace) {
#define HEC_K(WD, NWW, RP) \
    (trace ? reinterpret_cast<void*>(&k_wave<WD, NWW, RP, true>) : reinterpret_cast<void*>(&k_wave<WD, NWW, RP, false>))
#define HEC_PICK(WD)                                                                                  \
    case WD:                                                                                          \
        if (warps > 1) return HEC_K(WD, 16, 1);                                                       \
        return rpl >= 8 ? HEC_K(WD, 1, 8) : rpl >= 4 ? HEC_K(WD, 1, 4) : HEC_K(WD, 1, 2);
    switch (width) {
        HEC_PICK(1) HEC_PICK(2) HEC_PICK(3) HEC_PICK(4) HEC_PICK(5) HEC_PICK(6)
        HEC_PICK(7) HEC_PICK(8) HEC_PICK(10) HEC_PICK(13) HEC_PICK(16)
        default: return nullptr;
    }
#undef HEC_PICK
#undef HEC_K
}

}  // namespace hec::dev
