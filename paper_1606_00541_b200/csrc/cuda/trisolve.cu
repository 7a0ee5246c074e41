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
//  * k_pipeline     persistent, one CTA per SM. CTA c owns a contiguous block of
//                   lower-frame rows; its rows of level k form one chunk. Warp
//                   roles: 0 = producer (cp.async.bulk of the next chunk blobs
//                   into a shared-memory slot ring + cp.async gather of b),
//                   1 = waiter (polls the mailbox words carrying the foreign x
//                   values a chunk needs and stages them in shared memory),
//                   2.. = solvers (own recent x values from a shared-memory
//                   ring; foreign ones from the staged halo). The reference's
//                   level barrier becomes a per-value dataflow handoff: the
//                   producing thread's plain 8-byte store IS the signal (the
//                   empty sentinel is a signalling NaN no arithmetic result can
//                   equal), so no fence or flag sits on the critical path.

#include <cuda_runtime.h>

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
    double acc = a.b[a.bidx[r]];
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

// ------------------------------------------------------------ PIPELINE ----
using plan::ChunkHeader;
constexpr unsigned long long kEmpty = plan::kMailboxEmpty;

// Shared-memory word of dependency code d < 0 (see tri_plan.hpp): the own-x
// ring, its zero slot, or -- beyond the zero slot -- the chunk's staged halo,
// which sits `hoff` doubles further from the ring base.
__device__ __forceinline__ int smem_word(int d, int ring_n, int hoff) {
    const int s = -d - 1;
    return s + (s > ring_n ? hoff : 0);
}

// Any dependency code, including d >= 0 (own rows older than the ring: global x).
__device__ __forceinline__ double dep_value(int d, const double* xs, const double* ring, int ring_n, int hoff) {
    double v = ring[d < 0 ? smem_word(d, ring_n, hoff) : 0];
    if (d >= 0) v = xs[d];
    return v;
}

// acc -= sum over W sliced-ELL slots, all loads issued before the FP chain.
template <int W>
__device__ __forceinline__ double accumulate_fixed(double acc, const int* dep, const double* val, int mp, int t,
                                                   const double* ring, int ring_n, int hoff) {
    double xv[W], vv[W];
#pragma unroll
    for (int u = 0; u < W; ++u) {
        xv[u] = ring[smem_word(dep[u * mp + t], ring_n, hoff)];
        vv[u] = val[u * mp + t];
    }
#pragma unroll
    for (int u = 0; u < W; ++u) acc = sub_prod(acc, vv[u], xv[u]);
    return acc;
}

// Runtime width, any dependency kind (global x allowed); groups of 8 loads.
__device__ __noinline__ double accumulate_generic(double acc, int w, const int* dep, const double* val, int mp, int t,
                                                  const double* xs, const double* ring, int ring_n, int hoff) {
    for (int k0 = 0; k0 < w; k0 += 8) {
        double xv[8], vv[8];
#pragma unroll
        for (int u = 0; u < 8; ++u) {
            const bool on = k0 + u < w;
            const int d = on ? dep[(k0 + u) * mp + t] : -(ring_n + 1);
            vv[u] = on ? val[(k0 + u) * mp + t] : 0.0;
            xv[u] = dep_value(d, xs, ring, ring_n, hoff);
        }
#pragma unroll
        for (int u = 0; u < 8; ++u)
            if (k0 + u < w) acc = sub_prod(acc, vv[u], xv[u]);
    }
    return acc;
}

__device__ __forceinline__ double accumulate(double acc, int w, bool global, const int* dep, const double* val,
                                             int mp, int t, const double* xs, const double* ring, int ring_n,
                                             int hoff) {
    if (!global) {
        switch (w) {
#define HEC_W(N) \
    case N: return accumulate_fixed<N>(acc, dep, val, mp, t, ring, ring_n, hoff);
            case 0: return acc;
            HEC_W(1) HEC_W(2) HEC_W(3) HEC_W(4) HEC_W(5) HEC_W(6) HEC_W(7) HEC_W(8)
            HEC_W(9) HEC_W(10) HEC_W(11) HEC_W(12) HEC_W(13) HEC_W(14) HEC_W(15) HEC_W(16)
#undef HEC_W
            default: break;
        }
    }
    return accumulate_generic(acc, w, dep, val, mp, t, xs, ring, ring_n, hoff);
}

template <int NSOLVE, bool TRACE>
__global__ void __launch_bounds__(kPipelineRoleThreads + NSOLVE, 1) k_pipeline(PipeArgs a) {
    extern __shared__ __align__(128) unsigned char smem[];
    const int NS = a.nslots;
    uint64_t* bar_full = reinterpret_cast<uint64_t*>(smem);
    uint64_t* bar_clear = bar_full + NS;
    uint64_t* bar_empty = bar_clear + NS;
    double* ring = reinterpret_cast<double*>(smem + a.ring_off);
    unsigned char* slots = smem + a.slot_off;
    __shared__ int s_cta;

    const int tid = threadIdx.x;
    const int warp = tid >> 5, lane = tid & 31;
    if (tid == 0) {
        s_cta = static_cast<int>(atomicAdd(&a.counters[0], 1u));
        for (int s = 0; s < NS; ++s) {
            mbar_init(&bar_full[s], 1);
            // 32 producer lanes (b gather, cp.async arrive-on) + the waiter's arrive
            mbar_init(&bar_clear[s], 33);
            mbar_init(&bar_empty[s], 1);
        }
        asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
        ring[a.ring] = 0.0;  // the zero slot that padding entries point at
    }
    __syncthreads();
    const int c = s_cta;
    const int c0 = a.cta_chunk0[c];
    const int nch = a.cta_chunk0[c + 1] - c0;
    // slot = [gathered b : b_bytes][staged halo : halo_bytes][blob]
    auto slot_ptr = [&](int s) { return slots + static_cast<size_t>(s) * a.slot_bytes; };
    const int blob_off = a.b_bytes + a.halo_bytes;
    auto tr = [&](int j, int k) -> unsigned long long& { return a.trace[static_cast<size_t>(c0 + j) * 16 + k]; };

    if (warp == 0) {
        // ---------------- producer: blob prefetch + b gather ----------------
        const int lag = a.lag;
        int2 span_reg = make_int2(0, 0);
        for (int j = 0; j < nch + lag; ++j) {
            if (j < nch) {
                if ((j & 31) == 0) {
                    const int g = j + lane;
                    span_reg = g < nch ? a.spans[c0 + g] : make_int2(0, 0);
                }
                const int off16 = __shfl_sync(0xffffffffu, span_reg.x, j & 31);
                const int bytes = __shfl_sync(0xffffffffu, span_reg.y, j & 31);
                const int s = j % NS, use = j / NS;
                if (use > 0) mbar_wait(&bar_empty[s], (use - 1) & 1);
                if (lane == 0) {
                    if (TRACE) tr(j, 0) = gtimer();
                    mbar_expect_tx(&bar_full[s], static_cast<uint32_t>(bytes));
                    bulk_g2s(slot_ptr(s) + blob_off, a.blobs + static_cast<size_t>(off16) * 16,
                             static_cast<uint32_t>(bytes), &bar_full[s]);
                }
                __syncwarp();
            }
            const int g = j - lag;
            if (g >= 0 && g < nch) {
                const int s = g % NS, use = g / NS;
                mbar_wait(&bar_full[s], use & 1);
                unsigned char* sp = slot_ptr(s);
                const ChunkHeader* h = reinterpret_cast<const ChunkHeader*>(sp + blob_off);
                const int m = h->m;
                const int* bidx = reinterpret_cast<const int*>(sp + blob_off + h->bidx);
                double* bst = reinterpret_cast<double*>(sp);
                if (TRACE && lane == 0) tr(g, 1) = gtimer();
                for (int t = lane; t < m; t += 32) cp_async8(bst + t, a.b + bidx[t]);
                cp_async_arrive(&bar_clear[s]);
            }
        }
    } else if (warp == 1) {
        // ---------------- waiter: poll foreign values, stage them ----------------
        for (int j = 0; j < nch; ++j) {
            const int s = j % NS, use = j / NS;
            mbar_wait(&bar_full[s], use & 1);
            unsigned char* sp = slot_ptr(s);
            const unsigned char* blob = sp + blob_off;
            const int nhalo = reinterpret_cast<const ChunkHeader*>(blob)->nhalo;
            if (TRACE && lane == 0) tr(j, 2) = gtimer();
            const int* hcode = reinterpret_cast<const int*>(blob + plan::kChunkHeaderBytes);
            double* hst = reinterpret_cast<double*>(sp + a.b_bytes);
            for (int t0 = 0; t0 < nhalo; t0 += 128) {
                unsigned long long v[4];
                int code[4];
#pragma unroll
                for (int u = 0; u < 4; ++u) {  // 4 polls in flight per lane
                    const int t = t0 + u * 32 + lane;
                    code[u] = t < nhalo ? hcode[t] : -1;
                    v[u] = code[u] >= 0 ? ld_relaxed_u64(a.mbox + (code[u] >> 1)) : 0ULL;
                }
#pragma unroll
                for (int u = 0; u < 4; ++u) {
                    if (code[u] < 0) continue;
                    unsigned long long* mb = a.mbox + (code[u] >> 1);
                    while (v[u] == kEmpty) v[u] = ld_relaxed_u64(mb);
                    hst[t0 + u * 32 + lane] = __longlong_as_double(static_cast<long long>(v[u]));
                    if (code[u] & 1) st_relaxed_u64(mb, kEmpty);  // last use this solve: re-arm
                }
            }
            __syncwarp();
            if (TRACE && lane == 0) tr(j, 3) = gtimer();
            if (lane == 0) mbar_arrive(&bar_clear[s]);
        }
    } else {
        // ---------------- solvers: one row per thread per pass ----------------
        const int st = tid - kPipelineRoleThreads;
        const int ring_mask = a.ring - 1;
        const int ring_n = a.ring;
        for (int j = 0; j < nch; ++j) {
            const int s = j % NS, use = j / NS;
            mbar_wait(&bar_clear[s], use & 1);
            long long clk0 = 0;
            if (TRACE && st == 0) {
                tr(j, 4) = gtimer();
                clk0 = clock64();
            }
            unsigned char* sp = slot_ptr(s);
            const unsigned char* blob = sp + blob_off;
            const ChunkHeader h = *reinterpret_cast<const ChunkHeader*>(blob);
            const double* bst = reinterpret_cast<const double*>(sp);
            // staged halo, addressed relative to the ring base (both in shared memory)
            const int hoff =
                static_cast<int>((sp + a.b_bytes - reinterpret_cast<unsigned char*>(ring)) / 8) - (ring_n + 1);
            const bool global = (h.flags & 8) != 0;
            if (TRACE && st == 0) tr(j, 8) = clock64() - clk0;
            for (int t = st; t < h.m; t += NSOLVE) {
                double acc = accumulate(bst[t], h.w, global, reinterpret_cast<const int*>(blob + h.dep),
                                        reinterpret_cast<const double*>(blob + h.val), h.mp, t, a.xs, ring, ring_n,
                                        hoff);
                if (h.flags & 1) {
                    const int* tptr = reinterpret_cast<const int*>(blob + h.tptr);
                    const double* tval = reinterpret_cast<const double*>(blob + h.tval);
                    const int* tdep = reinterpret_cast<const int*>(blob + h.tdep);
                    for (int e = tptr[t]; e < tptr[t + 1]; ++e)
                        acc = sub_prod(acc, tval[e], dep_value(tdep[e], a.xs, ring, ring_n, hoff));
                }
                if (TRACE && t == 0) {
                    asm volatile("" ::"d"(acc) : "memory");
                    tr(j, 9) = clock64() - clk0;
                }
                const double x = __ddiv_rn(acc, reinterpret_cast<const double*>(blob + h.diag)[t]);
                if (TRACE && t == 0) {
                    asm volatile("" ::"d"(x) : "memory");
                    tr(j, 10) = clock64() - clk0;
                }
                if (h.flags & 4) {  // feed the consumers' mailboxes first: they are on the critical path
                    const int* mbptr = reinterpret_cast<const int*>(blob + h.mbptr);
                    const int* mbid = reinterpret_cast<const int*>(blob + h.mbid);
                    const unsigned long long xb = static_cast<unsigned long long>(__double_as_longlong(x));
                    for (int k = mbptr[t]; k < mbptr[t + 1]; ++k) st_relaxed_u64(a.mbox + mbid[k], xb);
                }
                ring[(h.q0 + t) & ring_mask] = x;
                a.xs[reinterpret_cast<const int*>(blob + h.xidx)[t]] = x;
                if (h.flags & 2) {
                    const int o = reinterpret_cast<const int*>(blob + h.oidx)[t];
                    if (o >= 0) a.out[o] = x;
                }
            }
            if (TRACE && st == 0) tr(j, 11) = clock64() - clk0;
            named_bar_sync(1, NSOLVE);
            if (TRACE && st == 0) {
                tr(j, 5) = gtimer();
                tr(j, 7) = static_cast<unsigned long long>(clock64() - clk0);
            }
            if (st == 0) mbar_arrive(&bar_empty[s]);
        }
    }

    __syncthreads();
    if (tid == 0) {
        __threadfence();
        const uint32_t finished = atomicAdd(&a.counters[1], 1u);
        if (finished == static_cast<uint32_t>(a.ctas) - 1) {
            // last CTA out: re-arm the tickets for the next launch on this stream
            a.counters[0] = 0;
            a.counters[1] = 0;
            __threadfence();
        }
    }
}

template __global__ void k_pipeline<128, false>(PipeArgs);
template __global__ void k_pipeline<256, false>(PipeArgs);
template __global__ void k_pipeline<128, true>(PipeArgs);
template __global__ void k_pipeline<256, true>(PipeArgs);

void* pipeline_kernel(int nsolve, bool trace) {
    if (trace)
        return nsolve >= 256 ? reinterpret_cast<void*>(&k_pipeline<256, true>)
                             : reinterpret_cast<void*>(&k_pipeline<128, true>);
    return nsolve >= 256 ? reinterpret_cast<void*>(&k_pipeline<256, false>)
                         : reinterpret_cast<void*>(&k_pipeline<128, false>);
}

// Fill a mailbox array with the empty sentinel.
__global__ void k_fill_u64(unsigned long long* p, long long n, unsigned long long v) {
    for (long long i = blockIdx.x * static_cast<long long>(blockDim.x) + threadIdx.x; i < n;
         i += static_cast<long long>(gridDim.x) * blockDim.x)
        p[i] = v;
}

void fill_mailboxes(unsigned long long* p, long long n, cudaStream_t st) {
    if (n <= 0) return;
    k_fill_u64<<<296, 256, 0, st>>>(p, n, kEmpty);
}

}  // namespace hec::dev
