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
//                   1 = waiter (acquire-polls the progress counters of the
//                   CTAs a chunk depends on), 2 = publisher (release-stores this
//                   CTA's progress), 3.. = solvers. Own recent x values live in
//                   a shared-memory ring; older / foreign ones come from L2.
//                   Level barriers become point-to-point CTA progress waits.

#include <cuda_runtime.h>

#include <cstdint>

#include "tri_kernels.cuh"

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
__device__ __forceinline__ uint32_t ld_acquire(const uint32_t* p) {
    uint32_t v;
    asm volatile("ld.acquire.gpu.global.u32 %0, [%1];" : "=r"(v) : "l"(p) : "memory");
    return v;
}
__device__ __forceinline__ void st_release(uint32_t* p, uint32_t v) {
    asm volatile("st.release.gpu.global.u32 [%0], %1;" ::"l"(p), "r"(v) : "memory");
}
__device__ __forceinline__ void named_bar_sync(int id, int count) {
    asm volatile("bar.sync %0, %1;" ::"r"(id), "r"(count) : "memory");
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
struct ChunkHeader {
    int m, w, q0, flags;
    int nwait, ntail, pad0, pad1;
};

__device__ __forceinline__ int rup(int v, int m) { return (v + m - 1) / m * m; }

struct Sections {
    int diag, val, dep, bidx, xidx, oidx, tptr, tval, tdep;
};
__device__ __forceinline__ Sections sections(const ChunkHeader& h) {
    Sections s;
    const int mp = rup(h.m, 4);
    int at = 32 + rup(8 * h.nwait, 16);
    s.diag = at; at += 8 * mp;
    s.val = at;  at += 8 * mp * h.w;
    s.dep = at;  at += 4 * mp * h.w;
    s.bidx = at; at += 4 * mp;
    s.xidx = at; at += 4 * mp;
    s.oidx = at; if (h.flags & 2) at += 4 * mp;
    s.tptr = at; if (h.flags & 1) at += 4 * rup(mp + 1, 4);
    s.tval = at; if (h.flags & 1) at += 8 * rup(h.ntail, 2);
    s.tdep = at;
    return s;
}

template <int NSOLVE>
__global__ void __launch_bounds__(96 + NSOLVE, 1) k_pipeline(PipeArgs a) {
    extern __shared__ __align__(128) unsigned char smem[];
    const int NS = a.nslots;
    uint64_t* bar_full = reinterpret_cast<uint64_t*>(smem);
    uint64_t* bar_ready = bar_full + NS;
    uint64_t* bar_clear = bar_ready + NS;
    uint64_t* bar_done = bar_clear + NS;
    uint64_t* bar_empty = bar_done + NS;
    double* ring = reinterpret_cast<double*>(smem + a.ring_off);
    unsigned char* slots = smem + a.slot_off;
    __shared__ int s_cta;

    const int tid = threadIdx.x;
    const int warp = tid >> 5, lane = tid & 31;
    if (tid == 0) {
        s_cta = static_cast<int>(atomicAdd(&a.counters[0], 1u));
        for (int s = 0; s < NS; ++s) {
            mbar_init(&bar_full[s], 1);
            mbar_init(&bar_ready[s], 32);
            mbar_init(&bar_clear[s], 1);
            mbar_init(&bar_done[s], 1);
            mbar_init(&bar_empty[s], 1);
        }
        asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
        ring[a.ring] = 0.0;  // the zero slot that padding entries point at
    }
    __syncthreads();
    const int c = s_cta;
    const int c0 = a.cta_chunk0[c];
    const int nch = a.cta_chunk0[c + 1] - c0;
    auto slot_ptr = [&](int s) { return slots + static_cast<size_t>(s) * a.slot_bytes; };
    // slot = [gathered b : a.b_bytes][blob]

    if (warp == 0) {
        // ---------------- producer ----------------
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
                    mbar_expect_tx(&bar_full[s], static_cast<uint32_t>(bytes));
                    bulk_g2s(slot_ptr(s) + a.b_bytes, a.blobs + static_cast<size_t>(off16) * 16,
                             static_cast<uint32_t>(bytes), &bar_full[s]);
                }
                __syncwarp();
            }
            const int g = j - lag;
            if (g >= 0 && g < nch) {
                const int s = g % NS, use = g / NS;
                mbar_wait(&bar_full[s], use & 1);
                unsigned char* sp = slot_ptr(s);
                const ChunkHeader h = *reinterpret_cast<const ChunkHeader*>(sp + a.b_bytes);
                const Sections sec = sections(h);
                const int* bidx = reinterpret_cast<const int*>(sp + a.b_bytes + sec.bidx);
                double* bst = reinterpret_cast<double*>(sp);
                for (int t = lane; t < h.m; t += 32) cp_async8(bst + t, a.b + bidx[t]);
                cp_async_arrive(&bar_ready[s]);
            }
        }
    } else if (warp == 1) {
        // ---------------- waiter ----------------
        for (int j = 0; j < nch; ++j) {
            const int s = j % NS, use = j / NS;
            mbar_wait(&bar_full[s], use & 1);
            mbar_wait(&bar_ready[s], use & 1);
            const unsigned char* blob = slot_ptr(s) + a.b_bytes;
            const ChunkHeader h = *reinterpret_cast<const ChunkHeader*>(blob);
            const int2* waits = reinterpret_cast<const int2*>(blob + 32);
            for (int t = lane; t < h.nwait; t += 32) {
                const int2 wv = waits[t];
                const uint32_t* pc = a.progress + wv.x;
                while (ld_acquire(pc) < static_cast<uint32_t>(wv.y)) {
                }
            }
            __syncwarp();
            if (lane == 0) mbar_arrive(&bar_clear[s]);
        }
    } else if (warp == 2) {
        // ---------------- publisher ----------------
        if (lane == 0) {
            for (int j = 0; j < nch; ++j) {
                const int s = j % NS, use = j / NS;
                mbar_wait(&bar_done[s], use & 1);
                const ChunkHeader* h = reinterpret_cast<const ChunkHeader*>(slot_ptr(s) + a.b_bytes);
                const uint32_t q_end = static_cast<uint32_t>(h->q0 + h->m);
                st_release(a.progress + c, q_end);
                mbar_arrive(&bar_empty[s]);
            }
        }
    } else {
        // ---------------- solvers ----------------
        const int st = tid - 96;
        const int ring_mask = a.ring - 1;
        for (int j = 0; j < nch; ++j) {
            const int s = j % NS, use = j / NS;
            mbar_wait(&bar_clear[s], use & 1);
            unsigned char* sp = slot_ptr(s);
            const unsigned char* blob = sp + a.b_bytes;
            const ChunkHeader h = *reinterpret_cast<const ChunkHeader*>(blob);
            const Sections sec = sections(h);
            const int mp = rup(h.m, 4);
            const double* bst = reinterpret_cast<const double*>(sp);
            const double* diag = reinterpret_cast<const double*>(blob + sec.diag);
            const double* val = reinterpret_cast<const double*>(blob + sec.val);
            const int* dep = reinterpret_cast<const int*>(blob + sec.dep);
            const int* xidx = reinterpret_cast<const int*>(blob + sec.xidx);
            for (int t = st; t < h.m; t += NSOLVE) {
                double acc = bst[t];
                for (int k = 0; k < h.w; ++k) {
                    const int d = dep[k * mp + t];
                    const double xv = d >= 0 ? a.xs[d] : ring[-d - 1];
                    acc = sub_prod(acc, val[k * mp + t], xv);
                }
                if (h.flags & 1) {
                    const int* tptr = reinterpret_cast<const int*>(blob + sec.tptr);
                    const double* tval = reinterpret_cast<const double*>(blob + sec.tval);
                    const int* tdep = reinterpret_cast<const int*>(blob + sec.tdep);
                    for (int e = tptr[t]; e < tptr[t + 1]; ++e) {
                        const int d = tdep[e];
                        const double xv = d >= 0 ? a.xs[d] : ring[-d - 1];
                        acc = sub_prod(acc, tval[e], xv);
                    }
                }
                const double x = __ddiv_rn(acc, diag[t]);
                ring[(h.q0 + t) & ring_mask] = x;
                a.xs[xidx[t]] = x;
                if (h.flags & 2) {
                    const int o = reinterpret_cast<const int*>(blob + sec.oidx)[t];
                    if (o >= 0) a.out[o] = x;
                }
            }
            named_bar_sync(1, NSOLVE);
            if (st == 0) mbar_arrive(&bar_done[s]);
        }
    }

    __syncthreads();
    if (tid == 0) {
        __threadfence();
        const uint32_t finished = atomicAdd(&a.counters[1], 1u);
        if (finished == static_cast<uint32_t>(a.ctas) - 1) {
            // last CTA out: re-arm the workspace for the next launch on this stream
            for (int k = 0; k < a.ctas; ++k) a.progress[k] = 0;
            a.counters[0] = 0;
            a.counters[1] = 0;
            __threadfence();
        }
    }
}

template __global__ void k_pipeline<128>(PipeArgs);
template __global__ void k_pipeline<256>(PipeArgs);

void* pipeline_kernel(int nsolve) {
    return nsolve >= 256 ? reinterpret_cast<void*>(&k_pipeline<256>) : reinterpret_cast<void*>(&k_pipeline<128>);
}

}  // namespace hec::dev
