// k_cols: the column-state triangular solve for 7-point grid factors (layout
// and reasoning: tri_plan.hpp, COLUMNS).
//
// One CTA per x-y tile of columns, one lane per column. At level L a lane
// solves row (x, y, z = L - x - y) of its column with the reference's
// arithmetic (src/triangular.cpp:118-126: b, minus value * x for each entry in
// ELL-then-CSR order, then one IEEE division by the diagonal), taking
//   (x, y, z-1)  from its own register (the column's latest value),
//   (x-1, y, z)  from lane-1 by shuffle, or from the left warp's edge buffer,
//                or from the left CTA's mailbox,
//   (x, y-1, z)  from lane-8 by shuffle, or the lower warp's edge buffer, or
//                the lower CTA's mailbox,
// all of them produced at level L-1. The CTA's warps move in lockstep (one
// named barrier per level orders the edge buffers); a producer warp streams
// each level's row data and b (one TMA bulk copy each) through a ring of
// shared-memory slots ahead of the solver warps. Mailbox values are loaded four
// levels ahead and re-polled only if they were not produced yet, so the lag
// behind a neighbouring CTA settles where the prefetch finds them ready.
#include "wave_kernel.cuh"

namespace hec::dev {

namespace {

// The value of row z from a neighbouring CTA's mailbox p (v: loaded a few levels
// ago). If it was not produced yet, this CTA has caught up with its neighbour:
// it then waits until the neighbour is `gap` rows further down the column, so
// that the following levels' early loads find their rows ready again (a lag of
// a few levels per CTA boundary instead of a round trip to L2 on every level).
// Rows of a column are produced in order, but another SM may see them out of
// order: row z itself is re-polled until it is there.
__device__ __noinline__ double mail_late(const unsigned long long* p, int ahead, uint32_t ep, uint64_t deadline,
                                         uint32_t& polls) {
    ulonglong2 w = ld_relaxed_v2(p + 2 * ahead);
    while (!mail_ok(w, ep)) {
        watchdog(polls, deadline);
        w = ld_relaxed_v2(p + 2 * ahead);
    }
    ulonglong2 v = ld_relaxed_v2(p);
    while (!mail_ok(v, ep)) {
        watchdog(polls, deadline);
        v = ld_relaxed_v2(p);
    }
    return mail_value(v);
}
__device__ __forceinline__ double mail_get(ulonglong2 v, const unsigned long long* p, int ahead, uint32_t ep,
                                           uint64_t deadline, uint32_t& polls) {
    if (__builtin_expect(mail_ok(v, ep), 1)) return mail_value(v);
    ++polls;
    return mail_late(p, ahead, ep, deadline, polls);
}

template <int NW, bool UNIT, bool TRACE, bool ZYX>
__global__ void __launch_bounds__(32 * NW, 1) k_cols(ColArgs a) {
    constexpr int SX = 8, SY = 4, NS = 32 * NW, D = 3, GAP = 5;
    extern __shared__ __align__(128) unsigned char smem[];
    uint64_t* full = reinterpret_cast<uint64_t*>(smem);
    double* edge_r = reinterpret_cast<double*>(smem + 256);  // [2][NW][SY]: right column of each warp
    double* edge_t = edge_r + 2 * NW * SY;                   // [2][NW][SX]: top row of each warp
    unsigned char* ring = smem + plan::kColCtrlBytes;
    __shared__ int s_cta;
    __shared__ uint32_t s_epoch;
    __shared__ uint64_t s_ebar[2];  // level parity: every warp's edges of that level written
    const int R = a.ring;
    const int per_level = a.block_bytes + 8 * NS;
    const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
    const uint64_t deadline = static_cast<uint64_t>(clock64()) + a.watchdog_cycles;
    if (tid == 0) {
        s_cta = static_cast<int>(atomicAdd(&a.counters[0], 1u));
        s_epoch = ld_relaxed_u32(&a.counters[2]);
        for (int s = 0; s < R; ++s) mbar_init(&full[s], 1);
        mbar_init(&s_ebar[0], NW);
        mbar_init(&s_ebar[1], NW);
        asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    }
    __syncthreads();
    const int c = s_cta;
    const int4 ci = a.cta[c];  // first level, level count, first slot / NS, first block
    const int lev0 = ci.x, nl = ci.y;
    const long long slot0 = static_cast<long long>(ci.z) * NS;
    // The slot ring: level l's row data and b (one TMA bulk copy each) in slot l % R.
    // Thread 0 fills the first R levels, then refills slot (l-1) % R with level
    // l-1+R at level l: by then every warp has passed level l-1 (the edge barrier
    // of level l-1 completed), so that slot is consumed -- no producer warp.
    auto fill = [&](int l) {
        const int s = l % R;
        unsigned char* dst = ring + s * per_level;
        const double* bs = a.bp_reversed ? a.bp + (a.slots - slot0 - static_cast<long long>(l + 1) * NS)
                                         : a.bp + slot0 + static_cast<long long>(l) * NS;
        mbar_expect_tx(&full[s], static_cast<uint32_t>(per_level));
        bulk_g2s(dst, a.blocks + (static_cast<size_t>(ci.w) + l) * a.block_bytes, static_cast<uint32_t>(a.block_bytes),
                 &full[s]);
        bulk_g2s(dst + a.block_bytes, bs, 8u * NS, &full[s]);
    };
    if (tid == 0)
        for (int l = 0; l < R && l < nl; ++l) fill(l);
    {
        // ------------- solver warps: one column per lane -------------
        const int w = warp;
        const int lx = lane & (SX - 1), ly = lane / SX;
        const int wx = w % a.WX, wy = w / a.WX;
        const int px = c % a.PX, py = c / a.PX;
        const int TX = SX * a.WX, TY = SY * a.WY;
        const int x = px * TX + wx * SX + lx - a.ox, y = py * TY + wy * SY + ly - a.oy;
        const bool col_ok = x >= 0 && x < a.nx && y >= 0 && y < a.ny;
        const int k = w * 32 + lane;
        const int nz = a.nz;
        // the rows' common entry order: position p reads neighbour dir_p (uniform)
        const int d0 = a.order & 3, d1 = (a.order >> 2) & 3, d2 = (a.order >> 4) & 3;
        const uint32_t ep = s_epoch;
        // where the left / lower neighbour's latest value comes from when it is not a
        // shuffle away: the neighbouring warp's edge buffer, or a mailbox of the
        // neighbouring CTA (right edges first, TY * nz per CTA, then top edges, TX * nz)
        const bool lx0 = lx == 0, ly0 = ly == 0;
        const bool mb_left = col_ok && lx0 && wx == 0 && px > 0;
        const bool mb_down = col_ok && ly0 && wy == 0 && py > 0;
        const bool pub_right = col_ok && lx == SX - 1 && wx == a.WX - 1 && px < a.PX - 1;
        const bool pub_top = col_ok && ly == SY - 1 && wy == a.WY - 1 && py < a.PY - 1;
        const long long yl = wy * SY + ly, xl = wx * SX + lx;
        const int zc = lev0 - x - y;  // z of this column's row at the CTA's level 0
        // mailbox cursors at z = zc (advanced by one row per level)
        const unsigned long long* mbl =
            a.mbox + 2 * (mb_left ? (static_cast<long long>(c - 1) * TY + yl) * nz + zc : 0);
        const unsigned long long* mbd =
            a.mbox + 2 * (mb_down ? a.mbox_top0 + (static_cast<long long>(c - a.PX) * TX + xl) * nz + zc : 0);
        unsigned long long* mpr = a.mbox + 2 * (pub_right ? (static_cast<long long>(c) * TY + yl) * nz + zc : 0);
        unsigned long long* mpt =
            a.mbox + 2 * (pub_top ? a.mbox_top0 + (static_cast<long long>(c) * TX + xl) * nz + zc : 0);
        // edge buffers: this lane reads (parity of level l-1) and writes (parity of l)
        const double* er_rd = edge_r + ((wx > 0 ? w - 1 : w) * SY + ly);
        const double* et_rd = edge_t + ((wy > 0 ? w - a.WX : w) * SX + lx);
        const bool wr_r = NW > 1 && lx == SX - 1, wr_t = NW > 1 && ly == SY - 1;
        double* const er_wr = edge_r + (w * SY + ly);
        double* const et_wr = edge_t + (w * SX + lx);
        ulonglong2 ql[D], qd[D];
#pragma unroll
        for (int j = 0; j < D; ++j) {
            const bool in = static_cast<unsigned>(zc + j) < static_cast<unsigned>(nz);
            ql[j] = (mb_left && in) ? ld_relaxed_v2(mbl + 2 * j) : make_ulonglong2(0, 0);
            qd[j] = (mb_down && in) ? ld_relaxed_v2(mbd + 2 * j) : make_ulonglong2(0, 0);
        }
        // row data of the next level, read from the ring before this level's barrier
        double v[3] = {0.0, 0.0, 0.0}, dd = 1.0, rr = 1.0, bb = 0.0;
        uint32_t msk = 0;
        int rs = 0;
        uint32_t rph = 0;
        auto load_level = [&]() {
            mbar_wait(&full[rs], rph);
            const unsigned char* base = ring + rs * per_level;
            const double* f = reinterpret_cast<const double*>(base);
            v[0] = f[k];
            v[1] = f[NS + k];
            v[2] = f[2 * NS + k];
            if (!UNIT) {
                dd = f[3 * NS + k];
                rr = f[4 * NS + k];
            }
            msk = base[(UNIT ? 24 : 40) * NS + k];
            bb = reinterpret_cast<const double*>(base + a.block_bytes)[a.bp_reversed ? NS - 1 - k : k];
            // unit diagonal: the reference's final division by 1.0 only quiets a
            // signalling NaN; applied to b instead, it leaves the chain (exact
            // otherwise: (b*1 - t...) == (b - t...)/1 bit for bit)
            if (UNIT) bb = __dmul_rn(bb, 1.0);
        };
        if (nl > 0) load_level();
        double last = 0.0;  // the column's latest x (row z-1 at level L)
        double* xw = a.xw + slot0 + k;
        int z = zc;
        for (int l0 = 0; l0 < nl; l0 += D) {
#pragma unroll
            for (int j = 0; j < D; ++j) {
                const int l = l0 + j;
                if (l >= nl) break;
                const bool act = col_ok && static_cast<unsigned>(z) < static_cast<unsigned>(nz);
                const int pr = (l & 1) ? 0 : NW;  // parity offset of level l-1 (SY / SX doubles per warp)
                uint32_t pl = 0, pd = 0;
                unsigned long long* tr = TRACE ? a.trace + 8 * (static_cast<size_t>(ci.w) + l) : nullptr;
                long long c0 = 0;
                if (TRACE && k == 0) {
                    tr[3] = gtimer();
                    c0 = clock64();
                }
#define HEC_CSTAMP(K_, DEP)                                                                   \
    if (TRACE && k == 0) {                                                                     \
        asm volatile("" ::"d"(DEP) : "memory");                                               \
        tr[4 + (K_)] = static_cast<unsigned long long>(clock64() - c0);                         \
    }
                // ---- critical section: level l-1's values in, this level's x out to the neighbours
                if (NW > 1 && l > 0) mbar_wait(&s_ebar[(l - 1) & 1], ((l - 1) >> 1) & 1);  // edges of level l-1
                const double sl = __shfl_up_sync(0xffffffffu, last, 1);
                const double sd = __shfl_up_sync(0xffffffffu, last, SX);
                const double el = er_rd[pr * SY], ed = et_rd[pr * SX];
                double left = lx0 ? el : sl, down = ly0 ? ed : sd;
                if (mb_left && act) left = mail_get(ql[j], mbl, min(GAP, nz - 1 - z), ep, deadline, pl);
                if (mb_down && act) down = mail_get(qd[j], mbd, min(GAP, nz - 1 - z), ep, deadline, pd);
                HEC_CSTAMP(0, left + down)
                // b - v0*x0 - v1*x1 - v2*x2 in the reference's order; an absent entry has
                // value 0 and operand 0.0, an exact no-op like the reference's skip. ZYX: the
                // order of every natural-order 7-point factor, (z-1, y-1, x-1)
                double o0, o1, o2;
                if (ZYX) {
                    o0 = (msk & 1u) ? last : 0.0;
                    o1 = (msk & 2u) ? down : 0.0;
                    o2 = (msk & 4u) ? left : 0.0;
                } else {
                    auto nb = [&](int d) { return d == 0 ? left : (d == 1 ? down : last); };
                    o0 = (msk & 1u) ? nb(d0) : 0.0;
                    o1 = (msk & 2u) ? nb(d1) : 0.0;
                    o2 = (msk & 4u) ? nb(d2) : 0.0;
                }
                double acc = __dsub_rn(bb, __dmul_rn(v[0], o0));
                acc = __dsub_rn(acc, __dmul_rn(v[1], o1));
                acc = __dsub_rn(acc, __dmul_rn(v[2], o2));
                double xn;
                if (UNIT) {
                    xn = acc;  // b was multiplied by 1.0 (load_level)
                } else {
                    const double ad = fabs(dd);
                    bool ok;
                    xn = markstein_dok(acc, dd, rr, (ad > 0x1p-449) & (ad < 0x1p449), ok);
                    if (__builtin_expect(!ok, 0)) xn = div_slow(acc, dd);
                }
                if (act) last = xn;
                if (wr_r) er_wr[(NW - pr) * SY] = last;
                if (wr_t) et_wr[(NW - pr) * SX] = last;
                __syncwarp();
                if (NW > 1 && lane == 0) mbar_arrive(&s_ebar[l & 1]);  // release: this warp's edges of level l
                HEC_CSTAMP(1, xn)
                // ---- off the chain: other CTAs, the output, the slot ring, the next level's data
                if (act) {
                    if (pub_right) mail_store(mpr, xn, ep);
                    if (pub_top) mail_store(mpt, xn, ep);
                }
                if (k == 0 && l >= 1 && l - 1 + R < nl) fill(l - 1 + R);  // slot of level l-1: consumed
                if (act) *xw = xn;
                {
                    const bool in = static_cast<unsigned>(z + D) < static_cast<unsigned>(nz);
                    if (mb_left && in) ql[j] = ld_relaxed_v2(mbl + 2 * D);
                    if (mb_down && in) qd[j] = ld_relaxed_v2(mbd + 2 * D);
                }
                HEC_CSTAMP(2, 0.0)
                if (++rs == R) rs = 0, rph ^= 1u;
                if (l + 1 < nl) load_level();
                HEC_CSTAMP(3, bb + v[0])
                if (TRACE && k == 0) {
                    tr[2] = gtimer();
                    tr[0] = gtimer();
                    tr[1] = pl | static_cast<unsigned long long>(pd) << 32;
                }
#undef HEC_CSTAMP
                ++z;
                xw += NS;
                mbl += 2;
                mbd += 2;
                mpr += 2;
                mpt += 2;
            }
        }
    }

    __syncthreads();
    if (tid == 0) {
        __threadfence();
        const uint32_t finished = atomicAdd(&a.counters[1], 1u);
        if (finished == static_cast<uint32_t>(a.ctas) - 1) {
            a.counters[0] = 0;
            a.counters[1] = 0;
            a.counters[2] = s_epoch == 0xffffffffu ? 1u : s_epoch + 1u;
            __threadfence();
        }
    }
}

template <int NW, bool ZYX>
void* pick(bool unit, bool trace) {
    if (trace)
        return unit ? reinterpret_cast<void*>(&k_cols<NW, true, true, ZYX>)
                    : reinterpret_cast<void*>(&k_cols<NW, false, true, ZYX>);
    return unit ? reinterpret_cast<void*>(&k_cols<NW, true, false, ZYX>)
                : reinterpret_cast<void*>(&k_cols<NW, false, false, ZYX>);
}
template <bool ZYX>
void* pick_nw(int warps, bool unit, bool trace) {
    switch (warps) {
        case 1: return pick<1, ZYX>(unit, trace);
        case 2: return pick<2, ZYX>(unit, trace);
        case 4: return pick<4, ZYX>(unit, trace);
        case 8: return pick<8, ZYX>(unit, trace);
        case 16: return pick<16, ZYX>(unit, trace);
        default: return nullptr;
    }
}

}  // namespace

void* cols_kernel(int warps, bool unit, bool trace, int order) {
    return order == kColOrderZYX ? pick_nw<true>(warps, unit, trace) : pick_nw<false>(warps, unit, trace);
}

}  // namespace hec::dev
