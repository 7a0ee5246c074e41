// k_cols: the column-state triangular solve for 7-point grid factors (layout
// and reasoning: tri_plan.hpp, COLUMNS).
//
// One CTA per x-y tile of columns, four columns per lane. At level L a lane
// solves row (x, y, z = L - x - y) of each of its columns with the reference's
// arithmetic (src/triangular.cpp:118-126: b, minus value * x for each entry in
// ELL-then-CSR order, then one IEEE division by the diagonal), taking
//   (x, y, z-1)  from its own register (the column's latest value),
//   (x, y-1, z)  from its own register (the lane's previous column) or, for its
//                first column, from lane-8 by shuffle, the lower warp's edge
//                ring or the lower CTA's mailbox,
//   (x-1, y, z)  from lane-1 by shuffle, the left warp's edge ring or the left
//                CTA's mailbox,
// all of them produced at level L-1. Warps run free: a warp starts level L
// once its left and lower neighbour warps have published level L-1 (progress
// counters in shared memory). A producer warp streams each level's row data
// and b (one TMA bulk copy each) through a ring of shared-memory slots.
// Mailbox values are loaded a few levels ahead; when one was not produced yet
// the CTA waits until its neighbour is several rows further, so the lag behind
// a neighbouring CTA settles where those early loads find their rows ready.
#include "wave_kernel.cuh"

namespace hec::dev {

namespace {

constexpr int kEdge = plan::kColEdgeLevels;  // levels in the warp edge rings (> slot ring depth + 1)

// Warp edge rings in shared memory carry each value as two 8-byte words
// {lo32 | tag << 32, hi32 | tag << 32} (tag = level + 1): every word is written
// atomically, so a reader polls until both words carry the level it needs -- no
// flag, hence no memory fence in the level loop (a release would wait for the
// warp's global loads and stores in flight). Writers are never more than the
// slot ring's depth ahead of their readers, so a ring of kEdge levels suffices.
__device__ __forceinline__ void edge_put(ulonglong2* e, double x, uint32_t tag) {
    const unsigned long long bits = static_cast<unsigned long long>(__double_as_longlong(x));
    const unsigned long long t = static_cast<unsigned long long>(tag) << 32;
    asm volatile("st.volatile.shared.v2.u64 [%0], {%1, %2};" ::"r"(smem_u32(e)), "l"((bits & 0xffffffffULL) | t),
                 "l"((bits >> 32) | t)
                 : "memory");
}
__device__ __forceinline__ ulonglong2 lds_v2(const ulonglong2* e) {
    ulonglong2 v;
    asm volatile("ld.volatile.shared.v2.u64 {%0, %1}, [%2];" : "=l"(v.x), "=l"(v.y) : "r"(smem_u32(e)) : "memory");
    return v;
}
__device__ __forceinline__ bool tag_ok(ulonglong2 v, uint32_t tag) { return mail_ok(v, tag); }
__device__ __noinline__ ulonglong2 edge_wait(const ulonglong2* e, uint32_t tag) {
    ulonglong2 v;
    do {
        v = lds_v2(e);
    } while (!mail_ok(v, tag));
    return v;
}
// A neighbouring CTA's mailbox p that was not produced yet when it was loaded
// early: this CTA has caught up with its neighbour, so it waits until the
// neighbour is `ahead` rows further down the column (later early loads then
// find their rows ready), then re-polls row z itself (rows of a column are
// produced in order but may be seen out of order). Returns the mailbox words.
__device__ __noinline__ ulonglong2 mail_late2(const unsigned long long* p, int ahead, uint32_t ep, uint64_t deadline,
                                              uint32_t& polls) {
    ++polls;
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
    return v;
}
__device__ __forceinline__ void mbar_arrive_relaxed(uint64_t* bar) {
    asm volatile("mbarrier.arrive.relaxed.cta.shared::cta.b64 _, [%0];" ::"r"(smem_u32(bar)) : "memory");
}

template <int NW, int kRpl, bool UNIT, bool TRACE, bool ZYX>
__global__ void __launch_bounds__(32 * NW + 32, 1) k_cols(ColArgs a) {
    constexpr int SX = 8, SY = 4 * kRpl, NS = 32 * kRpl * NW, D = 3, GAP = 5;
    extern __shared__ __align__(128) unsigned char smem[];
    uint64_t* full = reinterpret_cast<uint64_t*>(smem);
    uint64_t* empty = full + 16;
    ulonglong2* edge_r = reinterpret_cast<ulonglong2*>(smem + 256);  // [kEdge][64]: right column of each warp (w * SY + y)
    ulonglong2* edge_t = edge_r + kEdge * 64;                          // [kEdge][128]: top row of each warp (w * 8 + x)
    unsigned char* ring = smem + plan::kColCtrlBytes;
    __shared__ int s_cta;
    __shared__ uint32_t s_epoch;
    const int R = a.ring;
    const int per_level = a.block_bytes + 8 * NS;
    const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
    const uint64_t deadline = static_cast<uint64_t>(clock64()) + a.watchdog_cycles;
    if (tid == 0) {
        s_cta = static_cast<int>(atomicAdd(&a.counters[0], 1u));
        s_epoch = ld_relaxed_u32(&a.counters[2]);
        for (int s = 0; s < R; ++s) {
            mbar_init(&full[s], 1);
            mbar_init(&empty[s], NW);
        }
        asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    }
    for (int i = tid; i < kEdge * 192; i += blockDim.x) edge_r[i] = make_ulonglong2(0, 0);  // tag 0: empty
    __syncthreads();
    const int c = s_cta;
    const int4 ci = a.cta[c];  // first level, level count, first slot / NS, first block
    const int lev0 = ci.x, nl = ci.y;
    const long long slot0 = static_cast<long long>(ci.z) * NS;

    if (warp == NW) {
        // ------------- producer: level blocks and b through the slot ring -------------
        if (lane == 0) {
            const unsigned char* src = a.blocks + static_cast<size_t>(ci.w) * a.block_bytes;
            const double* bs = a.bp_reversed ? a.bp + (a.slots - slot0 - NS) : a.bp + slot0;
            const long long bstep = a.bp_reversed ? -NS : NS;
            for (int l = 0, s = 0, ph = 0; l < nl; ++l) {
                if (l >= R) mbar_wait(&empty[s], ph ^ 1);
                unsigned char* dst = ring + s * per_level;
                mbar_expect_tx(&full[s], static_cast<uint32_t>(per_level));
                bulk_g2s(dst, src, static_cast<uint32_t>(a.block_bytes), &full[s]);
                bulk_g2s(dst + a.block_bytes, bs, 8u * NS, &full[s]);
                src += a.block_bytes;
                bs += bstep;
                if (++s == R) s = 0, ph ^= 1;
            }
        }
    } else {
        // ------------- solver warps: four columns per lane -------------
        const int w = warp;
        const int lx = lane & (SX - 1), lq = lane >> 3;
        const int wx = w % a.WX, wy = w / a.WX;
        const int px = c % a.PX, py = c / a.PX;
        const int TX = SX * a.WX, TY = SY * a.WY;
        const int x = px * TX + wx * SX + lx - a.ox;
        const int y0 = py * TY + wy * SY + kRpl * lq - a.oy;  // the lane's columns: y0 .. y0+kRpl-1
        const bool x_ok = x >= 0 && x < a.nx;
        bool col_ok[kRpl];
#pragma unroll
        for (int r = 0; r < kRpl; ++r) col_ok[r] = x_ok && y0 + r >= 0 && y0 + r < a.ny;
        const int kb = (w * 32 + lane) * kRpl;  // first slot of the lane in a level
        const int nz = a.nz;
        const uint32_t ep = s_epoch;
        const int d0 = a.order & 3, d1 = (a.order >> 2) & 3, d2 = (a.order >> 4) & 3;
        // neighbours outside the warp: left (lx == 0) and lower (lq == 0, first column)
        const bool lx0 = lx == 0, lq0 = lq == 0;
        const bool w_left = wx > 0, w_down = wy > 0;  // a neighbour warp in this CTA
        const bool mb_left = lx0 && !w_left && px > 0 && x_ok;
        const bool mb_down = lq0 && !w_down && py > 0 && col_ok[0];
        const bool pub_right = lx == SX - 1 && wx == a.WX - 1 && px < a.PX - 1 && x_ok;
        const bool pub_top = lq == 3 && wy == a.WY - 1 && py < a.PY - 1 && col_ok[kRpl - 1];
        const long long yl = wy * SY + kRpl * lq, xl = wx * SX + lx;  // in-tile offsets
        const int zc = lev0 - x - y0;  // z of column 0's row at the CTA's level 0 (column r: zc - r)
        // mailbox cursors at column 0's z = zc (one row further per level); column r's
        // mailbox of the same level sits r rows up in y and r rows back in z
        const long long nzl = nz;
        const unsigned long long* mbl =
            a.mbox + 2 * (mb_left ? ((c - 1) * static_cast<long long>(TY) + yl) * nzl + zc : 0);
        const unsigned long long* mbd =
            a.mbox + 2 * (mb_down ? a.mbox_top0 + ((c - a.PX) * static_cast<long long>(TX) + xl) * nzl + zc : 0);
        unsigned long long* mpr = a.mbox + 2 * (pub_right ? (c * static_cast<long long>(TY) + yl) * nzl + zc : 0);
        unsigned long long* mpt =
            a.mbox + 2 * (pub_top ? a.mbox_top0 + (c * static_cast<long long>(TX) + xl) * nzl + zc - (kRpl - 1) : 0);
        const long long rstride = 2 * (nzl - 1);  // column r+1's mailbox of the same level, in words
        ulonglong2 ql[D][kRpl], qd[D];
#pragma unroll
        for (int j = 0; j < D; ++j) {
#pragma unroll
            for (int r = 0; r < kRpl; ++r) {
                const bool in = static_cast<unsigned>(zc + j - r) < static_cast<unsigned>(nz);
                ql[j][r] = (mb_left && col_ok[r] && in) ? ld_relaxed_v2(mbl + 2 * j + r * rstride)
                                                         : make_ulonglong2(0, 0);
            }
            const bool in = static_cast<unsigned>(zc + j) < static_cast<unsigned>(nz);
            qd[j] = (mb_down && in) ? ld_relaxed_v2(mbd + 2 * j) : make_ulonglong2(0, 0);
        }
        double last[kRpl];  // the columns' latest x
#pragma unroll
        for (int r = 0; r < kRpl; ++r) last[r] = 0.0;
        double* xw = a.xw + slot0 + kb;
        int z = zc, rs = 0;
        uint32_t rph = 0;
        for (int l0 = 0; l0 < nl; l0 += D) {
#pragma unroll
            for (int j = 0; j < D; ++j) {
                const int l = l0 + j;
                if (l >= nl) break;
                uint32_t pl = 0, pd = 0;
                unsigned long long* tr = TRACE ? a.trace + 8 * (static_cast<size_t>(ci.w) + l) : nullptr;
                long long c0 = 0;
                if (TRACE && lane == 0 && w == 0) {
                    tr[3] = gtimer();
                    c0 = clock64();
                }
#define HEC_CSTAMP(K_, DEP)                                                                   \
    if (TRACE && lane == 0 && w == 0) {                                                        \
        asm volatile("" ::"d"(DEP) : "memory");                                               \
        tr[4 + (K_)] = static_cast<unsigned long long>(clock64() - c0);                         \
    }
                // ---- this level's row data (the producer is levels ahead)
                mbar_wait(&full[rs], rph);
                HEC_CSTAMP(0, 0.0)
                const unsigned char* base = ring + rs * per_level;
                const double* f = reinterpret_cast<const double*>(base);
                double v[3][kRpl], dd[kRpl], rr[kRpl], bb[kRpl];
                auto ld4 = [&](const double* src, double* dst) {  // kRpl consecutive doubles
#pragma unroll
                    for (int h = 0; h < kRpl; h += 2) {
                        const double2 p = *reinterpret_cast<const double2*>(src + h);
                        dst[h] = p.x;
                        if (h + 1 < kRpl) dst[h + 1] = p.y;
                    }
                };
                static_assert(kRpl == 1 || kRpl % 2 == 0, "columns per lane: 1, 2 or 4");
#pragma unroll
                for (int u = 0; u < 3; ++u) {
                    if (kRpl == 1) v[u][0] = f[u * NS + kb];
                    else ld4(f + u * NS + kb, v[u]);
                }
                if (!UNIT) {
                    if (kRpl == 1) {
                        dd[0] = f[3 * NS + kb];
                        rr[0] = f[4 * NS + kb];
                    } else {
                        ld4(f + 3 * NS + kb, dd);
                        ld4(f + 4 * NS + kb, rr);
                    }
                }
                uint32_t msk4;
                {
                    const unsigned char* mb = base + (UNIT ? 24 : 40) * NS + kb;
                    if (kRpl == 4) msk4 = *reinterpret_cast<const uint32_t*>(mb);
                    else if (kRpl == 2) msk4 = *reinterpret_cast<const uint16_t*>(mb);
                    else msk4 = *mb;
                }
                {
                    const double* bsm = reinterpret_cast<const double*>(base + a.block_bytes);
                    if (a.bp_reversed) {  // slot s reads bp[S-1-s]: this lane's slots in reverse
                        double t[kRpl];
                        if (kRpl == 1) t[0] = bsm[NS - 1 - kb];
                        else ld4(bsm + NS - kRpl - kb, t);
#pragma unroll
                        for (int r = 0; r < kRpl; ++r) bb[r] = t[kRpl - 1 - r];
                    } else {
                        if (kRpl == 1) bb[0] = bsm[kb];
                        else ld4(bsm + kb, bb);
                    }
                }
                HEC_CSTAMP(1, v[2][kRpl - 1] + bb[kRpl - 1])
                // ---- neighbours' values of level l-1. Common path without branches: every lane
                // reads its edge-ring candidates, one vote decides whether anyone must wait.
                const int er = (l + kEdge - 1) % kEdge;  // edge ring slot of level l-1
                double left[kRpl];
#pragma unroll
                for (int r = 0; r < kRpl; ++r) left[r] = __shfl_up_sync(0xffffffffu, last[r], 1);
                double down0 = __shfl_up_sync(0xffffffffu, last[kRpl - 1], SX);
                const ulonglong2* el = edge_r + (er * 64 + (w_left ? w - 1 : w) * SY + kRpl * lq);
                const ulonglong2* ed = edge_t + (er * 128 + (w_down ? w - a.WX : w) * 8 + lx);
                const uint32_t tg = static_cast<uint32_t>(l);
                ulonglong2 ev[kRpl], dv;
#pragma unroll
                for (int r = 0; r < kRpl; ++r) ev[r] = lds_v2(el + r);
                dv = lds_v2(ed);
                const bool need_l = lx0 && w_left, need_d = lq0 && w_down;
                bool need_m[kRpl];
                bool stale = false;
#pragma unroll
                for (int r = 0; r < kRpl; ++r) {
                    need_m[r] = mb_left && col_ok[r] && static_cast<unsigned>(z - r) < static_cast<unsigned>(nz);
                    stale |= (need_l && !tag_ok(ev[r], tg)) | (need_m[r] && !mail_ok(ql[j][r], ep));
                }
                const bool need_md = mb_down && static_cast<unsigned>(z) < static_cast<unsigned>(nz);
                stale |= (need_d && !tag_ok(dv, tg)) | (need_md && !mail_ok(qd[j], ep));
                if (__any_sync(0xffffffffu, stale)) {  // someone is early: wait for what is missing
#pragma unroll
                    for (int r = 0; r < kRpl; ++r) {
                        if (need_l && !tag_ok(ev[r], tg)) ev[r] = edge_wait(el + r, tg);
                        if (need_m[r] && !mail_ok(ql[j][r], ep))
                            ql[j][r] = mail_late2(mbl + r * rstride, min(GAP, nz - 1 - (z - r)), ep, deadline, pl);
                    }
                    if (need_d && !tag_ok(dv, tg)) dv = edge_wait(ed, tg);
                    if (need_md && !mail_ok(qd[j], ep)) qd[j] = mail_late2(mbd, min(GAP, nz - 1 - z), ep, deadline, pd);
                }
#pragma unroll
                for (int r = 0; r < kRpl; ++r)
                    left[r] = need_l ? mail_value(ev[r]) : (need_m[r] ? mail_value(ql[j][r]) : left[r]);
                down0 = need_d ? mail_value(dv) : (need_md ? mail_value(qd[j]) : down0);
                // ---- the rows: b - v0*x0 - v1*x1 - v2*x2 in the reference's order; an absent
                // entry has value 0 and operand 0.0, an exact no-op like the reference's skip
                double xn[kRpl];
#pragma unroll
                for (int r = 0; r < kRpl; ++r) {
                    const uint32_t m = msk4 >> (8 * r);
                    const double dn = r == 0 ? down0 : last[r - 1];
                    double o0, o1, o2;
                    if (ZYX) {
                        o0 = (m & 1u) ? last[r] : 0.0;
                        o1 = (m & 2u) ? dn : 0.0;
                        o2 = (m & 4u) ? left[r] : 0.0;
                    } else {
                        const double lr = left[r], br = last[r];
                        auto nb = [&](int d) { return d == 0 ? lr : (d == 1 ? dn : br); };
                        o0 = (m & 1u) ? nb(d0) : 0.0;
                        o1 = (m & 2u) ? nb(d1) : 0.0;
                        o2 = (m & 4u) ? nb(d2) : 0.0;
                    }
                    const double b1 = UNIT ? __dmul_rn(bb[r], 1.0) : bb[r];  // x / 1.0 == x * 1.0, moved to b
                    double acc = __dsub_rn(b1, __dmul_rn(v[0][r], o0));
                    acc = __dsub_rn(acc, __dmul_rn(v[1][r], o1));
                    acc = __dsub_rn(acc, __dmul_rn(v[2][r], o2));
                    if (UNIT) {
                        xn[r] = acc;
                    } else {
                        const double ad = fabs(dd[r]);
                        bool ok;
                        xn[r] = markstein_dok(acc, dd[r], rr[r], (ad > 0x1p-449) & (ad < 0x1p449), ok);
                        if (__builtin_expect(!ok, 0)) xn[r] = div_slow(acc, dd[r]);
                    }
                }
                HEC_CSTAMP(2, xn[0] + xn[kRpl - 1])
                bool act[kRpl];
#pragma unroll
                for (int r = 0; r < kRpl; ++r) {
                    act[r] = col_ok[r] && static_cast<unsigned>(z - r) < static_cast<unsigned>(nz);
                    if (act[r]) last[r] = xn[r];
                }
                // ---- publish level l to the neighbour warps (edge ring slot l % kEdge)
                const int ew = l % kEdge;
                if (lx == SX - 1 && wx < a.WX - 1) {
                    ulonglong2* e = edge_r + (ew * 64 + w * SY + kRpl * lq);
#pragma unroll
                    for (int r = 0; r < kRpl; ++r) edge_put(e + r, last[r], static_cast<uint32_t>(l + 1));
                }
                if (lq == 3 && wy < a.WY - 1) edge_put(edge_t + ew * 128 + w * 8 + lx, last[kRpl - 1], static_cast<uint32_t>(l + 1));
                HEC_CSTAMP(3, 0.0)
                // ---- off the chain: other CTAs, the output, the slot ring, early mailbox loads
                if (pub_right) {
#pragma unroll
                    for (int r = 0; r < kRpl; ++r)
                        if (act[r]) mail_store(mpr + r * rstride, xn[r], ep);
                }
                if (pub_top && act[kRpl - 1]) mail_store(mpt, xn[kRpl - 1], ep);
                if (kRpl == 1) {
                    *xw = xn[0];
                } else {
#pragma unroll
                    for (int h = 0; h < kRpl; h += 2)  // padding slots take garbage
                        reinterpret_cast<double2*>(xw)[h / 2] = make_double2(xn[h], xn[h + 1 < kRpl ? h + 1 : h]);
                }
                __syncwarp();
                if (lane == 0) mbar_arrive_relaxed(&empty[rs]);  // the slot's values were used above
                if (mb_left) {
#pragma unroll
                    for (int r = 0; r < kRpl; ++r) {
                        const int zr = z + D - r;
                        if (col_ok[r] && static_cast<unsigned>(zr) < static_cast<unsigned>(nz))
                            ql[j][r] = ld_relaxed_v2(mbl + 2 * D + r * rstride);
                    }
                }
                if (mb_down && static_cast<unsigned>(z + D) < static_cast<unsigned>(nz))
                    qd[j] = ld_relaxed_v2(mbd + 2 * D);
                if (TRACE && lane == 0 && w == 0) {
                    tr[0] = gtimer();
                    tr[1] = pl | static_cast<unsigned long long>(pd) << 32;
                    tr[2] = static_cast<unsigned long long>(clock64() - c0);
                }
#undef HEC_CSTAMP
                if (++rs == R) rs = 0, rph ^= 1u;
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

template <int NW, int RPL, bool ZYX>
void* pick(bool unit, bool trace) {
    if (trace)
        return unit ? reinterpret_cast<void*>(&k_cols<NW, RPL, true, true, ZYX>)
                    : reinterpret_cast<void*>(&k_cols<NW, RPL, false, true, ZYX>);
    return unit ? reinterpret_cast<void*>(&k_cols<NW, RPL, true, false, ZYX>)
                : reinterpret_cast<void*>(&k_cols<NW, RPL, false, false, ZYX>);
}
// the (warps, columns per lane) shapes plan::build_columns chooses from
template <bool ZYX>
void* pick_shape(int warps, int rpl, bool unit, bool trace) {
    if (warps == 16 && rpl == 1) return pick<16, 1, ZYX>(unit, trace);
    if (warps == 8 && rpl == 2) return pick<8, 2, ZYX>(unit, trace);
    if (warps == 4 && rpl == 4) return pick<4, 4, ZYX>(unit, trace);
    if (warps == 4 && rpl == 1) return pick<4, 1, ZYX>(unit, trace);
    if (warps == 1 && rpl == 4) return pick<1, 4, ZYX>(unit, trace);
    return nullptr;
}

}  // namespace

void* cols_kernel(int warps, int rpl, bool unit, bool trace, int order) {
    return order == kColOrderZYX ? pick_shape<true>(warps, rpl, unit, trace) : pick_shape<false>(warps, rpl, unit, trace);
}

}  // namespace hec::dev
