// Builders for the device layouts of a prepared triangle (host, once per
// prepare). See tri_plan.hpp for the layouts and DESIGN.md §3 for the
// reasoning. Arithmetic order per row is kept exactly as the reference's
// solve (proj/src/triangular.cpp:118-126): ELL slots 0..w-1 (padding skipped,
// it contributes acc - 0*0 == acc there), CSR entries in storage order, then
// one IEEE division by the diagonal (the CSR row's last entry).

#include "tri_plan.hpp"

#include <algorithm>
#include <cstring>
#include <stdexcept>
#include <string>
#include <unordered_map>

namespace hec::plan {

namespace {

inline int sol_index(const TriSource& s, int reordered) {
    const int i = s.inv_perm[reordered];
    return s.reversed ? s.n - 1 - i : i;
}

// Visits the off-diagonal entries of reordered row r in solve order.
template <class F>
inline void for_each_entry(const TriSource& s, int r, F&& f) {
    for (int k = 0; k < s.ell_width; ++k) {
        const std::size_t slot = static_cast<std::size_t>(k) * s.n + r;
        const int c = s.ell_cols[slot];
        if (c == r) continue;  // padding (reference hec.cpp:69,76)
        f(c, s.ell_vals[slot]);
    }
    for (int k = s.csr_rp[r]; k < s.csr_rp[r + 1] - 1; ++k) f(s.csr_cols[k], s.csr_vals[k]);
}

inline int entry_count(const TriSource& s, int r) {
    int cnt = 0;
    for (int k = 0; k < s.ell_width; ++k)
        if (s.ell_cols[static_cast<std::size_t>(k) * s.n + r] != r) ++cnt;
    return cnt + (s.csr_rp[r + 1] - s.csr_rp[r] - 1);
}

}  // namespace

void validate(const TriSource& s) {
    if (s.n < 0 || s.nlev < 0 || s.ell_width < 0)
        throw std::invalid_argument("hec_tri_create: negative size");
    if (s.n == 0) return;
    if (!s.level_starts || !s.inv_perm || !s.csr_rp || (s.ell_width > 0 && (!s.ell_cols || !s.ell_vals)))
        throw std::invalid_argument("hec_tri_create: missing array");
    if (s.level_starts[0] != 0 || s.level_starts[s.nlev] != s.n)
        throw std::invalid_argument("hec_tri_create: level_starts must span [0, n]");
    for (int k = 0; k < s.nlev; ++k)
        if (s.level_starts[k + 1] <= s.level_starts[k])
            throw std::invalid_argument("hec_tri_create: empty or decreasing level");
    std::vector<int> level_of_r(s.n);
    for (int k = 0; k < s.nlev; ++k)
        for (int r = s.level_starts[k]; r < s.level_starts[k + 1]; ++r) level_of_r[r] = k;
    std::vector<char> seen(s.n, 0);
    for (int r = 0; r < s.n; ++r) {
        const int i = s.inv_perm[r];
        if (i < 0 || i >= s.n || seen[i]) throw std::invalid_argument("hec_tri_create: inv_perm is not a permutation");
        seen[i] = 1;
        if (s.csr_rp[r + 1] <= s.csr_rp[r])
            throw std::invalid_argument("hec_tri_create: row " + std::to_string(r) + " has no diagonal");
        if (s.csr_cols[s.csr_rp[r + 1] - 1] != r)
            throw std::invalid_argument("hec_tri_create: CSR row " + std::to_string(r) + " must end on its diagonal");
        bool ok = true;
        for_each_entry(s, r, [&](int c, double) {
            if (c < 0 || c >= s.n || level_of_r[c] >= level_of_r[r]) ok = false;
        });
        if (!ok)
            throw std::invalid_argument("hec_tri_create: row " + std::to_string(r) +
                                        " depends on a row of the same or a later level");
    }
}

LevelLayout build_levels(const TriSource& s) {
    LevelLayout L;
    L.n = s.n;
    L.ld = round_up(std::max(s.n, 1), 32);
    L.width = s.ell_width;
    L.nlev = s.nlev;
    L.level_starts.assign(s.level_starts, s.level_starts + s.nlev + 1);
    L.xidx.resize(s.n);
    L.bidx.resize(s.n);
    if (s.out_map) L.oidx.resize(s.n);
    L.ell_dep.assign(static_cast<std::size_t>(L.width) * L.ld, -1);
    L.ell_val.assign(static_cast<std::size_t>(L.width) * L.ld, 0.0);
    L.diag.resize(s.n);
    L.tail_rp.assign(static_cast<std::size_t>(s.n) + 1, 0);
    for (int r = 0; r < s.n; ++r) L.tail_rp[r + 1] = L.tail_rp[r] + (s.csr_rp[r + 1] - s.csr_rp[r] - 1);
    L.tail_dep.resize(L.tail_rp[s.n]);
    L.tail_val.resize(L.tail_rp[s.n]);
#pragma omp parallel for schedule(static)
    for (int r = 0; r < s.n; ++r) {
        const int o = sol_index(s, r);
        L.xidx[r] = o;
        L.bidx[r] = s.b_map ? s.b_map[o] : o;
        if (s.out_map) L.oidx[r] = s.out_map[o];
        for (int k = 0; k < s.ell_width; ++k) {
            const std::size_t src = static_cast<std::size_t>(k) * s.n + r;
            const std::size_t dst = static_cast<std::size_t>(k) * L.ld + r;
            if (s.ell_cols[src] == r) continue;
            L.ell_dep[dst] = sol_index(s, s.ell_cols[src]);
            L.ell_val[dst] = s.ell_vals[src];
        }
        int t = L.tail_rp[r];
        for (int k = s.csr_rp[r]; k < s.csr_rp[r + 1] - 1; ++k, ++t) {
            L.tail_dep[t] = sol_index(s, s.csr_cols[k]);
            L.tail_val[t] = s.csr_vals[k];
        }
        L.diag[r] = s.csr_vals[s.csr_rp[r + 1] - 1];
    }
    return L;
}

PipelineLayout build_pipeline(const TriSource& s, const PipelineConfig& cfg) {
    PipelineLayout P;
    const int n = s.n;
    const int C = std::max(1, std::min(cfg.ctas, std::max(n, 1)));
    P.n = n;
    P.nlev = s.nlev;
    P.ctas = C;
    P.ring = cfg.ring;
    P.has_out = s.out_map != nullptr;
    const int per = n > 0 ? (n + C - 1) / C : 1;
    auto owner_of_i = [&](int i) { return std::min(i / per, C - 1); };

    // 1. chunk discovery: level-major walk, runs of equal owner (split by size)
    struct Chunk { int cta, level, r0, m, w, ntail; };
    std::vector<int> cnt(n);
#pragma omp parallel for schedule(static)
    for (int r = 0; r < n; ++r) cnt[r] = entry_count(s, r);

    std::vector<std::vector<Chunk>> per_cta(C);
    const int flags_out = P.has_out ? 2 : 0;
    for (int k = 0; k < s.nlev; ++k) {
        int r = s.level_starts[k];
        const int re = s.level_starts[k + 1];
        while (r < re) {
            const int c = owner_of_i(s.inv_perm[r]);
            Chunk ch{c, k, r, 0, 0, 0};
            while (r < re && owner_of_i(s.inv_perm[r]) == c) {
                const int w2 = std::max(ch.w, std::min(cnt[r], cfg.max_width));
                const int t2 = ch.ntail + std::max(0, cnt[r] - cfg.max_width);
                const int fl = (t2 > 0 ? 1 : 0) | flags_out | 4;
                // blob + gathered b + (typical) one halo value and one mailbox per row
                const int bytes = blob_sections(ch.m + 1, w2, ch.m + 1, ch.m + 1, t2, fl).end +
                                  16 * round_up(ch.m + 1, 4);
                if (ch.m > 0 && bytes > cfg.slot_cap) break;
                ch.w = w2;
                ch.ntail = t2;
                ++ch.m;
                ++r;
            }
            per_cta[c].push_back(ch);
        }
    }

    // 2. owner, sequence number and chunk position of every reordered row
    std::vector<int> owner_r(n), seq_r(n), chunk_pos_r(n);
    P.cta_chunk0.assign(static_cast<std::size_t>(C) + 1, 0);
    for (int c = 0; c < C; ++c) {
        P.cta_chunk0[c + 1] = P.cta_chunk0[c] + static_cast<int>(per_cta[c].size());
        int q = 0;
        for (std::size_t j = 0; j < per_cta[c].size(); ++j) {
            const Chunk& ch = per_cta[c][j];
            for (int t = 0; t < ch.m; ++t) {
                owner_r[ch.r0 + t] = c;
                seq_r[ch.r0 + t] = q + t;
                chunk_pos_r[ch.r0 + t] = static_cast<int>(j);
            }
            q += ch.m;
        }
    }
    P.chunks = P.cta_chunk0[C];

    // 3. consumer side (parallel over CTAs): dependency codes, per-chunk halo
    //    lists and the CTA's mailboxes (one per foreign producer row).
    struct CtaWork {
        std::vector<std::vector<int>> dep, tdep, tptr, halo;  // per chunk
        std::vector<std::vector<double>> val, tval;
        std::vector<int> mb_row;        // local mailbox -> producer reordered row
        std::vector<int> mb_last;       // local mailbox -> last chunk that reads it
        std::vector<char> has_global;   // per chunk: some dependency read from global x
        long long ring_deps = 0, global_deps = 0, halo_deps = 0;
        bool bad = false;
    };
    std::vector<CtaWork> work(C);
#pragma omp parallel for schedule(dynamic, 1)
    for (int c = 0; c < C; ++c) {
        CtaWork& W = work[c];
        const std::size_t nchk = per_cta[c].size();
        W.dep.resize(nchk);
        W.val.resize(nchk);
        W.tdep.resize(nchk);
        W.tval.resize(nchk);
        W.tptr.resize(nchk);
        W.halo.resize(nchk);
        W.has_global.assign(nchk, 0);
        std::unordered_map<int, int> mb_of;   // producer row -> local mailbox
        std::unordered_map<int, int> halo_of; // local mailbox -> halo slot (this chunk)
        int q0 = 0;
        for (std::size_t j = 0; j < nchk; ++j) {
            const Chunk& ch = per_cta[c][j];
            const int q_end = q0 + ch.m;
            const int m = ch.m, w = ch.w, mp = round_up(m, 4);
            halo_of.clear();
            auto& halo = W.halo[j];
            auto encode = [&](int col) -> int {
                const int oc = owner_r[col];
                if (oc == c) {
                    if (chunk_pos_r[col] >= static_cast<int>(j)) W.bad = true;
                    if (seq_r[col] >= q_end - cfg.ring) {
                        ++W.ring_deps;
                        return -((seq_r[col] & (cfg.ring - 1)) + 1);
                    }
                    ++W.global_deps;
                    W.has_global[j] = 1;
                    return sol_index(s, col);
                }
                if (oc > c) W.bad = true;
                auto it = mb_of.find(col);
                int mb;
                if (it == mb_of.end()) {
                    mb = static_cast<int>(W.mb_row.size());
                    mb_of.emplace(col, mb);
                    W.mb_row.push_back(col);
                    W.mb_last.push_back(static_cast<int>(j));
                } else {
                    mb = it->second;
                    W.mb_last[mb] = static_cast<int>(j);
                }
                auto hit = halo_of.find(mb);
                int h;
                if (hit == halo_of.end()) {
                    h = static_cast<int>(halo.size());
                    halo_of.emplace(mb, h);
                    halo.push_back(mb);
                } else {
                    h = hit->second;
                }
                ++W.halo_deps;
                return -(cfg.ring + 2 + h);
            };
            auto& dep = W.dep[j];
            auto& val = W.val[j];
            auto& tptr = W.tptr[j];
            dep.assign(static_cast<std::size_t>(w) * mp, -(cfg.ring + 1));
            val.assign(static_cast<std::size_t>(w) * mp, 0.0);
            tptr.assign(round_up(mp + 1, 4), 0);
            for (int t = 0; t < m; ++t) {
                const int r = ch.r0 + t;
                int e = 0;
                for_each_entry(s, r, [&](int col, double v) {
                    const int d = encode(col);
                    if (e < w) {
                        dep[static_cast<std::size_t>(e) * mp + t] = d;
                        val[static_cast<std::size_t>(e) * mp + t] = v;
                    } else {
                        W.tdep[j].push_back(d);
                        W.tval[j].push_back(v);
                    }
                    ++e;
                });
                tptr[t + 1] = static_cast<int>(W.tdep[j].size());
            }
            for (int t = m; t < static_cast<int>(tptr.size()) - 1; ++t) tptr[t + 1] = tptr[t];
            q0 = q_end;
        }
    }
    for (int c = 0; c < C; ++c)
        if (work[c].bad) throw std::invalid_argument("hec_tri_create: dependency order violates the level schedule");

    // 4. global mailbox ids and the producer-side lists (reordered row -> ids)
    std::vector<long long> mb_base(static_cast<std::size_t>(C) + 1, 0);
    for (int c = 0; c < C; ++c) mb_base[c + 1] = mb_base[c] + static_cast<long long>(work[c].mb_row.size());
    P.mailboxes = mb_base[C];
    if (P.mailboxes > 0x3fffffffLL) throw std::overflow_error("hec_tri_create: too many cross-CTA values");
    std::vector<int> feed_ptr(static_cast<std::size_t>(n) + 1, 0);
    for (int c = 0; c < C; ++c)
        for (int r : work[c].mb_row) ++feed_ptr[r + 1];
    for (int r = 0; r < n; ++r) feed_ptr[r + 1] += feed_ptr[r];
    std::vector<int> feed(static_cast<std::size_t>(feed_ptr[n]));
    {
        std::vector<int> fill(feed_ptr.begin(), feed_ptr.end() - 1);
        for (int c = 0; c < C; ++c)
            for (std::size_t l = 0; l < work[c].mb_row.size(); ++l)
                feed[fill[work[c].mb_row[l]]++] = static_cast<int>(mb_base[c] + static_cast<long long>(l));
    }

    // 5. emit blobs (parallel over CTAs)
    P.span.assign(2 * static_cast<std::size_t>(P.chunks), 0);
    std::vector<std::vector<unsigned char>> cta_blob(C);
    std::vector<int> blob_max(C, 0), rows_max(C, 0), halo_max(C, 0);
#pragma omp parallel for schedule(dynamic, 1)
    for (int c = 0; c < C; ++c) {
        CtaWork& W = work[c];
        auto& out = cta_blob[c];
        int q0 = 0;
        for (std::size_t j = 0; j < per_cta[c].size(); ++j) {
            const Chunk& ch = per_cta[c][j];
            const int m = ch.m, w = ch.w, mp = round_up(m, 4);
            std::vector<int> mbptr(round_up(mp + 1, 4), 0), mbid;
            for (int t = 0; t < m; ++t) {
                const int r = ch.r0 + t;
                for (int k = feed_ptr[r]; k < feed_ptr[r + 1]; ++k) mbid.push_back(feed[k]);
                mbptr[t + 1] = static_cast<int>(mbid.size());
            }
            for (int t = m; t < static_cast<int>(mbptr.size()) - 1; ++t) mbptr[t + 1] = mbptr[t];
            const int nmb = static_cast<int>(mbid.size());
            const int nhalo = static_cast<int>(W.halo[j].size());
            const int ntail = static_cast<int>(W.tdep[j].size());
            const int flags = (ntail > 0 ? 1 : 0) | flags_out | (nmb > 0 ? 4 : 0) | (W.has_global[j] ? 8 : 0);
            const BlobSections sec = blob_sections(m, w, nhalo, nmb, ntail, flags);
            const std::size_t base = out.size();
            out.resize(base + sec.end, 0);
            unsigned char* b = out.data() + base;
            const ChunkHeader hdr{m,        w,         q0,       flags,    nhalo,    ntail,     nmb,
                                  mp,       sec.halo,  sec.mbptr, sec.mbid, sec.diag, sec.val,   sec.dep,
                                  sec.bidx, sec.xidx,  sec.oidx, sec.tptr, sec.tval, sec.tdep, {0, 0, 0, 0}};
            std::memcpy(b, &hdr, sizeof(hdr));
            for (int h = 0; h < nhalo; ++h) {
                const int l = W.halo[j][h];
                const long long gid = mb_base[c] + l;
                const int code = static_cast<int>(gid * 2 + (W.mb_last[l] == static_cast<int>(j) ? 1 : 0));
                std::memcpy(b + sec.halo + 4 * h, &code, 4);
            }
            if (flags & 4) {
                std::memcpy(b + sec.mbptr, mbptr.data(), 4 * mbptr.size());
                std::memcpy(b + sec.mbid, mbid.data(), 4 * mbid.size());
            }
            auto put_i = [&](int off, int idx, int v) { std::memcpy(b + off + 4 * idx, &v, 4); };
            auto put_d = [&](int off, int idx, double v) { std::memcpy(b + off + 8 * idx, &v, 8); };
            for (int t = 0; t < m; ++t) {
                const int r = ch.r0 + t;
                const int o = sol_index(s, r);
                put_d(sec.diag, t, s.csr_vals[s.csr_rp[r + 1] - 1]);
                put_i(sec.bidx, t, s.b_map ? s.b_map[o] : o);
                put_i(sec.xidx, t, o);
                if (flags & 2) put_i(sec.oidx, t, s.out_map[o]);
            }
            std::memcpy(b + sec.val, W.val[j].data(), 8 * W.val[j].size());
            std::memcpy(b + sec.dep, W.dep[j].data(), 4 * W.dep[j].size());
            if (flags & 1) {
                std::memcpy(b + sec.tptr, W.tptr[j].data(), 4 * W.tptr[j].size());
                std::memcpy(b + sec.tval, W.tval[j].data(), 8 * W.tval[j].size());
                std::memcpy(b + sec.tdep, W.tdep[j].data(), 4 * W.tdep[j].size());
            }
            blob_max[c] = std::max(blob_max[c], sec.end);
            rows_max[c] = std::max(rows_max[c], m);
            halo_max[c] = std::max(halo_max[c], nhalo);
            const int gj = P.cta_chunk0[c] + static_cast<int>(j);
            P.span[2 * gj + 0] = static_cast<int>(base / 16);  // CTA-relative for now
            P.span[2 * gj + 1] = sec.end;
            q0 += m;
            // free the consumer-side scratch as we go
            std::vector<int>().swap(W.dep[j]);
            std::vector<double>().swap(W.val[j]);
        }
    }

    // 6. concatenate CTA streams (16-byte aligned offsets)
    std::size_t total = 0;
    std::vector<std::size_t> cta_base(C);
    for (int c = 0; c < C; ++c) {
        cta_base[c] = total;
        total += cta_blob[c].size();
    }
    if (total / 16 > 0x7fffffffULL) throw std::overflow_error("hec_tri_create: layout exceeds 32 GiB");
    P.blob.resize(total);
    for (int c = 0; c < C; ++c) {
        std::memcpy(P.blob.data() + cta_base[c], cta_blob[c].data(), cta_blob[c].size());
        std::vector<unsigned char>().swap(cta_blob[c]);
        for (int gj = P.cta_chunk0[c]; gj < P.cta_chunk0[c + 1]; ++gj)
            P.span[2 * gj] += static_cast<int>(cta_base[c] / 16);
        P.max_blob = std::max(P.max_blob, blob_max[c]);
        P.max_rows = std::max(P.max_rows, rows_max[c]);
        P.max_halo = std::max(P.max_halo, halo_max[c]);
        P.ring_deps += work[c].ring_deps;
        P.global_deps += work[c].global_deps;
        P.halo_deps += work[c].halo_deps;
    }
    return P;
}

}  // namespace hec::plan
