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
                // would this row still fit the slot budget?
                const int w2 = std::max(ch.w, std::min(cnt[r], cfg.max_width));
                const int t2 = ch.ntail + std::max(0, cnt[r] - cfg.max_width);
                const int fl = (t2 > 0 ? 1 : 0) | flags_out;
                const int bytes = blob_sections(ch.m + 1, w2, 0, t2, fl).end + 8 * round_up(ch.m + 1, 4) + 16 * 8;
                if (ch.m > 0 && bytes > cfg.slot_cap) break;
                ch.w = w2;
                ch.ntail = t2;
                ++ch.m;
                ++r;
            }
            per_cta[c].push_back(ch);
        }
    }

    // 2. sequence numbers and the progress value that covers each row
    std::vector<int> owner_r(n), seq_r(n), done_r(n), chunk_pos_r(n);
    P.cta_chunk0.assign(static_cast<std::size_t>(C) + 1, 0);
    for (int c = 0; c < C; ++c) {
        P.cta_chunk0[c + 1] = P.cta_chunk0[c] + static_cast<int>(per_cta[c].size());
        int q = 0;
        for (std::size_t j = 0; j < per_cta[c].size(); ++j) {
            const Chunk& ch = per_cta[c][j];
            for (int t = 0; t < ch.m; ++t) {
                owner_r[ch.r0 + t] = c;
                seq_r[ch.r0 + t] = q + t;
                done_r[ch.r0 + t] = q + ch.m;
                chunk_pos_r[ch.r0 + t] = static_cast<int>(j);
            }
            q += ch.m;
        }
    }
    P.chunks = P.cta_chunk0[C];

    // 3. emit blobs
    P.span.assign(2 * static_cast<std::size_t>(P.chunks), 0);
    std::vector<std::vector<unsigned char>> cta_blob(C);
    std::vector<long long> ring_deps(C, 0), global_deps(C, 0), waits_cnt(C, 0);
    std::vector<int> slot_max(C, 0), rows_max(C, 0);
    std::vector<char> bad(C, 0);
#pragma omp parallel for schedule(dynamic, 1)
    for (int c = 0; c < C; ++c) {
        std::vector<int> waited(C, 0);
        std::vector<int> need(C, 0);
        std::vector<int> touched;
        auto& out = cta_blob[c];
        int q0 = 0;
        for (std::size_t j = 0; j < per_cta[c].size(); ++j) {
            const Chunk& ch = per_cta[c][j];
            const int q_end = q0 + ch.m;
            // dependency encoding + cross-CTA needs
            touched.clear();
            auto encode = [&](int col) -> int {
                const int oc = owner_r[col];
                if (oc == c) {
                    if (chunk_pos_r[col] >= static_cast<int>(j)) bad[c] = 1;
                    if (seq_r[col] >= q_end - cfg.ring) {
                        ++ring_deps[c];
                        return -((seq_r[col] & (cfg.ring - 1)) + 1);
                    }
                } else {
                    if (oc > c) bad[c] = 1;
                    if (need[oc] == 0) touched.push_back(oc);
                    need[oc] = std::max(need[oc], done_r[col]);
                }
                ++global_deps[c];
                return sol_index(s, col);
            };
            const int m = ch.m, w = ch.w, mp = round_up(m, 4);
            std::vector<int> dep(static_cast<std::size_t>(w) * mp, -(cfg.ring + 1));
            std::vector<double> val(static_cast<std::size_t>(w) * mp, 0.0);
            std::vector<int> tptr(round_up(mp + 1, 4), 0), tdep;
            std::vector<double> tval;
            for (int t = 0; t < m; ++t) {
                const int r = ch.r0 + t;
                int e = 0;
                for_each_entry(s, r, [&](int col, double v) {
                    const int d = encode(col);
                    if (e < w) {
                        dep[static_cast<std::size_t>(e) * mp + t] = d;
                        val[static_cast<std::size_t>(e) * mp + t] = v;
                    } else {
                        tdep.push_back(d);
                        tval.push_back(v);
                    }
                    ++e;
                });
                tptr[t + 1] = static_cast<int>(tdep.size());
            }
            for (int t = m; t < round_up(mp + 1, 4) - 1; ++t) tptr[t + 1] = tptr[t];
            std::vector<int> waits;
            for (int oc : touched) {
                if (need[oc] > waited[oc]) {
                    waits.push_back(oc);
                    waits.push_back(need[oc]);
                    waited[oc] = need[oc];
                }
                need[oc] = 0;
            }
            const int nwait = static_cast<int>(waits.size() / 2);
            waits_cnt[c] += nwait;
            const int ntail = static_cast<int>(tdep.size());
            const int flags = (ntail > 0 ? 1 : 0) | flags_out;
            const BlobSections sec = blob_sections(m, w, nwait, ntail, flags);
            const std::size_t base = out.size();
            out.resize(base + sec.end, 0);
            unsigned char* b = out.data() + base;
            const int hdr[8] = {m, w, q0, flags, nwait, ntail, 0, 0};
            std::memcpy(b, hdr, sizeof(hdr));
            if (nwait) std::memcpy(b + 32, waits.data(), 8 * static_cast<std::size_t>(nwait));
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
            for (int t = m; t < mp; ++t) {  // padded rows are never processed
                put_i(sec.bidx, t, 0);
                put_i(sec.xidx, t, 0);
            }
            std::memcpy(b + sec.val, val.data(), 8 * val.size());
            std::memcpy(b + sec.dep, dep.data(), 4 * dep.size());
            if (flags & 1) {
                std::memcpy(b + sec.tptr, tptr.data(), 4 * tptr.size());
                std::memcpy(b + sec.tval, tval.data(), 8 * tval.size());
                std::memcpy(b + sec.tdep, tdep.data(), 4 * tdep.size());
            }
            slot_max[c] = std::max(slot_max[c], sec.end);
            rows_max[c] = std::max(rows_max[c], m);
            const int gj = P.cta_chunk0[c] + static_cast<int>(j);
            P.span[2 * gj + 0] = static_cast<int>(base / 16);  // CTA-relative for now
            P.span[2 * gj + 1] = sec.end;
            q0 = q_end;
        }
    }
    for (int c = 0; c < C; ++c)
        if (bad[c]) throw std::invalid_argument("hec_tri_create: dependency order violates the level schedule");

    // 4. concatenate CTA streams (16-byte aligned offsets)
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
        for (int gj = P.cta_chunk0[c]; gj < P.cta_chunk0[c + 1]; ++gj)
            P.span[2 * gj] += static_cast<int>(cta_base[c] / 16);
        P.max_blob = std::max(P.max_blob, slot_max[c]);
        P.max_rows = std::max(P.max_rows, rows_max[c]);
        P.ring_deps += ring_deps[c];
        P.global_deps += global_deps[c];
        P.cross_waits += waits_cnt[c];
    }
    return P;
}

}  // namespace hec::plan
