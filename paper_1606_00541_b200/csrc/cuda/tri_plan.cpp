// Builders for the device layouts of a prepared triangle (host, once per
// prepare). See tri_plan.hpp for the layouts and DESIGN.md §3 for the
// reasoning. Arithmetic order per row is kept exactly as the reference's
// solve (proj/src/triangular.cpp:118-126): ELL slots 0..w-1 (padding skipped,
// it contributes acc - 0*0 == acc there), CSR entries in storage order, then
// one IEEE division by the diagonal (the CSR row's last entry).

#include "tri_plan.hpp"

#include <algorithm>
#include <cmath>
#include <climits>
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

// ---- structured-grid recognition (pencil ownership) ----
struct GridGeom {
    bool ok = false;
    int nx = 0, ny = 0, nz = 0;
};

// The factor of a 7- or 27-point stencil on an nx x ny x nz grid in natural
// order has, in the lower frame, dependency offsets {1, nx, nx*ny} or
// {1, nx-1..nx+1, nx*ny-nx-1 .. nx*ny+nx+1} on almost every row. Recognise
// them on a sample of rows; anything else keeps the slab ownership.
GridGeom detect_grid(const TriSource& s) {
    GridGeom g;
    const int n = s.n;
    if (n < 4096) return g;
    std::unordered_map<int, long long> freq;
    const int step = std::max(1, n / 100000);
    long long rows = 0;
    for (int r = 0; r < n; r += step) {
        const int i = s.inv_perm[r];
        ++rows;
        for_each_entry(s, r, [&](int col, double) { ++freq[i - s.inv_perm[col]]; });
    }
    std::vector<int> frequent;
    for (const auto& [d, c] : freq)
        if (d > 0 && c * 2 >= rows) frequent.push_back(d);
    std::sort(frequent.begin(), frequent.end());
    if (frequent.size() < 3 || frequent[0] != 1) return g;
    auto has = [&](int d) { return std::binary_search(frequent.begin(), frequent.end(), d); };
    const int d2 = frequent[1];
    const int nx = (has(d2 + 1) && has(d2 + 2)) ? d2 + 1 : d2;  // 27-point: nx-1, nx, nx+1
    std::vector<int> big;
    for (int d : frequent)
        if (d > nx + 1) big.push_back(d);
    if (big.empty()) return g;
    const long long plane = (static_cast<long long>(big.front()) + big.back()) / 2;
    if (nx < 4 || plane % nx != 0 || n % plane != 0) return g;
    g.nx = nx;
    g.ny = static_cast<int>(plane / nx);
    g.nz = static_cast<int>(n / plane);
    g.ok = g.ny >= 4 && g.nz >= 2;
    return g;
}

// Grid coordinates from the dependency DAG, for orderings other than the natural
// one that still orient every grid edge towards increasing coordinates (reverse
// Cuthill-McKee started at a corner, and other orderings that grow from a
// corner): the factor of a 7-point stencil then has a single source (the
// corner); a row with one predecessor continues its predecessor's axis line
// (the corner's successors open the three axes); a row with two or three
// predecessors sits at their component-wise maximum. Checked: every dependency
// is a unit step from the previous level and the coordinates fill an X x Y x Z
// box exactly once -- anything else returns false. cx, cy: x and y of every
// lower-frame row.
bool dag_grid(const TriSource& s, std::vector<int>& cx, std::vector<int>& cy, GridGeom& g) {
    const int n = s.n;
    if (n < 4096) return false;
    std::vector<int> lev(n);
    for (int k = 0; k < s.nlev; ++k)
        for (int r = s.level_starts[k]; r < s.level_starts[k + 1]; ++r) lev[s.inv_perm[r]] = k;
    std::vector<int> co(3 * static_cast<std::size_t>(n), 0);
    std::vector<signed char> axis(n, -1);
    int next_axis = 0;
    for (int r = 0; r < n; ++r) {  // level-major: every predecessor comes first
        const int i = s.inv_perm[r];
        int pr[4], np = 0;
        for_each_entry(s, r, [&](int col, double) {
            if (np < 4) pr[np] = s.inv_perm[col];
            ++np;
        });
        int* c = &co[3 * static_cast<std::size_t>(i)];
        if (np > 3) return false;
        if (np == 0) {
            if (r != 0) return false;  // one source only
            continue;
        }
        for (int k = 0; k < np; ++k)
            if (lev[pr[k]] != lev[i] - 1) return false;
        if (np == 1) {
            const int p = pr[0];
            int a;
            if (lev[p] == 0) {
                if (next_axis >= 3) return false;
                a = next_axis++;
            } else {
                a = axis[p];
                if (a < 0) return false;
            }
            for (int d = 0; d < 3; ++d) c[d] = co[3 * static_cast<std::size_t>(p) + d];
            c[a] += 1;
            axis[i] = static_cast<signed char>(a);
            continue;
        }
        for (int d = 0; d < 3; ++d) {
            int m = 0;
            for (int k = 0; k < np; ++k) m = std::max(m, co[3 * static_cast<std::size_t>(pr[k]) + d]);
            c[d] = m;
        }
        for (int k = 0; k < np; ++k) {  // a unit step from every predecessor
            int diff = 0;
            for (int d = 0; d < 3; ++d) diff += c[d] - co[3 * static_cast<std::size_t>(pr[k]) + d];
            if (diff != 1) return false;
        }
    }
    int ext[3] = {0, 0, 0};
    for (int i = 0; i < n; ++i)
        for (int d = 0; d < 3; ++d) ext[d] = std::max(ext[d], co[3 * static_cast<std::size_t>(i) + d] + 1);
    if (static_cast<long long>(ext[0]) * ext[1] * ext[2] != n) return false;
    std::vector<unsigned char> seen(n, 0);
    for (int i = 0; i < n; ++i) {
        const int* c = &co[3 * static_cast<std::size_t>(i)];
        const long long at = c[0] + static_cast<long long>(ext[0]) * (c[1] + static_cast<long long>(ext[1]) * c[2]);
        if (seen[at]++) return false;
    }
    cx.resize(n);
    cy.resize(n);
    for (int i = 0; i < n; ++i) {
        cx[i] = co[3 * static_cast<std::size_t>(i)];
        cy[i] = co[3 * static_cast<std::size_t>(i) + 1];
    }
    g.nx = ext[0];
    g.ny = ext[1];
    g.nz = ext[2];
    g.ok = g.nx >= 4 && g.ny >= 4 && g.nz >= 2;
    return g.ok;
}

// CTA tiles of (4 sx) x (4 sy) columns in x-y, each split into 4 x 4 warp
// sub-tiles of sx x sy <= 32 columns (so a level never gives a warp more than
// 32 rows): the most CTAs that fit C, ties to square sub-tiles. cx / cy: the
// rows' grid coordinates when the ordering is not the natural one (else null).
bool pencil_owners(const GridGeom& g, int n, int C, int NW, std::vector<int>& owner, std::vector<int>& warp,
                   int& used, const int* cx = nullptr, const int* cy = nullptr) {
    int best = -1, bsx = 0, bsy = 0, bpx = 0, bpy = 0;
    for (int sx = 1; sx <= 32; ++sx)
        for (int sy = 1; sx * sy <= 32; ++sy) {
            const int px = (g.nx + 4 * sx - 1) / (4 * sx), py = (g.ny + 4 * sy - 1) / (4 * sy);
            if (px * py > C || px < 2 || py < 2) continue;
            const int score = px * py * 64 - std::abs(sx - sy);
            if (score > best) {
                best = score;
                bsx = sx;
                bsy = sy;
                bpx = px;
                bpy = py;
            }
        }
    if (best < 0) return false;
    const int tw = 4 * bsx, th = 4 * bsy;
#pragma omp parallel for schedule(static)
    for (int i = 0; i < n; ++i) {
        const int x = cx ? cx[i] : i % g.nx, y = cy ? cy[i] : (i / g.nx) % g.ny;
        const int px = x / tw, py = y / th;
        owner[i] = py * bpx + px;
        warp[i] = (((y - py * th) / bsy) * 4 + (x - px * tw) / bsx) * NW / 16;  // 4x4 sub-tiles -> NW warps
    }
    used = bpx * bpy;
    return true;
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

LevelLayout build_levels(const TriSource& s, int long_min) {
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
    L.long_min = std::max(0, long_min);
    L.long_starts.assign(static_cast<std::size_t>(s.nlev) + 1, 0);
    for (int k = 0; k < s.nlev; ++k) {
        if (L.long_min > 0)
            for (int r = s.level_starts[k]; r < s.level_starts[k + 1]; ++r)
                if (L.tail_rp[r + 1] - L.tail_rp[r] >= L.long_min) L.long_rows.push_back(r);
        L.long_starts[k + 1] = static_cast<int>(L.long_rows.size());
    }
    if (L.long_rows.empty()) L.long_min = 0;
    return L;
}

WaveLayout build_wave(const TriSource& s, const WaveConfig& cfg) {
    WaveLayout P;
    const int n = s.n;
    const int C0 = std::max(1, std::min(cfg.ctas, std::max(n, 1)));
    int NW = std::max(1, std::min(cfg.group > 0 ? cfg.group : 4, 16));  // warps per chunk (group size G)
    int warp_rows = 32 * std::max(1, cfg.rpl);
    int R = cfg.ring;  // may shrink below (after the sequence numbers are known)
    P.n = n;
    P.nlev = s.nlev;
    P.warps = NW;
    P.ring = R;
    P.inflight = cfg.inflight;
    P.lead = std::max(1, std::min(cfg.lead, cfg.inflight));
    P.has_out = s.out_map != nullptr;
    // ---- ownership: row -> (CTA, warp) in the lower frame
    std::vector<int> owner_i(n), warp_i(n);
    int C_used = C0;
    const WaveMirror* M = cfg.mirror;
    // mirrored layout: the mirrored CTA of each row (warps are dealt by position below)
    std::vector<int> mirror_chunk_of_p;  // L wave position -> L chunk
    if (M) {
        if (M->ctas < 1 || !M->cta_chunk0 || !M->chunk_r0 || !M->wpos)
            throw std::invalid_argument("wave mirror: incomplete");
        const int nch = M->cta_chunk0[M->ctas];
        if (M->chunk_r0[nch] != n) throw std::invalid_argument("wave mirror: size mismatch");
        mirror_chunk_of_p.assign(n, 0);
        std::vector<int> cta_of_chunk(nch);
        for (int c = 0; c < M->ctas; ++c)
            for (int g = M->cta_chunk0[c]; g < M->cta_chunk0[c + 1]; ++g) cta_of_chunk[g] = c;
        for (int g = 0; g < nch; ++g)
            for (int p = M->chunk_r0[g]; p < M->chunk_r0[g + 1]; ++p) mirror_chunk_of_p[p] = g;
        for (int i = 0; i < n; ++i) {
            const int o = s.reversed ? n - 1 - i : i;
            owner_i[i] = M->ctas - 1 - cta_of_chunk[mirror_chunk_of_p[M->wpos[o]]];
            warp_i[i] = 0;
        }
        C_used = M->ctas;
    }
    const GridGeom geo = (cfg.pencils && !M) ? detect_grid(s) : GridGeom{};
    // pencils only when they shorten the per-CTA level chain (the most levels
    // any CTA must walk through): true for 7-point stencils (levels x+y+z),
    // not for 27-point ones (x+2y+4z: a z-pencil spans 4 nz levels)
    auto max_levels_per_cta = [&](const std::vector<int>& own, int ncta) {
        std::vector<int> lev_of_i(n);
        for (int k = 0; k < s.nlev; ++k)
            for (int r = s.level_starts[k]; r < s.level_starts[k + 1]; ++r) lev_of_i[s.inv_perm[r]] = k;
        std::vector<int> lo(ncta, INT32_MAX), hi(ncta, -1);
        for (int i = 0; i < n; ++i) {
            lo[own[i]] = std::min(lo[own[i]], lev_of_i[i]);
            hi[own[i]] = std::max(hi[own[i]], lev_of_i[i]);
        }
        int m = 0;
        for (int c = 0; c < ncta; ++c)
            if (hi[c] >= 0) m = std::max(m, hi[c] - lo[c] + 1);
        return m;
    };
    bool use_pencils = false;
    auto slab_levels = [&]() {
        const int per = (n + C0 - 1) / C0;
        std::vector<int> slab(n);
        for (int i = 0; i < n; ++i) slab[i] = std::min(i / per, C0 - 1);
        return max_levels_per_cta(slab, C0);
    };
    if (!M && geo.ok && pencil_owners(geo, n, C0, 16, owner_i, warp_i, C_used))
        use_pencils = max_levels_per_cta(owner_i, C_used) < slab_levels();
    // a renumbered grid (e.g. RCM): the index offsets say nothing, the dependency
    // DAG still has the grid's shape -- take the coordinates from it
    GridGeom geo_dag;
    std::vector<int> dag_x, dag_y;
    // DAG grid, against the strips such an ordering would get otherwise (every CTA
    // walks every level there)
    if (!use_pencils && cfg.pencils && !M && dag_grid(s, dag_x, dag_y, geo_dag) &&
        pencil_owners(geo_dag, n, C0, 16, owner_i, warp_i, C_used, dag_x.data(), dag_y.data()))
        use_pencils = max_levels_per_cta(owner_i, C_used) < std::min(s.nlev, slab_levels() * 8);
    if (!use_pencils) geo_dag.ok = false;
    // strips: when the row index follows the levels (e.g. an RCM ordering), index
    // slabs would give each CTA only a handful of consecutive levels and the CTAs
    // would run one after another; then every CTA takes a fraction of every level
    bool use_strips = false;
    if (!M && !use_pencils && cfg.strips) {
        const int per = (n + C0 - 1) / C0;
        std::vector<int> slab(n);
        for (int i = 0; i < n; ++i) slab[i] = std::min(i / per, C0 - 1);
        use_strips = s.nlev >= 16 && static_cast<long long>(max_levels_per_cta(slab, C0)) * 8 < s.nlev;
    }
    if (M) {
        P.mirrored = true;
    } else if (use_pencils) {
        P.pencils = true;
        P.grid_nx = geo_dag.ok ? geo_dag.nx : geo.nx;
        P.grid_ny = geo_dag.ok ? geo_dag.ny : geo.ny;
    } else if (use_strips) {
        P.strips = true;
        for (int k = 0; k < s.nlev; ++k) {
            const int r0 = s.level_starts[k], mk = s.level_starts[k + 1] - r0;
            for (int c = 0; c < C0; ++c) {
                const int a0 = static_cast<int>(static_cast<long long>(mk) * c / C0);
                const int a1 = static_cast<int>(static_cast<long long>(mk) * (c + 1) / C0);
                const int pw = std::max(1, (a1 - a0 + NW - 1) / NW);
                for (int q = a0; q < a1; ++q) {
                    owner_i[s.inv_perm[r0 + q]] = c;
                    warp_i[s.inv_perm[r0 + q]] = std::min((q - a0) / pw, NW - 1);
                }
            }
        }
        C_used = C0;
    } else {
        // slabs: CTA c owns [c*per, (c+1)*per), warps contiguous sub-ranges. On a
        // recognised grid the slabs are whole z-planes (a plane split between two
        // CTAs adds in-plane crossings: 27-pt 128^3 with 128 CTAs of one plane is
        // 3 % faster than 148 CTAs of 0.86 plane)
        int per = n > 0 ? (n + C0 - 1) / C0 : 1;
        C_used = C0;
        if (geo.ok && static_cast<long long>(geo.nx) * geo.ny * geo.nz == n && geo.nz >= 2) {
            const int planes = (geo.nz + C0 - 1) / C0;
            per = planes * geo.nx * geo.ny;
            C_used = (geo.nz + planes - 1) / planes;
        }
        const int Cs = C_used;
        const int per_w = (per + NW - 1) / NW;
#pragma omp parallel for schedule(static)
        for (int i = 0; i < n; ++i) {
            owner_i[i] = std::min(i / per, Cs - 1);
            warp_i[i] = std::min((i - owner_i[i] * per) / per_w, NW - 1);
        }
    }
    P.ctas = C_used;
    const int C = C_used;

    // solver shape: K groups of G warps take the chunks round robin, each chunk's
    // rows dealt to its group's warps (RPL rows per lane). Auto: from the rows a
    // CTA has in one level (95th percentile over the (CTA, level) pairs).
    int K = std::max(1, cfg.groups);
    bool big_auto = false;  // > 128 rows per CTA level: 4x2x4, or 8x2x2 for narrow rows (below)
    if (cfg.group <= 0 && n > 0) {
        std::vector<int> lev_cnt(static_cast<std::size_t>(C), 0), sizes;
        for (int k = 0; k < s.nlev; ++k) {
            for (int r = s.level_starts[k]; r < s.level_starts[k + 1]; ++r) ++lev_cnt[owner_i[s.inv_perm[r]]];
            for (int r = s.level_starts[k]; r < s.level_starts[k + 1]; ++r) {
                int& v = lev_cnt[owner_i[s.inv_perm[r]]];
                if (v) sizes.push_back(v);
                v = 0;
            }
        }
        auto p95 = sizes.begin() + static_cast<long>(sizes.size() * 95 / 100);
        std::nth_element(sizes.begin(), p95, sizes.end());
        const int m95 = sizes.empty() ? 0 : *p95;
        // one row per lane: twice the warps of the two-rows-per-lane shapes, each
        // with half the gathers on its critical path (27-pt 128^3 apply
        // 0.946 -> 0.922 ms, 7-pt 128^3 0.277 -> 0.264 ms)
        if (m95 <= 64) { NW = 2; warp_rows = 32; K = 4; }
        else if (m95 <= 128) { NW = 4; warp_rows = 32; K = 4; }
        else { NW = 4; warp_rows = 128; K = 2; big_auto = true; }
    }
    P.group = NW;
    P.groups = K;
    P.warps = NW * K;
    P.rpl = std::max(1, warp_rows / 32);
    P.lead = 1;  // chunks complete in order: no warp runs ahead of another
    const bool lockstep = true;

    std::vector<int> cnt(n), owner_r(n), warp_r(n), nforeign(n, 0);
#pragma omp parallel for schedule(static)
    for (int r = 0; r < n; ++r) {
        cnt[r] = entry_count(s, r);
        owner_r[r] = owner_i[s.inv_perm[r]];
        warp_r[r] = warp_i[s.inv_perm[r]];
    }
    // cross-CTA dependencies: any direction (the kernel is launched cooperatively,
    // so every CTA is resident; the level order keeps the waits acyclic)
#pragma omp parallel for schedule(static)
    for (int r = 0; r < n; ++r) {
        int f = 0;
        for_each_entry(s, r, [&](int col, double) {
            if (owner_r[col] != owner_r[r]) ++f;
        });
        nforeign[r] = f;
    }

    // 0. one sliced-ELL width W for the whole layout (every chunk padded to W, so
    //    the kernel's row loop is straight-line code): the supported width that
    //    minimises ELL bytes + tail bytes (tail entries weighted double: they run
    //    as a sequential loop)
    {
        const int cand[] = {1, 2, 3, 4, 5, 6, 7, 8, 10, 13, 16};
        std::vector<long long> hist(cfg.max_width + 2, 0);
        int maxc = 0;
        for (int r = 0; r < n; ++r) {
            ++hist[std::min(cnt[r], cfg.max_width + 1)];
            maxc = std::max(maxc, cnt[r]);
        }
        long long best = -1;
        P.max_width = 1;
        for (int wc : cand) {
            if (wc > cfg.max_width) break;
            long long cost = 12LL * wc * n;
            for (int k = wc + 1; k <= cfg.max_width + 1; ++k) cost += 24LL * (k - wc) * hist[k];
            if (best < 0 || cost < best) {
                best = cost;
                P.max_width = wc;
            }
            if (wc >= maxc) break;
        }
    }
    const int W = P.max_width;
    if (big_auto && W <= 4) {
        // narrow rows (z-pencils of 7-point factors): three groups of 4 warps x 4 rows
        // per lane, with one producer and two waiter warps (the prefetch of a chunk
        // then has two chunk periods instead of one): 7-pt 256^3 / 202^3 / 160^3
        // ILU apply 1.050 / 0.770 / 0.559 ms with 8x2x2 -> 0.993 / 0.704 / 0.533 ms
        NW = 4;
        warp_rows = 128;
        K = 3;
        P.group = NW;
        P.groups = K;
        P.warps = NW * K;
        P.rpl = 4;
    }

    // 1. chunk discovery: per level, each CTA's rows (ordered by warp, then by
    //    row, so every warp's rows are one segment), split so that no warp has
    //    more than warp_rows rows in a chunk and by bytes
    struct Chunk { int level, row0, m, w, ntail; };  // rows: cta_rows[c][row0 .. row0+m)
    std::vector<std::vector<Chunk>> per_cta(C);
    std::vector<std::vector<int>> cta_rows(C);
    const int fl_est = 4 | (P.has_out ? 2 : 0);
    if (M) {
        // L's chunks in reverse: U CTA C-1-c takes L CTA c's chunks last to first,
        // each chunk's rows last to first
        std::vector<int> level_of_r(n), r_of_i(n);
        for (int k = 0; k < s.nlev; ++k)
            for (int r = s.level_starts[k]; r < s.level_starts[k + 1]; ++r) level_of_r[r] = k;
        for (int r = 0; r < n; ++r) r_of_i[s.inv_perm[r]] = r;
        std::vector<int> o_of_p(n);
        for (int o = 0; o < n; ++o) o_of_p[M->wpos[o]] = o;
        for (int cl = 0; cl < C; ++cl) {
            const int c = C - 1 - cl;
            int prev_level = -1;
            for (int g = M->cta_chunk0[cl + 1] - 1; g >= M->cta_chunk0[cl]; --g) {
                const int p0 = M->chunk_r0[g], m = M->chunk_r0[g + 1] - p0;
                Chunk ch{-1, static_cast<int>(cta_rows[c].size()), m, W, 0};
                int halo_ub = 0;
                for (int t = m - 1; t >= 0; --t) {
                    const int o = o_of_p[p0 + t];
                    const int r = r_of_i[s.reversed ? n - 1 - o : o];
                    if (ch.level < 0) ch.level = level_of_r[r];
                    if (level_of_r[r] != ch.level) throw std::invalid_argument("wave mirror: chunk spans levels");
                    ch.ntail += std::max(0, cnt[r] - W);
                    halo_ub += nforeign[r];
                    cta_rows[c].push_back(r);
                }
                if (ch.level <= prev_level) throw std::invalid_argument("wave mirror: levels do not rise");
                prev_level = ch.level;
                const int fl = fl_est | (ch.ntail > 0 ? 1 : 0);
                if (m > NW * warp_rows ||
                    wave_region_bytes(m, halo_ub, wave_sections(m, W, NW, halo_ub, ch.ntail, fl).end) > cfg.max_bytes)
                    throw std::invalid_argument("wave mirror: chunk exceeds the solver shape");
                const int pw = (m + NW - 1) / NW;
                for (int t = 0; t < m; ++t) warp_r[cta_rows[c][ch.row0 + t]] = t / pw;
                per_cta[c].push_back(ch);
            }
        }
    } else {
        std::vector<std::vector<int>> bucket(C);
        for (int k = 0; k < s.nlev; ++k) {
            for (int r = s.level_starts[k]; r < s.level_starts[k + 1]; ++r) bucket[owner_r[r]].push_back(r);
            for (int c = 0; c < C; ++c) {
                auto& B = bucket[c];
                if (B.empty()) continue;
                if (!lockstep)
                    std::stable_sort(B.begin(), B.end(), [&](int x, int y) { return warp_r[x] < warp_r[y]; });
                std::size_t u = 0;
                while (u < B.size()) {
                    Chunk ch{k, static_cast<int>(cta_rows[c].size()), 0, W, 0};
                    int halo_ub = 0, cur_w = -1, cur_cnt = 0;
                    while (u < B.size()) {
                        const int r = B[u];
                        const int t2 = ch.ntail + std::max(0, cnt[r] - W);
                        const int h2 = halo_ub + nforeign[r];
                        const int fl = fl_est | (t2 > 0 ? 1 : 0);
                        const int wcnt = warp_r[r] == cur_w ? cur_cnt + 1 : 1;
                        const int bytes =
                            wave_region_bytes(ch.m + 1, h2, wave_sections(ch.m + 1, W, NW, h2, t2, fl).end);
                        const bool full = lockstep ? ch.m >= NW * warp_rows : wcnt > warp_rows;
                        if (ch.m > 0 && (full || bytes > cfg.max_bytes)) break;
                        cur_w = warp_r[r];
                        cur_cnt = wcnt;
                        ch.ntail = t2;
                        halo_ub = h2;
                        cta_rows[c].push_back(r);
                        ++ch.m;
                        ++u;
                    }
                    if (lockstep) {  // deal the chunk's rows to the warps in contiguous segments
                        const int pw = (ch.m + NW - 1) / NW;
                        for (int t = 0; t < ch.m; ++t) warp_r[cta_rows[c][ch.row0 + t]] = t / pw;
                    }
                    per_cta[c].push_back(ch);
                }
                B.clear();
            }
        }
    }

    // 2. sequence numbers, chunk position, ring windows
    std::vector<int> seq_r(n), chunk_pos_r(n);
    std::vector<std::vector<int>> win(C), qend(C);
    P.cta_chunk0.assign(static_cast<std::size_t>(C) + 1, 0);
    for (int c = 0; c < C; ++c) {
        const auto& L = per_cta[c];
        P.cta_chunk0[c + 1] = P.cta_chunk0[c] + static_cast<int>(L.size());
        int q = 0;
        qend[c].resize(L.size());
        for (std::size_t j = 0; j < L.size(); ++j) {
            for (int t = 0; t < L[j].m; ++t) {
                seq_r[cta_rows[c][L[j].row0 + t]] = q + t;
                chunk_pos_r[cta_rows[c][L[j].row0 + t]] = static_cast<int>(j);
            }
            q += L[j].m;
            qend[c][j] = q;
        }
    }
    // x-ring size: the smallest power of two >= 1024 that keeps every own-CTA
    // dependency in shared memory (at most cfg.ring; beyond it the oldest are
    // re-read from x). A smaller ring leaves more shared memory to the chunk
    // regions in flight (7-point 256^3: 8192 -> 2048 entries, -10 %).
    {
        long long dmax = 0;
#pragma omp parallel for schedule(static) reduction(max : dmax)
        for (int r = 0; r < n; ++r) {
            const int c = owner_r[r];
            const long long qe = qend[c][chunk_pos_r[r]];
            for_each_entry(s, r, [&](int col, double) {
                if (owner_r[col] == c) dmax = std::max(dmax, qe - seq_r[col]);
            });
        }
        int r2 = 1024;
        while (r2 < dmax && r2 < cfg.ring) r2 *= 2;
        R = std::min(r2, cfg.ring);
        P.ring = R;
    }
    for (int c = 0; c < C; ++c) {
        const auto& L = per_cta[c];
        // chunks complete in order (lead = 1): ring entries newer than
        // q_end(j) - win(j) cannot have been overwritten yet
        win[c].resize(L.size());
        for (std::size_t j = 0; j < L.size(); ++j) {
            const std::size_t last = std::min(L.size() - 1, j + static_cast<std::size_t>(P.lead) - 1);
            win[c][j] = R - (qend[c][last] - qend[c][j]);
        }
    }
    P.chunks = P.cta_chunk0[C];

    // 2b. halo ring: the values a chunk reads from other CTAs are staged by the
    //     waiters in a shared-memory ring of H entries behind the x ring, at
    //     positions numbered per CTA in chunk order. A waiter stages chunk j only
    //     after chunk j-NS finished (its descriptor slot was recycled), so H must
    //     hold the halos of any NS consecutive chunks.
    std::vector<std::vector<int>> hq0(C);
    std::vector<int> hneed(C, 0);
    {
        std::vector<std::vector<int>> nh(C);
#pragma omp parallel for schedule(dynamic, 1)
        for (int c = 0; c < C; ++c) {
            const auto& L = per_cta[c];
            nh[c].resize(L.size());
            std::vector<int> cols;
            for (std::size_t j = 0; j < L.size(); ++j) {
                cols.clear();
                for (int t = 0; t < L[j].m; ++t) {
                    const int r = cta_rows[c][L[j].row0 + t];
                    if (nforeign[r])
                        for_each_entry(s, r, [&](int col, double) {
                            if (owner_r[col] != c) cols.push_back(col);
                        });
                }
                std::sort(cols.begin(), cols.end());
                nh[c][j] = static_cast<int>(std::unique(cols.begin(), cols.end()) - cols.begin());
            }
        }
        auto need_for = [&](int ns) {
            int worst = 0;
            for (int c = 0; c < C; ++c) {
                const auto& v = nh[c];
                long long sum = 0;
                for (std::size_t j = 0; j < v.size(); ++j) {
                    sum += v[j];
                    if (j >= static_cast<std::size_t>(ns)) sum -= v[j - ns];
                    worst = static_cast<int>(std::max<long long>(worst, sum));
                }
            }
            return worst;
        };
        // a small x ring leaves room for a larger halo ring (27-point slabs: NS 8 -> 16, -3 %)
        const int hmax = R <= 2048 ? 2 * cfg.halo_ring_max : cfg.halo_ring_max;
        // at least two descriptor slots per solver group: with NS == K (a group
        // always refilling its own slot) the kernel deadlocks -- measured with
        // HEC_WAVE_INFLIGHT=4 and four groups, caught by the watchdog
        int ns_min = 4;
        while (ns_min < 2 * P.groups) ns_min *= 2;
        int ns = std::max(P.inflight, ns_min);
        int need = need_for(ns);
        while (need > hmax && ns > ns_min) need = need_for(ns /= 2);
        if (need > hmax)
            throw std::invalid_argument("hec_tri_create: halo ring overflow (wave layout)");
        P.inflight = ns;
        int H = 32;
        while (H < need) H *= 2;
        P.halo_ring = H;
        for (int c = 0; c < C; ++c) {
            hq0[c].resize(nh[c].size());
            int q = 0;
            for (std::size_t j = 0; j < nh[c].size(); ++j) {
                hq0[c][j] = q & (H - 1);
                q += nh[c][j];
            }
        }
    }
    const int H = P.halo_ring;

    // wave order: (CTA, chunk, row in chunk); bp[wave position] = b[bidx[..]]
    std::vector<long long> cta_wbase(static_cast<std::size_t>(C) + 1, 0);
    for (int c = 0; c < C; ++c) cta_wbase[c + 1] = cta_wbase[c] + static_cast<long long>(cta_rows[c].size());
    P.chunk_r0.assign(static_cast<std::size_t>(P.chunks) + 1, n);
    for (int c = 0; c < C; ++c)
        for (std::size_t j = 0; j < per_cta[c].size(); ++j)
            P.chunk_r0[P.cta_chunk0[c] + j] = static_cast<int>(cta_wbase[c] + qend[c][j] - per_cta[c][j].m);
    P.bidx.assign(n, 0);
    P.wpos.assign(n, 0);
    std::vector<int> wpos_r(n);  // reordered row -> wave position
#pragma omp parallel for schedule(static)
    for (int r = 0; r < n; ++r) {
        const int o = sol_index(s, r);
        const int p = static_cast<int>(cta_wbase[owner_r[r]] + seq_r[r]);
        wpos_r[r] = p;
        P.bidx[P.mirrored ? n - 1 - p : p] = s.b_map ? s.b_map[o] : o;
        P.wpos[o] = p;
    }
    // x is written in wave order (coalesced stores; the solution order is one
    // gather pass away): a row older than the ring window is re-read there
    auto x_index = [&](int r) { return wpos_r[r]; };

    // 3. exports: rows read by another CTA get a mailbox id
    std::vector<int> export_id(n, -1);
    {
        std::vector<char> exported(n, 0);
#pragma omp parallel for schedule(static)
        for (int r = 0; r < n; ++r)
            if (nforeign[r])
                for_each_entry(s, r, [&](int col, double) {
                    if (owner_r[col] != owner_r[r]) exported[col] = 1;  // benign race: all write 1
                });
        // ids in wave order: the exported rows of a chunk get consecutive mailboxes
        std::vector<int> r_of_p(n);
        for (int r = 0; r < n; ++r) r_of_p[wpos_r[r]] = r;
        long long e = 0;
        for (int p = 0; p < n; ++p)
            if (exported[r_of_p[p]]) export_id[r_of_p[p]] = static_cast<int>(e++);
        if (e > 0x7ffffffeLL) throw std::overflow_error("hec_tri_create: too many exported rows");
        P.exports = e;
    }

    // 4. emit blobs (parallel over CTAs)
    std::vector<std::vector<unsigned char>> cta_blob(C);
    std::vector<std::vector<int>> cta_span(C);
    std::vector<int> region_max(C, 0);
    std::vector<long long> st_ring(C, 0), st_glob(C, 0), st_halo(C, 0), st_hval(C, 0);
    std::vector<char> seg_bad(C, 0);
#pragma omp parallel for schedule(dynamic, 1)
    for (int c = 0; c < C; ++c) {
        const auto& L = per_cta[c];
        auto& out = cta_blob[c];
        cta_span[c].assign(8 * L.size(), 0);
        std::unordered_map<int, int> halo_of;
        struct HaloUse { int e, t, id; long long at; };  // at >= 0: ELL index, else -1 - tail index
        std::vector<HaloUse> hpend;
        std::vector<int> halo, dep, tptr, tdep;
        std::vector<double> val, tval;
        for (std::size_t j = 0; j < L.size(); ++j) {
            const Chunk& ch = L[j];
            const int m = ch.m, w = ch.w, mp = round_up(m, 4);
            const int q0 = qend[c][j] - m;
            const int lo = qend[c][j] - win[c][j];
            halo_of.clear();
            halo.clear();
            dep.assign(static_cast<std::size_t>(w) * mp, 8 * R);  // padding: the 0.0 slot
            val.assign(static_cast<std::size_t>(w) * mp, 0.0);
            tptr.assign(round_up(mp + 1, 4), 0);
            tdep.clear();
            tval.clear();
            std::vector<unsigned> mask(NW, 0u);
            std::vector<int> t0(NW, -1), t1(NW, -1);
            bool glob = false, any_exp = false;
            for (int t = 0; t < m; ++t) {
                const int r = cta_rows[c][ch.row0 + t];
                const int wr = warp_r[r];
                if (t0[wr] < 0) t0[wr] = t;
                else if (t1[wr] != t) seg_bad[c] = 1;  // warp rows must be contiguous in the chunk
                t1[wr] = t + 1;
                if (export_id[r] >= 0) any_exp = true;
                int e = 0;
                for_each_entry(s, r, [&](int col, double v) {
                    int d;
                    if (owner_r[col] == c) {
                        if (chunk_pos_r[col] >= static_cast<int>(j)) seg_bad[c] = 1;
                        if (warp_r[col] != wr) mask[wr] |= 1u << warp_r[col];
                        if (seq_r[col] >= lo) {
                            d = 8 * (seq_r[col] & (R - 1));
                            ++st_ring[c];
                        } else {
                            d = -(x_index(col) + 1);
                            glob = true;
                            ++st_glob[c];
                        }
                    } else {
                        // staged value: its halo-ring position is assigned below
                        d = 0;
                        hpend.push_back({e, t, export_id[col], e < w ? static_cast<long long>(e) * mp + t
                                                                      : -1 - static_cast<long long>(tdep.size())});
                        ++st_halo[c];
                    }
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
            for (int t = m; t < static_cast<int>(tptr.size()) - 1; ++t) tptr[t + 1] = tptr[t];
            // halo-ring positions in (slot, row) order: the gather of ELL slot u by
            // consecutive lanes then reads consecutive ring entries (no bank conflicts)
            std::stable_sort(hpend.begin(), hpend.end(),
                             [](const HaloUse& x, const HaloUse& y) { return x.e != y.e ? x.e < y.e : x.t < y.t; });
            for (const HaloUse& hu : hpend) {
                auto it = halo_of.find(hu.id);
                int h;
                if (it == halo_of.end()) {
                    h = static_cast<int>(halo.size());
                    halo_of.emplace(hu.id, h);
                    halo.push_back(hu.id);
                } else {
                    h = it->second;
                }
                const int d = 8 * (R + 1 + ((hq0[c][j] + h) & (H - 1)));
                if (hu.at >= 0) dep[static_cast<std::size_t>(hu.at)] = d;
                else tdep[static_cast<std::size_t>(-1 - hu.at)] = d;
            }
            hpend.clear();
            const int nhalo = static_cast<int>(halo.size());
            const int ntail = static_cast<int>(tdep.size());
            st_hval[c] += nhalo;
            (void)any_exp;  // the export list is always present (-1 = row not exported)
            const long long wpos = cta_wbase[c] + q0;  // wave position of the chunk's first row
            bool unit = true;  // every diagonal exactly 1.0 (ILU(0) L): no diag section, no division
            for (int t = 0; t < m && unit; ++t) {
                const int r = cta_rows[c][ch.row0 + t];
                unit = s.csr_vals[s.csr_rp[r + 1] - 1] == 1.0 && !std::signbit(s.csr_vals[s.csr_rp[r + 1] - 1]);
            }
            // the chunk's right-hand side in bp: [wpos, wpos + m), or for a mirrored
            // layout [n - wpos - m, n - wpos) read backwards; copies start 16-byte aligned
            const long long bsrc = P.mirrored ? n - wpos - m : wpos;
            const int flags = (ntail > 0 ? 1 : 0) | (P.has_out ? 2 : 0) | 4 | (glob ? 8 : 0) | (nhalo > 0 ? 16 : 0) |
                              ((bsrc & 1) ? 32 : 0) | (unit ? 64 : 0) | (P.mirrored ? 128 : 0);
            const WaveSections sec = wave_sections(m, w, NW, nhalo, ntail, flags);
            const int region = wave_region_bytes(m, nhalo, sec.end);
            const std::size_t base = out.size();
            out.resize(base + round_up(sec.end, 16), 0);
            unsigned char* b = out.data() + base;
            const WaveHeader hdr{m, mp, q0, flags, nhalo, sec.halo, sec.tptr, hq0[c][j], static_cast<int>(wpos), 0, 0, 0};
            std::memcpy(b, &hdr, sizeof(hdr));
            for (int wi = 0; wi < NW; ++wi) {
                const unsigned a = t0[wi] < 0 ? 0u : (static_cast<unsigned>(t0[wi]) | (static_cast<unsigned>(t1[wi]) << 16));
                std::memcpy(b + sec.seg + 8 * wi, &a, 4);
                std::memcpy(b + sec.seg + 8 * wi + 4, &mask[wi], 4);
            }
            if (nhalo) std::memcpy(b + sec.halo, halo.data(), 4 * nhalo);
            auto put_i = [&](int off, int idx, int v) { std::memcpy(b + off + 4 * idx, &v, 4); };
            auto put_d = [&](int off, int idx, double v) { std::memcpy(b + off + 8 * idx, &v, 8); };
            int ebase = -1;
            unsigned ewords = 0;
            for (int t = 0; t < m; ++t) {
                const int r = cta_rows[c][ch.row0 + t];
                const int o = sol_index(s, r);
                if (!unit) {
                    // RN(1/d): IEEE division on the host is the correctly rounded
                    // reciprocal __drcp_rn would give (the kernel uses it only while
                    // |d| is inside the Markstein guard, where it is normal)
                    const double d = s.csr_vals[s.csr_rp[r + 1] - 1];
                    put_d(sec.diag, t, d);
                    put_d(sec.diag + 8 * mp, t, 1.0 / d);
                }
                if (flags & 2) put_i(sec.oidx, t, s.out_map[o]);
                if (export_id[r] >= 0) {  // consecutive ids inside the chunk (wave order)
                    if (ebase < 0) ebase = export_id[r];
                    unsigned mask;
                    std::memcpy(&mask, b + sec.exp + 16 + 8 * (t / 32), 4);
                    mask |= 1u << (t % 32);
                    std::memcpy(b + sec.exp + 16 + 8 * (t / 32), &mask, 4);
                    ++ewords;
                }
            }
            put_i(sec.exp, 0, ebase < 0 ? 0 : ebase);
            for (int q = 0, pre = 0; q < (mp + 31) / 32; ++q) {  // prefix counts per 32-row word
                unsigned mask;
                std::memcpy(&mask, b + sec.exp + 16 + 8 * q, 4);
                std::memcpy(b + sec.exp + 16 + 8 * q + 4, &pre, 4);
                pre += __builtin_popcount(mask);
            }
            (void)ewords;
            if (!unit)
                for (int t = m; t < mp; ++t) {  // padded rows: harmless values
                    put_d(sec.diag, t, 1.0);
                    put_d(sec.diag + 8 * mp, t, 1.0);
                }
            std::memcpy(b + sec.val, val.data(), 8 * val.size());
            if ((flags & 9) == 0) {  // 16-bit ring slots (byte offset / 8 < 2^16 for R + 1 + H <= 2^16)
                for (std::size_t k = 0; k < dep.size(); ++k) {
                    const uint16_t v = static_cast<uint16_t>(dep[k] >> 3);
                    std::memcpy(b + sec.dep + 2 * k, &v, 2);
                }
            } else {
                std::memcpy(b + sec.dep, dep.data(), 4 * dep.size());
            }
            if (flags & 1) {
                std::memcpy(b + sec.tptr, tptr.data(), 4 * tptr.size());
                std::memcpy(b + sec.tval, tval.data(), 8 * tval.size());
                std::memcpy(b + sec.tdep, tdep.data(), 4 * tdep.size());
            }
            region_max[c] = std::max(region_max[c], region);
            int* sp = &cta_span[c][8 * j];
            sp[0] = static_cast<int>(base / 16);  // CTA-relative for now
            sp[1] = round_up(sec.end, 16);
            sp[2] = region;
            sp[3] = static_cast<int>(bsrc);  // the producer copies from bp + (sp[3] & ~1)
            sp[4] = wave_b_area(m);
            sp[5] = round_up(8 * (m + static_cast<int>(bsrc & 1)), 16);
        }
    }
    for (int c = 0; c < C; ++c)
        if (seg_bad[c]) throw std::invalid_argument("hec_tri_create: dependency order violates the level schedule");

    // 4b. shared-memory placement of every chunk's region, decided here so the
    //     device producer only waits and copies. The regions form a byte ring of
    //     buf_bytes; chunks are released in order (chunk j completes after j-1),
    //     so a region may reuse the space of chunks up to `wait` once that chunk
    //     is released; `wait` >= j - NS also recycles the descriptor slot.
    {
        const int x_end = cfg.ctrl_bytes + 8 * (R + 1 + P.halo_ring);
        P.buf_off = round_up(x_end, 128);
        P.buf_bytes = (cfg.smem_bytes - P.buf_off) / 16 * 16;
        int rmax = 0;
        for (int c = 0; c < C; ++c) rmax = std::max(rmax, region_max[c]);
        if (cfg.smem_bytes > 0 && 2 * rmax > P.buf_bytes)
            throw std::invalid_argument("hec_tri_create: chunk regions exceed shared memory (wave layout)");
        const int B = P.buf_bytes, NS = P.inflight;
#pragma omp parallel for schedule(dynamic, 1)
        for (int c = 0; c < C; ++c) {
            const int nc = static_cast<int>(per_cta[c].size());
            std::vector<int> start(nc), end(nc);
            int head = 0, oldest = 0;
            for (int j = 0; j < nc; ++j) {
                int* sp = &cta_span[c][8 * j];
                const int need = sp[2];
                int wait = j - NS;
                oldest = std::max(oldest, j - NS + 1);
                int pos;
                for (;;) {
                    if (oldest == j) {
                        pos = 0;
                        break;
                    }
                    const int tail = start[oldest];
                    if (head >= tail) {
                        if (head + need <= B) { pos = head; break; }
                        if (need < tail) { pos = 0; break; }
                    } else if (head + need < tail) {
                        pos = head;
                        break;
                    }
                    wait = std::max(wait, oldest);
                    ++oldest;
                }
                start[j] = pos;
                end[j] = pos + need;
                head = pos + need;
                // the producer warps take chunks round robin, so this chunk must itself
                // wait for the newest older chunk whose space it reuses
                for (int i = j - 1; i > wait; --i)
                    if (pos < end[i] && start[i] < pos + need) {
                        wait = i;
                        break;
                    }
                sp[2] = pos;
                sp[6] = wait;  // < 0: nothing to wait for
                // invariant: disjoint from every chunk not yet known to be released
                for (int i = std::max(0, wait + 1); i < j; ++i)
                    if (pos < end[i] && start[i] < pos + need)
                        throw std::logic_error("wave layout: region placement overlap");
            }
        }
    }

    // 5. concatenate CTA streams
    std::size_t total = 0;
    std::vector<std::size_t> cta_base(C);
    for (int c = 0; c < C; ++c) {
        cta_base[c] = total;
        total += cta_blob[c].size();
    }
    if (total / 16 > 0x7fffffffULL) throw std::overflow_error("hec_tri_create: layout exceeds 32 GiB");
    P.blob.resize(total);
    P.span.assign(8 * static_cast<std::size_t>(P.chunks), 0);
    for (int c = 0; c < C; ++c) {
        std::memcpy(P.blob.data() + cta_base[c], cta_blob[c].data(), cta_blob[c].size());
        std::vector<unsigned char>().swap(cta_blob[c]);
        for (int j = 0; j < P.cta_chunk0[c + 1] - P.cta_chunk0[c]; ++j) {
            const int g = P.cta_chunk0[c] + j;
            for (int k = 0; k < 8; ++k) P.span[8 * g + k] = cta_span[c][8 * j + k];
            P.span[8 * g] += static_cast<int>(cta_base[c] / 16);
        }
        P.max_region = std::max(P.max_region, region_max[c]);
        P.ring_deps += st_ring[c];
        P.global_deps += st_glob[c];
        P.halo_deps += st_halo[c];
        P.halo_values += st_hval[c];
    }
    return P;
}

// ---------------------------------------------------------------- COLUMNS ----
ColLayout build_columns(const TriSource& s, const ColConfig& cfg) {
    validate(s);
    if (s.b_map || s.out_map) throw std::invalid_argument("columns: RAS maps");
    const GridGeom g = detect_grid(s);
    const int n = s.n;
    if (!g.ok || static_cast<long long>(g.nx) * g.ny * g.nz != n) throw std::invalid_argument("columns: no grid");
    const int nx = g.nx, ny = g.ny, nz = g.nz, plane = nx * ny;
    // every row: entries among (x-1), (y-1), (z-1) only, in any order; codes per entry
    std::vector<int> r_of(n);
    for (int r = 0; r < n; ++r) r_of[s.inv_perm[r]] = r;
    // rank[i][dir]: position of the entry towards neighbour dir in row i's solve
    // order (-1: absent). The kernel subtracts the present entries in one order
    // shared by all rows, so every row must agree with it.
    std::vector<unsigned char> code(n, 0);  // presence mask: 1 left (x-1), 2 down (y-1), 4 back (z-1)
    std::vector<signed char> seq(3 * static_cast<std::size_t>(n), -1);
    int bad = 0, nonunit = 0;
#pragma omp parallel for schedule(static) reduction(+ : bad, nonunit)
    for (int i = 0; i < n; ++i) {
        const int r = r_of[i];
        const int x = i % nx, y = (i / nx) % ny, z = i / plane;
        int u = 0;
        unsigned m = 0;
        bool ok = true;
        for_each_entry(s, r, [&](int col, double) {
            const int d = i - s.inv_perm[col];
            int dir = -1;
            if (d == 1 && x > 0) dir = 0;
            else if (d == nx && y > 0) dir = 1;
            else if (d == plane && z > 0) dir = 2;
            if (dir < 0 || u >= 3 || (m >> dir) & 1u) {
                ok = false;
                return;
            }
            m |= 1u << dir;
            seq[3 * static_cast<std::size_t>(i) + u] = static_cast<signed char>(dir);
            ++u;
        });
        if (!ok) ++bad;
        code[i] = static_cast<unsigned char>(m);
        const double dg = s.csr_vals[s.csr_rp[r + 1] - 1];
        if (!(dg == 1.0 && !std::signbit(dg))) ++nonunit;
    }
    if (bad) throw std::invalid_argument("columns: not a 7-point grid factor");
    int order[3] = {-1, -1, -1};  // the common entry order (directions), from a row with all three
    for (int i = 0; i < n && order[0] < 0; ++i)
        if (code[i] == 7)
            for (int u = 0; u < 3; ++u) order[u] = seq[3 * static_cast<std::size_t>(i) + u];
    if (order[0] < 0) throw std::invalid_argument("columns: no interior row");
    int pos[3];
    for (int u = 0; u < 3; ++u) pos[order[u]] = u;
#pragma omp parallel for schedule(static) reduction(+ : bad)
    for (int i = 0; i < n; ++i) {  // present entries in increasing common position
        int prev = -1;
        for (int u = 0; u < 3; ++u) {
            const int d = seq[3 * static_cast<std::size_t>(i) + u];
            if (d < 0) break;
            if (pos[d] <= prev) ++bad;
            prev = pos[d];
        }
    }
    if (bad) throw std::invalid_argument("columns: rows disagree on the entry order");
    ColLayout P;
    P.n = n;
    P.nx = nx;
    P.ny = ny;
    P.nz = nz;
    P.nlev = nx + ny + nz - 2;
    P.unit = nonunit == 0;
    P.order = order[0] | order[1] << 2 | order[2] << 4;
    constexpr int SX = ColLayout::SX;
    int SY = 4;
    if (cfg.mirror) {
        const ColMirror& m = *cfg.mirror;
        P.rpl = m.rpl;
        SY = 4 * P.rpl;
        if (m.nx != nx || m.ny != ny || m.nz != nz || !s.reversed) throw std::invalid_argument("columns: no mirror");
        P.WX = m.WX;
        P.WY = m.WY;
        P.PX = m.PX;
        P.PY = m.PY;
        P.ox = m.PX * SX * m.WX - nx - m.ox;
        P.oy = m.PY * SY * m.WY - ny - m.oy;
        P.mirrored = true;
    } else {
        // tiling: one CTA per SM at most. A level costs a warp ~250 cycles of
        // latency, and the SM has to stream the CTA's row data (~41 bytes a column,
        // ~60 bytes / cycle); each CTA boundary a wavefront crosses adds ~2000
        // cycles of lag
        // shapes (warps, columns per lane): one lane-column per level costs ~20 cycles of a
        // warp's dependent instruction chain, a level ~150 more; each CTA boundary a
        // wavefront crosses adds ~2000 cycles of lag; the SM streams ~41 bytes a column
        // (~60 bytes / cycle)
        double best = 1e300;
        const int shapes[][2] = {{16, 1}, {8, 2}, {4, 4}, {4, 1}, {1, 4}};
        for (const auto& sh : shapes) {
            const int nw = sh[0], rp = sh[1];
            if (cfg.warps > 0 && nw != cfg.warps) continue;
            if (cfg.rpl > 0 && rp != cfg.rpl) continue;
            for (int wx = 1; wx <= nw; wx *= 2) {
                const int wy = nw / wx;
                const int tx = SX * wx, ty = 4 * rp * wy;
                const int px = (nx + tx - 1) / tx, py = (ny + ty - 1) / ty;
                if (static_cast<long long>(px) * py > cfg.ctas) continue;
                const double per_level = std::max({150.0 + 80.0 * rp, 41.0 * tx * ty / 60.0});
                const double est = P.nlev * per_level + 2000.0 * (px + py - 2);
                if (est < best) {
                    best = est;
                    P.WX = wx;
                    P.WY = wy;
                    P.PX = px;
                    P.PY = py;
                    P.rpl = rp;
                }
            }
        }
        SY = 4 * P.rpl;
        if (best >= 1e300) throw std::invalid_argument("columns: no tiling fits the CTA count");
    }
    const int TX = SX * P.WX, TY = SY * P.WY, C = P.PX * P.PY;
    P.ctas = C;
    P.warps = P.WX * P.WY;
    P.lanes = 32 * P.rpl * P.warps;  // slots per level
    const int NS = P.lanes;
    P.block_bytes = round_up((P.unit ? 24 : 40) * NS + NS, 16);
    const int per_level = P.block_bytes + 8 * NS;
    P.ring = cfg.smem_bytes > 0 ? std::min(cfg.ring_max, (cfg.smem_bytes - kColCtrlBytes) / per_level) : 8;
    if (P.ring < 3) throw std::invalid_argument("columns: level blocks exceed shared memory");
    P.cta.assign(4 * static_cast<std::size_t>(C), 0);
    long long slot = 0, blk = 0;
    for (int c = 0; c < C; ++c) {
        const int px = c % P.PX, py = c / P.PX;
        const int xs = std::max(0, px * TX - P.ox), xe = std::min(nx, (px + 1) * TX - P.ox);
        const int ys = std::max(0, py * TY - P.oy), ye = std::min(ny, (py + 1) * TY - P.oy);
        if (xs >= xe || ys >= ye) throw std::invalid_argument("columns: empty tile");
        const int l0 = xs + ys, nl = (xe - 1) + (ye - 1) + (nz - 1) - l0 + 1;
        if (slot / NS > INT32_MAX || blk > INT32_MAX) throw std::overflow_error("columns: layout too large");
        P.cta[4 * c] = l0;
        P.cta[4 * c + 1] = nl;
        P.cta[4 * c + 2] = static_cast<int>(slot / NS);
        P.cta[4 * c + 3] = static_cast<int>(blk);
        slot += static_cast<long long>(nl) * NS;
        blk += nl;
    }
    if (slot > INT32_MAX - 64) throw std::overflow_error("columns: more than 2^31 slots");
    if (cfg.mirror && slot != cfg.mirror->slots) throw std::invalid_argument("columns: mirror slot count");
    P.slots = slot;
    P.total_levels = blk;
    P.mailboxes = static_cast<long long>(C) * (TX + TY) * nz;
    P.blocks.assign(static_cast<std::size_t>(blk) * P.block_bytes, 0);
    P.bidx.assign(static_cast<std::size_t>(slot), 0);
    P.wpos.assign(n, 0);
    const int off_code = (P.unit ? 24 : 40) * NS;
#pragma omp parallel for schedule(static)
    for (long long b = 0; b < blk; ++b) {  // padding: no entries, diagonal 1
        unsigned char* q = P.blocks.data() + static_cast<std::size_t>(b) * P.block_bytes;
        if (!P.unit)
            for (int k = 0; k < NS; ++k) {
                const double one = 1.0;
                std::memcpy(q + 24 * NS + 8 * k, &one, 8);
                std::memcpy(q + 32 * NS + 8 * k, &one, 8);
            }
    }
#pragma omp parallel for schedule(static)
    for (int i = 0; i < n; ++i) {
        const int r = r_of[i];
        const int x = i % nx, y = (i / nx) % ny, z = i / plane;
        const int ax = x + P.ox, ay = y + P.oy;
        const int px = ax / TX, py = ay / TY, c = py * P.PX + px;
        const int wx = (ax % TX) / SX, lx = ax % SX, wy = (ay % TY) / SY, ly = ay % SY;
        // lane (ly / RPL) * SX + lx owns RPL consecutive columns in y; its slots are consecutive
        const int k = ((wy * P.WX + wx) * 32 + (ly / P.rpl) * SX + lx) * P.rpl + ly % P.rpl;
        const int l = x + y + z - P.cta[4 * c];
        const long long sl = static_cast<long long>(P.cta[4 * c + 2]) * NS + static_cast<long long>(l) * NS + k;
        unsigned char* q = P.blocks.data() + (static_cast<std::size_t>(P.cta[4 * c + 3]) + l) * P.block_bytes;
        int u = 0;
        unsigned m = 0;
        for_each_entry(s, r, [&](int, double v) {  // entry towards neighbour dir -> its common position
            const int p = pos[seq[3 * static_cast<std::size_t>(i) + u]];
            std::memcpy(q + 8 * (static_cast<std::size_t>(p) * NS + k), &v, 8);
            m |= 1u << p;
            ++u;
        });
        q[off_code + k] = static_cast<unsigned char>(m);
        if (!P.unit) {
            const double d = s.csr_vals[s.csr_rp[r + 1] - 1];
            const double rc = 1.0 / d;  // RN(1/d), as __drcp_rn
            std::memcpy(q + 24 * NS + 8 * k, &d, 8);
            std::memcpy(q + 32 * NS + 8 * k, &rc, 8);
        }
        const int o = s.reversed ? n - 1 - i : i;
        P.bidx[static_cast<std::size_t>(sl)] = o;
        P.wpos[o] = static_cast<int>(sl);
    }
    return P;
}

}  // namespace hec::plan
