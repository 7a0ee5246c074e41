/*
 * hec_oracle.c -- TEST INFRASTRUCTURE ONLY. CPU restatement, in plain C, of the
 * reference hecsolve path (arXiv 1606.00541, /root/reference/proj). It is the
 * checker for the B200 library: only tests/, __graft_entry__.smoke() and
 * bench.py's cpu_baseline leg may load it. Nothing in the product links it.
 *
 * Every function cites the reference code it restates. Scalar, single thread,
 * no FMA (build with -ffp-contract=off): the arithmetic order per row is the
 * reference's, so results are bitwise comparable.
 *
 * Pinned against (tests/test_oracle.py): the reference's own known answers
 * (test_triangular.cpp, test_hec.cpp, test_level_schedule.cpp, acceptance.cpp)
 * and golden vectors produced by the reference itself (tests/golden/, made by
 * tests/golden/make_golden.py through oracle/_ref).
 *
 * Conventions: CSR = (n, rp[n+1], ci[nnz], v[nnz]); caller allocates outputs.
 * Return value: >= 0 success (a count where documented), < 0 error code
 * (-1 invalid argument, -4 zero pivot).
 */
#include <math.h>
#include <stdlib.h>
#include <string.h>

#define ORC_EINVAL (-1)
#define ORC_EZERO (-4)

/* level_schedule.cpp:10-26 -- one ascending pass, level = 1 + max dep level. */
int orc_levels(int n, const int* rp, const int* ci, int* level) {
    int nlev = 0;
    for (int i = 0; i < n; ++i) {
        int deep = 0;
        for (int k = rp[i]; k < rp[i + 1]; ++k) {
            const int j = ci[k];
            if (j > i) return ORC_EINVAL;
            if (j < i && level[j] > deep) deep = level[j];
        }
        level[i] = deep + 1;
        if (level[i] > nlev) nlev = level[i];
    }
    return nlev;
}

/* level_schedule.cpp:28-58 -- stable counting sort by level. */
int orc_schedule(int n, const int* level, int nlev, int* perm, int* inv_perm, int* starts) {
    for (int k = 0; k <= nlev; ++k) starts[k] = 0;
    for (int i = 0; i < n; ++i) {
        if (level[i] < 1 || level[i] > nlev) return ORC_EINVAL;
        starts[level[i]]++;
    }
    for (int k = 1; k <= nlev; ++k) {
        if (starts[k] == 0) return ORC_EINVAL;
        starts[k] += starts[k - 1];
    }
    int* next = (int*)malloc(sizeof(int) * (nlev > 0 ? nlev : 1));
    for (int k = 0; k < nlev; ++k) next[k] = starts[k];
    for (int i = 0; i < n; ++i) {
        const int r = next[level[i] - 1]++;
        perm[i] = r;
        inv_perm[r] = i;
    }
    free(next);
    return 0;
}

/* level_schedule.cpp:60-89 -- symmetric permutation, rows re-sorted by column. */
void orc_reorder(int n, const int* rp, const int* ci, const double* v, const int* perm,
                 const int* inv_perm, int* orp, int* oci, double* ov) {
    orp[0] = 0;
    for (int r = 0; r < n; ++r) orp[r + 1] = orp[r] + (rp[inv_perm[r] + 1] - rp[inv_perm[r]]);
    for (int r = 0; r < n; ++r) {
        const int i = inv_perm[r];
        int len = 0;
        int* c = oci + orp[r];
        double* x = ov + orp[r];
        for (int k = rp[i]; k < rp[i + 1]; ++k, ++len) { /* insertion sort by new column */
            const int nc = perm[ci[k]];
            const double nv = v[k];
            int u = len;
            while (u > 0 && c[u - 1] > nc) {
                c[u] = c[u - 1];
                x[u] = x[u - 1];
                --u;
            }
            c[u] = nc;
            x[u] = nv;
        }
    }
}

/* triangular.cpp:43-63 -- i -> n-1-i on rows and columns (upper -> lower). */
void orc_reverse(int n, const int* rp, const int* ci, const double* v, int* orp, int* oci, double* ov) {
    orp[0] = 0;
    for (int r = 0; r < n; ++r) orp[r + 1] = orp[r] + (rp[n - r] - rp[n - 1 - r]);
    for (int i = 0; i < n; ++i) {
        int d = orp[n - 1 - i];
        for (int k = rp[i + 1] - 1; k >= rp[i]; --k, ++d) {
            oci[d] = n - 1 - ci[k];
            ov[d] = v[k];
        }
    }
}

static int cmp_int(const void* a, const void* b) {
    const int x = *(const int*)a, y = *(const int*)b;
    return (x > y) - (x < y);
}

/* hec.cpp:11-24 -- automatic width = element n/2 of the sorted counts. */
int orc_hec_width(int n, const int* rp, int triangular, int fixed_width) {
    if (fixed_width >= 0) return fixed_width;
    if (n == 0) return 0;
    int* cnt = (int*)malloc(sizeof(int) * n);
    int mx = 0;
    for (int i = 0; i < n; ++i) {
        cnt[i] = rp[i + 1] - rp[i] - (triangular ? 1 : 0);
        if (cnt[i] > mx) mx = cnt[i];
    }
    qsort(cnt, (size_t)n, sizeof(int), cmp_int);
    int w = cnt[n / 2];
    free(cnt);
    if (w < 0) w = 0;
    if (w > mx) w = mx;
    return w;
}

/* hec.cpp:28-86 -- ELL (column-major, pad = value 0 / column min(i, ncols-1))
 * plus CSR remainder (diagonal reserved in triangular mode). Returns CSR nnz;
 * call with null outputs first to size the CSR part. */
long long orc_hec_fill(int n, int ncols, const int* rp, const int* ci, const double* v, int triangular,
                       int w, int* ell_c, double* ell_v, int* crp, int* cci, double* cv) {
    const int keep = triangular ? 1 : 0;
    long long total = 0;
    for (int i = 0; i < n; ++i) {
        if (triangular && (rp[i + 1] == rp[i] || ci[rp[i + 1] - 1] != i)) return ORC_EINVAL;
        const int cnt = rp[i + 1] - rp[i] - keep;
        const int in_ell = cnt < w ? cnt : w;
        total += (cnt - in_ell) + keep;
    }
    if (!ell_c) return total;
    crp[0] = 0;
    for (int i = 0; i < n; ++i) {
        const int cnt = rp[i + 1] - rp[i] - keep;
        const int in_ell = cnt < w ? cnt : w;
        const int pad = ncols > 0 ? (i < ncols - 1 ? i : ncols - 1) : 0;
        for (int k = 0; k < w; ++k) {
            const size_t s = (size_t)k * n + i;
            ell_c[s] = k < in_ell ? ci[rp[i] + k] : pad;
            ell_v[s] = k < in_ell ? v[rp[i] + k] : 0.0;
        }
        int d = crp[i];
        for (int k = rp[i] + in_ell; k < rp[i + 1]; ++k, ++d) {
            cci[d] = ci[k];
            cv[d] = v[k];
        }
        crp[i + 1] = d;
    }
    return total;
}

/* triangular.cpp:90-135 -- Algorithm 2, one worker: permute in, level sweep
 * (ELL slots, CSR except the last entry, divide by the last entry), permute out.
 * xp starts at zero so padding slots read 0. */
void orc_solve(int n, int reversed, int nlev, const int* starts, const int* perm, int w, const int* ell_c,
               const double* ell_v, const int* crp, const int* cci, const double* cv, const double* b,
               double* x) {
    double* bp = (double*)malloc(sizeof(double) * (n > 0 ? n : 1));
    double* xp = (double*)calloc((size_t)(n > 0 ? n : 1), sizeof(double));
    for (int i = 0; i < n; ++i) bp[perm[reversed ? n - 1 - i : i]] = b[i];
    for (int lev = 0; lev < nlev; ++lev)
        for (int r = starts[lev]; r < starts[lev + 1]; ++r) {
            double acc = bp[r];
            for (int k = 0; k < w; ++k) {
                const size_t s = (size_t)k * n + r;
                acc -= ell_v[s] * xp[ell_c[s]];
            }
            const int last = crp[r + 1] - 1;
            for (int k = crp[r]; k < last; ++k) acc -= cv[k] * xp[cci[k]];
            xp[r] = acc / cv[last];
        }
    for (int i = 0; i < n; ++i) x[i] = xp[perm[reversed ? n - 1 - i : i]];
    free(bp);
    free(xp);
}

/* triangular.cpp:137-152 */
int orc_forward(int n, const int* rp, const int* ci, const double* v, const double* b, double* x) {
    for (int i = 0; i < n; ++i) {
        const int last = rp[i + 1] - 1;
        if (last < rp[i] || ci[last] != i) return ORC_EINVAL;
        double acc = b[i];
        for (int k = rp[i]; k < last; ++k) acc -= v[k] * x[ci[k]];
        x[i] = acc / v[last];
    }
    return 0;
}

/* triangular.cpp:154-169 */
int orc_backward(int n, const int* rp, const int* ci, const double* v, const double* b, double* x) {
    for (int i = n - 1; i >= 0; --i) {
        const int first = rp[i];
        if (rp[i + 1] == first || ci[first] != i) return ORC_EINVAL;
        double acc = b[i];
        for (int k = first + 1; k < rp[i + 1]; ++k) acc -= v[k] * x[ci[k]];
        x[i] = acc / v[first];
    }
    return 0;
}

/* csr.cpp:43-57 */
void orc_spmv(int n, const int* rp, const int* ci, const double* v, const double* x, double* y) {
    for (int i = 0; i < n; ++i) {
        double s = 0.0;
        for (int k = rp[i]; k < rp[i + 1]; ++k) s += v[k] * x[ci[k]];
        y[i] = s;
    }
}

/* ilu.cpp:23-46 -- IKJ on the fixed pattern, in place on v; dpos out.
 * On a zero / missing pivot returns ORC_EZERO with the row in *bad_row. */
int orc_ilu0_inplace(int n, const int* rp, const int* ci, double* v, int* dpos, int* bad_row) {
    int* pos = (int*)malloc(sizeof(int) * (n > 0 ? n : 1));
    for (int j = 0; j < n; ++j) pos[j] = -1;
    int rc = 0;
    for (int i = 0; i < n && rc == 0; ++i) {
        const int rs = rp[i], re = rp[i + 1];
        for (int k = rs; k < re; ++k) pos[ci[k]] = k;
        if (pos[i] < rs) { rc = ORC_EZERO; *bad_row = i; break; }
        dpos[i] = pos[i];
        for (int k = rs; k < re && ci[k] < i; ++k) {
            const int p = ci[k];
            const double m = v[k] / v[dpos[p]];
            v[k] = m;
            for (int t = dpos[p] + 1; t < rp[p + 1]; ++t)
                if (pos[ci[t]] >= rs) v[pos[ci[t]]] -= m * v[t];
        }
        if (v[dpos[i]] == 0.0) { rc = ORC_EZERO; *bad_row = i; break; }
    }
    free(pos);
    return rc;
}

/* precond.cpp:119-145 -- gather, L solve, U solve, restricted scatter. The
 * prepared pair is passed as two orc_solve argument sets. */
void orc_apply(int n, int n_ext, const int* ext_rows, const char* owned,
               int l_nlev, const int* l_starts, const int* l_perm, int l_w, const int* l_ec,
               const double* l_ev, const int* l_rp, const int* l_ci, const double* l_cv,
               int u_nlev, const int* u_starts, const int* u_perm, int u_w, const int* u_ec,
               const double* u_ev, const int* u_rp, const int* u_ci, const double* u_cv,
               const double* r, double* x) {
    double* rh = (double*)malloc(sizeof(double) * (n_ext > 0 ? n_ext : 1));
    double* y = (double*)malloc(sizeof(double) * (n_ext > 0 ? n_ext : 1));
    double* z = (double*)malloc(sizeof(double) * (n_ext > 0 ? n_ext : 1));
    for (int k = 0; k < n_ext; ++k) rh[k] = r[ext_rows[k]];
    orc_solve(n_ext, 0, l_nlev, l_starts, l_perm, l_w, l_ec, l_ev, l_rp, l_ci, l_cv, rh, y);
    orc_solve(n_ext, 1, u_nlev, u_starts, u_perm, u_w, u_ec, u_ev, u_rp, u_ci, u_cv, y, z);
    for (int i = 0; i < n; ++i) x[i] = 0.0;
    for (int k = 0; k < n_ext; ++k)
        if (owned[k]) x[ext_rows[k]] = z[k];
    free(rh);
    free(y);
    free(z);
}

/* poisson.cpp:8-43 -- entries written in ascending column order. Returns nnz
 * (call with rp == NULL to size). */
long long orc_poisson7(int nx, int ny, int nz, int* rp, int* ci, double* v) {
    const long long n = (long long)nx * ny * nz;
    const long long nnz = 7 * n - 2 * ((long long)nx * ny + (long long)ny * nz + (long long)nx * nz);
    if (!rp) return nnz;
    const long long plane = (long long)nx * ny;
    long long at = 0, id = 0;
    rp[0] = 0;
    for (int z = 0; z < nz; ++z)
        for (int y = 0; y < ny; ++y)
            for (int x = 0; x < nx; ++x, ++id) {
                if (z > 0) { ci[at] = (int)(id - plane); v[at++] = -1.0; }
                if (y > 0) { ci[at] = (int)(id - nx); v[at++] = -1.0; }
                if (x > 0) { ci[at] = (int)(id - 1); v[at++] = -1.0; }
                ci[at] = (int)id; v[at++] = 6.0;
                if (x < nx - 1) { ci[at] = (int)(id + 1); v[at++] = -1.0; }
                if (y < ny - 1) { ci[at] = (int)(id + nx); v[at++] = -1.0; }
                if (z < nz - 1) { ci[at] = (int)(id + plane); v[at++] = -1.0; }
                rp[id + 1] = (int)at;
            }
    return nnz;
}

/* gmres.cpp:11-17 -- serial dot. */
double orc_dot(int n, const double* a, const double* b) {
    double s = 0.0;
    for (int i = 0; i < n; ++i) s += a[i] * b[i];
    return s;
}

/* Generators of the configs the reference has no generator for (SURVEY.md
 * 8(d) C2/C3 definitions; the reference's gen_poisson7 pattern, poisson.cpp:8-43,
 * extended). Input data only: used by the golden script and bench.py's
 * reference arm so neither needs the product library. */

/* 27-point: diagonal 26, -1 for every existing neighbour, ascending columns. */
long long orc_poisson27(int nx, int ny, int nz, int* rp, int* ci, double* v) {
    long long at = 0, id = 0;
    if (rp) rp[0] = 0;
    for (int z = 0; z < nz; ++z)
        for (int y = 0; y < ny; ++y)
            for (int x = 0; x < nx; ++x, ++id) {
                for (int dz = -1; dz <= 1; ++dz)
                    for (int dy = -1; dy <= 1; ++dy)
                        for (int dx = -1; dx <= 1; ++dx) {
                            if (z + dz < 0 || z + dz >= nz || y + dy < 0 || y + dy >= ny || x + dx < 0 ||
                                x + dx >= nx)
                                continue;
                            if (rp) {
                                ci[at] = (int)(id + dx + (long long)nx * (dy + (long long)ny * dz));
                                v[at] = (dx == 0 && dy == 0 && dz == 0) ? 26.0 : -1.0;
                            }
                            ++at;
                        }
                if (rp) rp[id + 1] = (int)at;
            }
    return at;
}

/* std::mt19937_64 (the C++ standard's parameters), for gen_reservoir7's draws. */
typedef struct { unsigned long long mt[312]; int i; } orc_mt64;
static void mt64_seed(orc_mt64* s, unsigned long long seed) {
    s->mt[0] = seed;
    for (int i = 1; i < 312; ++i)
        s->mt[i] = 6364136223846793005ULL * (s->mt[i - 1] ^ (s->mt[i - 1] >> 62)) + (unsigned long long)i;
    s->i = 312;
}
static unsigned long long mt64_next(orc_mt64* s) {
    if (s->i >= 312) {
        for (int k = 0; k < 312; ++k) {
            const unsigned long long y = (s->mt[k] & 0xFFFFFFFF80000000ULL) | (s->mt[(k + 1) % 312] & 0x7FFFFFFFULL);
            s->mt[k] = s->mt[(k + 156) % 312] ^ (y >> 1) ^ ((y & 1ULL) ? 0xB5026F5AA96619E9ULL : 0ULL);
        }
        s->i = 0;
    }
    unsigned long long x = s->mt[s->i++];
    x ^= (x >> 29) & 0x5555555555555555ULL;
    x ^= (x << 17) & 0x71D67FFFEDA60000ULL;
    x ^= (x << 37) & 0xFFF7EEE000000000ULL;
    x ^= x >> 43;
    return x;
}

/* Reservoir-style 7-point: k_c = 10^(sigma (2u-1)), u =
 * (mt19937_64() >> 11) 2^-53 in cell order; vertical faces use kz_ratio k;
 * interior face T = 2ab/(a+b), a boundary face adds the cell's own k to the
 * diagonal; A_ii = sum of the six T, A_ij = -T. Pattern = gen_poisson7. */
long long orc_reservoir7(int nx, int ny, int nz, double sigma, double kz_ratio, unsigned long long seed, int* rp,
                         int* ci, double* v) {
    const long long n = (long long)nx * ny * nz;
    const long long nnz = 7 * n - 2 * ((long long)nx * ny + (long long)ny * nz + (long long)nx * nz);
    if (!rp) return nnz;
    double* k = (double*)malloc(sizeof(double) * (size_t)(n > 0 ? n : 1));
    orc_mt64* s = (orc_mt64*)malloc(sizeof(orc_mt64));
    mt64_seed(s, seed);
    for (long long c = 0; c < n; ++c) {
        const double u = (double)(mt64_next(s) >> 11) * 0x1.0p-53;
        k[c] = pow(10.0, sigma * (2.0 * u - 1.0));
    }
    free(s);
    const long long plane = (long long)nx * ny;
    long long at = 0, id = 0;
    rp[0] = 0;
    for (int z = 0; z < nz; ++z)
        for (int y = 0; y < ny; ++y)
            for (int x = 0; x < nx; ++x, ++id) {
                const double kh = k[id], kv = kz_ratio * k[id];
                const int has[6] = {z > 0, y > 0, x > 0, x + 1 < nx, y + 1 < ny, z + 1 < nz};
                const long long nb[6] = {id - plane, id - nx, id - 1, id + 1, id + nx, id + plane};
                double t[6], d = 0.0;
                for (int f = 0; f < 6; ++f) {
                    const int vert = (f == 0 || f == 5);
                    const double own = vert ? kv : kh;
                    if (has[f]) {
                        const double other = vert ? kz_ratio * k[nb[f]] : k[nb[f]];
                        t[f] = 2.0 * own * other / (own + other);
                    } else {
                        t[f] = own;
                    }
                }
                for (int f = 0; f < 6; ++f) d += t[f];
                for (int f = 0; f < 3; ++f)
                    if (has[f]) { ci[at] = (int)nb[f]; v[at++] = -t[f]; }
                ci[at] = (int)id; v[at++] = d;
                for (int f = 3; f < 6; ++f)
                    if (has[f]) { ci[at] = (int)nb[f]; v[at++] = -t[f]; }
                rp[id + 1] = (int)at;
            }
    free(k);
    return nnz;
}
