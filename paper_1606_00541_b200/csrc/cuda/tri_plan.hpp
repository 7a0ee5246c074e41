#pragma once
// Host-side construction of the B200 device layouts for one prepared triangle.
//
// Index spaces:
//   r  reordered row (level-major), the reference's HEC row index
//   i  lower-frame row = schedule.inv_perm[r]
//   o  solution index = reversal ? n-1-i : i  (the reference's output order)
// Every dependency column of the reference HEC (a reordered index) is rewritten
// as the solution index of that row, so the device never permutes vectors:
// b is gathered and x scattered directly in the original ordering
// (reference permute-in/out passes, proj/src/triangular.cpp:110-111,131-132,
// are folded into the row loads/stores).

#include <cstdint>
#include <vector>

namespace hec::plan {

// The fields of hec::PreparedTriangular that solve() reads
// (reference proj/src/triangular.cpp:96-103), plus optional RAS maps.
struct TriSource {
    int n = 0;
    bool reversed = false;
    int nlev = 0;
    const int* level_starts = nullptr;  // nlev + 1
    const int* inv_perm = nullptr;      // n
    int ell_width = 0;
    const int* ell_cols = nullptr;      // ell_width * n, column-major
    const double* ell_vals = nullptr;
    const int* csr_rp = nullptr;        // n + 1
    const int* csr_cols = nullptr;
    const double* csr_vals = nullptr;
    const int* b_map = nullptr;         // o -> index into the input vector (null: o)
    const int* out_map = nullptr;       // o -> index into a second output (-1: none)
};

void validate(const TriSource& s);  // throws std::invalid_argument

// ---------------------------------------------------------------- LEVELS ----
// One launch per level, thread per reordered row. ELL kept column-major with
// ld = round_up(n, 32) so every slot column starts 128-byte aligned for both
// the int32 and the FP64 arrays; padding slots carry dependency -1 (skipped).
struct LevelLayout {
    int n = 0, ld = 0, width = 0, nlev = 0;
    std::vector<int> level_starts;
    std::vector<int> xidx, bidx, oidx;       // per reordered row
    std::vector<int> ell_dep;                // width * ld
    std::vector<double> ell_val;             // width * ld
    std::vector<double> diag;                // n
    std::vector<int> tail_rp, tail_dep;      // CSR remainder without the diagonal
    std::vector<double> tail_val;
    // rows whose CSR remainder has >= long_min entries, level by level: solved by
    // a warp each (parallel loads and products, the differences in stored order)
    int long_min = 0;                        // 0: no warp rows
    std::vector<int> long_rows, long_starts; // long_starts: nlev + 1
};
constexpr int kLongRowMin = 32;  // measured: 40-entry remainders 0.42 -> 0.19 ms (tools/long_rows.py)
LevelLayout build_levels(const TriSource& s, int long_min = kLongRowMin);

// ------------------------------------------------------------------ WAVE ----
// Persistent wavefront kernel (one CTA per SM, cooperative launch so every
// CTA is resident). Row ownership, in the lower frame:
//  * default: CTA c owns rows [c*per, (c+1)*per) ("slabs");
//  * when the row index follows the levels (an RCM-like ordering), slabs would
//    hand each CTA a few consecutive levels only: then "strips" -- each CTA
//    owns the c-th fraction of every level;
//  * when the factor is recognised as a structured nx x ny x nz grid in natural
//    order (its dependency offsets are {1, nx, nx*ny} or the 27-point set),
//    CTA (px, py) owns the z-pencil of an x-y tile. A wavefront then crosses
//    ~sqrt(C) CTA boundaries per direction instead of C.
// The CTA's rows of one level form a "chunk" (split at the solver shape's
// capacity G x 32 x RPL rows and at max_bytes of shared memory); rows are
// numbered in "wave order" (CTA, chunk, row), the right-hand side is permuted
// into that order and x is written in it.
//
// Synchronisation replaces the reference's per-level barrier
// (triangular.cpp:128) by dataflow:
//   * inside a CTA: K groups of G solver warps take the chunks round robin; a
//     named barrier orders chunk j after chunk j-1, so chunks complete in order
//     (lead = 1: an own row is safe in the x ring while it is newer than
//     q_end(j) - R);
//   * across CTAs: rows read by another CTA are "exported": the producing
//     thread writes the value into a 16-byte mailbox as two 8-byte words
//     {lo32 | epoch, hi32 | epoch}; the consumer's waiter warps poll until
//     both words carry the current solve's epoch, then stage the value in the
//     shared-memory halo ring. Epochs advance per solve, so mailboxes are
//     never reset.
//
// Blob of one chunk (16-byte aligned, moved by one cp.async.bulk); mp =
// round_up(m, 4), W = the layout's sliced-ELL width, G = warps per chunk. Every
// section before the tail sits at an offset computable from mp alone:
//   WaveHeader (48 B)  {m, mp, q0, flags}, {nhalo, halo list, tail, hq0}, {r0, 0, 0, 0}
//   uint2 seg[G]         per warp of the group: (t0 | t1 << 16, 0)
//   double diag[mp], rcp[mp]  the diagonal and RN(1/diag), computed here once
//                        instead of per solve (absent when every diagonal of the
//                        chunk is 1.0, flags&64: x = num * 1.0, bitwise num / 1.0;
//                        the ILU(0) L factor)
//   double val[W][mp]    sliced ELL, slot-major (padding: value 0, dep -> 0.0 slot)
//   dep[W][mp]           fast chunks (no tail, no x re-reads, flags & 9 == 0):
//                        uint16 slot s of the x-ring array (own row q mod R,
//                        the 0.0 slot R, staged value R + 1 + pos mod H), padded
//                        to 16 bytes; otherwise int32 d: d >= 0 byte offset 8 s,
//                        d < 0: x[-d-1] (wave order)
//   exports              int base, 3 pad; uint2 {mask, prefix}[ceil(mp/32)]: row t
//                        is exported iff bit t%32 of mask[t/32] is set, to mailbox
//                        base + prefix + popc(lower bits) (mailbox ids follow the
//                        wave order, so a chunk's exported rows are consecutive);
//   (oidx[mp] if flags&2); row t's x goes to wave position r0 + t, so no per-row
//   solution index is stored
//   if flags&1: int tptr[mp+1 -> mult of 4], double tval[ntail -> even], int tdep[ntail -> mult of 4]
//   int halo[nhalo -> mult of 4]   export ids whose mailboxes this chunk stages,
//                                  in (ELL slot, row) order of first use
// The right-hand side arrives permuted into wave order (bp[p] = b[bidx[p]],
// one coalesced pass before the solve), so a chunk's b values are one
// contiguous range that a second bulk copy moves next to the blob. The
// shared-memory region of a chunk is [b: 8*mb][blob], mb = round_up(m + 1, 4);
// b starts one element in when r0 is odd (flags&32, the copy source is rounded
// down to 16 bytes). Regions are placed in the byte ring by the host (span).
// The chunk structure of another layout over the same solution indices (the L
// factor of an ILU pair), for building the U layout as its exact mirror: U's
// wave order is L's reversed, so U's right-hand side -- L's output -- is L's
// wave-ordered output read backwards, one contiguous range per chunk (no gather
// pass between the two solves). SURVEY/DESIGN: valid when every mirrored chunk's
// rows share one U level and the levels rise along each CTA (always so for the
// ILU(0) factors of a symmetric pattern on a natural-order grid); build_wave
// throws std::invalid_argument otherwise.
struct WaveMirror {
    int ctas = 0;
    const int* cta_chunk0 = nullptr;  // ctas + 1
    const int* chunk_r0 = nullptr;    // per chunk: wave position of its first row (chunks + 1 entries)
    const int* wpos = nullptr;        // solution index -> wave position (n)
};

struct WaveConfig {
    int ctas = 148;
    int group = 0;            // solver warps per chunk (G); 0 = auto from the rows per (CTA, level)
    int groups = 4;           // K groups of G warps take the chunks round robin
    int rpl = 2;              // rows per lane (a warp takes up to 32 * rpl rows of a chunk)
    int ring = 8192;          // x ring entries (power of two); slot `ring` holds 0.0
    int inflight = 16;        // max chunks in flight per CTA (descriptor slots)
    int lead = 4;             // a warp starts chunk j only after every warp finished chunk j-lead
    int max_bytes = 40960;    // chunk split: shared-memory region bytes
    int max_width = 16;       // sliced-ELL width cap; longer rows spill to the tail
    int halo_ring_max = 4096; // halo ring entries at most (shared memory)
    int smem_bytes = 0;       // dynamic shared memory per CTA (0: skip the placement check)
    int ctrl_bytes = 1536;    // control block in front of the x ring
    bool pencils = true;      // structured 3-D grid detected: CTAs own z-pencils (see build_wave)
    bool strips = true;       // row index follows the levels: every CTA takes a fraction of each level
    const WaveMirror* mirror = nullptr;  // build the exact mirror of this layout (see WaveMirror)
};

struct WaveLayout {
    int n = 0, nlev = 0, ctas = 0, warps = 0, rpl = 1, ring = 0, inflight = 0, lead = 0;
    int group = 1, groups = 1;            // solver shape: warps = group * groups
    int halo_ring = 32;                   // H: staged-halo ring entries (power of two)
    int buf_off = 0, buf_bytes = 0;       // byte ring of chunk regions (shared-memory offsets)
    int chunks = 0;
    int max_region = 0;                   // bytes of the largest chunk region
    int max_width = 0;                    // sliced-ELL width W of every chunk
    long long exports = 0;                // mailboxes
    bool has_out = false;
    bool pencils = false;                 // CTAs own z-pencils of a detected nx x ny x nz grid
    bool strips = false;                  // every CTA owns a fraction of every level
    int grid_nx = 0, grid_ny = 0;
    std::vector<int> cta_chunk0;          // ctas + 1: chunk range of each CTA
    std::vector<int> wpos;                // solution index -> wave position (where x lands)
    std::vector<int> chunk_r0;            // chunks + 1: wave position of each chunk's first row (+ n)
    bool mirrored = false;                // built as the mirror of another layout: bp runs backwards
                                          //   (bp[n-1-p] feeds wave position p; bidx is indexed that way)
    std::vector<int> span;                // 8 per chunk: blob offset / 16, blob bytes, region position in
                                          //   the byte ring, r0, b area bytes, b copy bytes, chunk to wait
                                          //   for (released before the region is reused; < 0: none), 0
    std::vector<int> bidx;                // n: input index of reordered row r (bp[r] = b[bidx[r]])
    std::vector<unsigned char> blob;      // all chunk blobs, 16-byte aligned
    long long ring_deps = 0, global_deps = 0, halo_deps = 0, halo_values = 0;
};
WaveLayout build_wave(const TriSource& s, const WaveConfig& cfg);

struct WaveSections {
    int seg, diag, val, dep, exp, oidx, tptr, tval, tdep, halo, end;
};

// First 32 bytes of every blob; read by the kernel as-is.
struct WaveHeader {
    int m, mp, q0, flags;          // flags: 1 tail, 2 out-map, 8 global deps, 16 halo, 32 odd r0,
                                   //        64 unit diagonal (no diag section, no division),
                                   //        128 right-hand side staged backwards (mirrored layout)
    int nhalo, halo, tptr, hq0;    // halo id list / tail offsets, halo ring position of the first staged value
    int r0, pad0, pad1, pad2;      // wave position of the chunk's first row (where its x values go)
};
static_assert(sizeof(WaveHeader) == 48, "wave header is three 16-byte words");
constexpr int kWaveHeaderBytes = 48;

inline int round_up(int v, int m) { return (v + m - 1) / m * m; }
// Offsets of the fixed sections (also computed this way on the device).
inline WaveSections wave_sections(int m, int w, int nw, int nhalo, int ntail, int flags) {
    WaveSections b{};
    const int mp = round_up(m, 4);
    int at = kWaveHeaderBytes;
    b.seg = at;   at += round_up(8 * nw, 16);
    b.diag = at;  if (!(flags & 64)) at += 16 * mp;  // diagonal + reciprocal; none when unit
    b.val = at;   at += 8 * mp * w;
    b.dep = at;   at += (flags & 9) == 0 ? round_up(2 * mp * w, 16) : 4 * mp * w;  // fast chunks: 16-bit ring slots
    b.exp = at;   at += 16 + 8 * ((mp + 31) / 32);    // export base id + {mask, prefix} per 32 rows
    b.oidx = at;  if (flags & 2) at += 4 * mp;
    b.tptr = at;  if (flags & 1) at += 4 * round_up(mp + 1, 4);
    b.tval = at;  if (flags & 1) at += 8 * round_up(ntail, 2);
    b.tdep = at;  if (flags & 1) at += 4 * round_up(ntail, 4);
    b.halo = at;  at += 4 * round_up(nhalo, 4);
    b.end = at;
    return b;
}
// --------------------------------------------------------------- COLUMNS ----
// The factor of a 7-point stencil on an nx x ny x nz grid in natural order
// (every dependency of row (x,y,z) is one of (x-1,y,z), (x,y-1,z), (x,y,z-1),
// in any ELL/CSR order): row (x,y,z) sits on level x+y+z, and along a grid
// column (x,y) the rows follow one another level by level. Each solver lane
// then owns four columns for the whole solve and keeps their latest x in
// registers: at level L, row (x,y,z) needs exactly the latest values of its own
// column (z-1), of column (x-1,y) and of column (x,y-1) -- registers, warp
// shuffles, and at warp / CTA tile edges a shared-memory edge ring or an
// epoch-tagged mailbox. No dependency indices, no x ring, no per-chunk blob
// decode: per level and lane only the rows' values, their presence mask and b
// are read (one TMA bulk copy per CTA level into a shared-memory ring). The
// warps of a CTA run free: each waits only for its left and lower neighbour
// warps' previous level (shared-memory progress counters).
//
// CTA (px, py) owns a TX x TY tile of columns, TX = 8 WX, TY = 4 rpl WY; warp
// (wx, wy) owns an 8 x 4 rpl sub-tile, lane lq * 8 + lx owns the columns
// (lx, rpl lq .. rpl lq + rpl - 1) of it (rpl = 1, 2 or 4 columns per lane). Column x = px*TX + wx*8 + lx - ox (y likewise);
// ox, oy anchor the tiling (0, or at the far end for the mirror of another
// layout). Slots: CTA-major, then the CTA's levels, then 32*rpl*NW per level
// ((warp * 32 + lane) * rpl + r; columns off the grid and rows outside [0, nz)
// are padding). The right-hand side is permuted into slot order (bidx), x
// comes out in slot order (wpos).
// shared memory in front of the level ring: full[16] / empty[16] mbarriers, then
// the warp edge rings (12 levels x (64 + 128) tagged values of 16 bytes)
constexpr int kColEdgeLevels = 12;
constexpr int kColCtrlBytes = 256 + kColEdgeLevels * 192 * 16;
struct ColMirror {
    int nx = 0, ny = 0, nz = 0, WX = 0, WY = 0, PX = 0, PY = 0, ox = 0, oy = 0;
    long long slots = 0;
    int order = 0, rpl = 1;
};
struct ColConfig {
    int ctas = 148;
    int warps = 0;                       // solver warps per CTA (WX*WY); 0 = chosen here
    int rpl = 0;                         // columns per lane; 0 = chosen here
    int smem_bytes = 0;                  // dynamic shared memory budget (level ring)
    int ring_max = kColEdgeLevels - 2;   // level blocks in flight at most (the edge rings hold kColEdgeLevels)
    const ColMirror* mirror = nullptr;   // build the exact mirror of this layout (U of an ILU pair)
};
struct ColLayout {
    static constexpr int SX = 8;         // warp sub-tile 8 x 4 rpl: lane (lq, lx) owns y = rpl lq .. rpl lq + rpl - 1
    int rpl = 1;                         // columns per lane (1, 2 or 4)
    int n = 0, nx = 0, ny = 0, nz = 0;
    int WX = 1, WY = 1, PX = 1, PY = 1, ox = 0, oy = 0;
    int ctas = 0, warps = 0, lanes = 0;  // lanes = 32 * rpl * warps slots per level
    int nlev = 0;                        // nx + ny + nz - 2 levels of the grid
    int block_bytes = 0;                 // one CTA level: val[3][lanes] f64 (by position in `order`),
                                         //   (diag, rcp)[lanes] f64 unless unit, mask[lanes] u8 (present positions)
    int order = 0;                       // the rows' entry order: directions o0 | o1 << 2 | o2 << 4 (0 x-1, 1 y-1, 2 z-1)
    int ring = 0;                        // level blocks in flight per CTA (shared memory)
    bool unit = false;                   // every diagonal exactly 1.0: x = num * 1.0
    bool mirrored = false;               // slot s is slot S-1-s of the mirrored layout
    long long slots = 0;                 // S
    long long mailboxes = 0;             // C * (TX + TY) * nz
    long long total_levels = 0;          // sum over CTAs of their level counts
    std::vector<int> cta;                // 4 per CTA: first level, level count, first slot / lanes, first block
    std::vector<unsigned char> blocks;   // total_levels * block_bytes
    std::vector<int> bidx;               // S: input index of the row in each slot (0 for padding)
    std::vector<int> wpos;               // n: solution index -> slot
    ColMirror mirror_info() const {
        return ColMirror{nx, ny, nz, WX, WY, PX, PY, ox, oy, slots, order, rpl};
    }
};
// Throws std::invalid_argument when the factor is not such a grid (or carries
// RAS maps): the caller falls back to the wave layout.
ColLayout build_columns(const TriSource& s, const ColConfig& cfg);

inline int wave_b_area(int m) { return 8 * round_up(m + 1, 4); }
// shared-memory bytes of a chunk region: b + blob + staged halo
inline int wave_region_bytes(int m, int nhalo, int blob_bytes) {
    (void)nhalo;  // staged into the halo ring, not the region
    return wave_b_area(m) + round_up(blob_bytes, 16);
}

}  // namespace hec::plan
