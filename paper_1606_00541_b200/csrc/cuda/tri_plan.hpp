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
};
LevelLayout build_levels(const TriSource& s);

// -------------------------------------------------------------- PIPELINE ----
// Persistent kernel, CTA c owns lower-frame rows [c*per, (c+1)*per). Its rows
// of one level form a contiguous reordered range ("chunk"); chunks are laid out
// back to back per CTA as self-describing 16-byte-aligned blobs that one
// cp.async.bulk moves into shared memory.
//
// Cross-CTA values travel through MAILBOXES: one FP64 word per (producer row,
// consumer CTA) pair. The producing solver thread stores x there (plain store,
// no fence); the consumer's waiter warp polls the word until it no longer holds
// the sentinel (a signalling NaN, which IEEE arithmetic can never produce),
// stages it into shared memory, and re-arms the word with the sentinel after
// its last use in this solve. No progress counters, no release/acquire fences.
//
// Blob layout (mp = round_up(m, 4)):
//   ChunkHeader (96 B: counts + every section offset, so the device decodes a
//                chunk with six 16-byte shared loads)
//                flags: 1 tail, 2 out-map, 4 mailbox stores, 8 global deps
//   int   halo[nhalo]   mailbox id * 2 + (1 if last use -> re-arm), pad 16 B
//   int   mbptr[mp+1]   (flags & 4) per-row range into mbid, pad 16 B
//   int   mbid[nmb]     (flags & 4) mailbox ids this chunk's rows feed, pad 16 B
//   double diag[mp]
//   double val[w][mp]               sliced ELL, slot-major
//   int    dep[w][mp]               >= 0 solution index (global, own rows older than the ring)
//                                    < 0: s = -d-1; s < ring: x ring slot; s == ring: 0.0;
//                                         s > ring: staged halo value s-ring-1
//   int    bidx[mp], xidx[mp], (oidx[mp] if flags & 2)
//   if flags & 1: int tptr[mp+1 -> mult of 4], double tval[ntail -> even], int tdep[ntail -> mult of 4]
// Shared-memory footprint of a chunk = blob + 8 * mp (gathered b) + 8 * nhalo.
constexpr unsigned long long kMailboxEmpty = 0x7FF4DEADBEEF0001ULL;  // signalling NaN

struct PipelineConfig {
    int ctas = 148;
    int ring = 4096;          // x ring entries (power of two); slot `ring` holds 0.0
    int max_width = 32;       // sliced-ELL width cap; longer rows spill to the tail
    int slot_cap = 24576;     // target shared-memory bytes of one chunk
};

struct PipelineLayout {
    int n = 0, nlev = 0, ctas = 0, ring = 0;
    int max_blob = 0;                     // bytes of the largest blob
    int chunks = 0;
    int max_rows = 0;                     // rows of the largest chunk
    int max_halo = 0;                     // halo values of the largest chunk
    bool has_out = false;
    long long mailboxes = 0;              // (producer row, consumer CTA) words
    std::vector<int> cta_chunk0;          // ctas + 1: chunk range of each CTA
    std::vector<int> span;                // 2 per chunk: (offset / 16, bytes)
    std::vector<unsigned char> blob;      // all chunk blobs, 16-byte aligned
    long long ring_deps = 0, global_deps = 0, halo_deps = 0;
};
PipelineLayout build_pipeline(const TriSource& s, const PipelineConfig& cfg);

// Blob section offsets (bytes from the blob start).
struct BlobSections {
    int halo, mbptr, mbid, diag, val, dep, bidx, xidx, oidx, tptr, tval, tdep, end;
};

// First 96 bytes of every blob; read by the kernel as-is.
struct ChunkHeader {
    int m, w, q0, flags;
    int nhalo, ntail, nmb, mp;
    int halo, mbptr, mbid, diag;
    int val, dep, bidx, xidx;
    int oidx, tptr, tval, tdep;
    int pad[4];
};
static_assert(sizeof(ChunkHeader) == 96, "chunk header is six 16-byte words");
constexpr int kChunkHeaderBytes = 96;

inline int round_up(int v, int m) { return (v + m - 1) / m * m; }
inline BlobSections blob_sections(int m, int w, int nhalo, int nmb, int ntail, int flags) {
    BlobSections b{};
    const int mp = round_up(m, 4);
    int at = kChunkHeaderBytes;
    b.halo = at;  at += round_up(4 * nhalo, 16);
    b.mbptr = at; if (flags & 4) at += 4 * round_up(mp + 1, 4);
    b.mbid = at;  if (flags & 4) at += round_up(4 * nmb, 16);
    b.diag = at;  at += 8 * mp;
    b.val = at;   at += 8 * mp * w;
    b.dep = at;   at += 4 * mp * w;
    b.bidx = at;  at += 4 * mp;
    b.xidx = at;  at += 4 * mp;
    b.oidx = at;  if (flags & 2) at += 4 * mp;
    b.tptr = at;  if (flags & 1) at += 4 * round_up(mp + 1, 4);
    b.tval = at;  if (flags & 1) at += 8 * round_up(ntail, 2);
    b.tdep = at;  if (flags & 1) at += 4 * round_up(ntail, 4);
    b.end = at;
    return b;
}

}  // namespace hec::plan
