#pragma once
// Kernel argument blocks shared by trisolve.cu and the device runtime.

#include <cuda_runtime.h>

#include <cstdint>

namespace hec::dev {

struct LevelArgs {
    const double* b;        // input vector (gathered through bidx)
    double* xs;             // solution vector (solution index space)
    double* out;            // optional second output (oidx), may be null
    const int* bidx;
    const int* xidx;
    const int* oidx;
    const int* ell_dep;     // width * ld, -1 = padding
    const double* ell_val;
    const double* diag;
    const int* tail_rp;
    const int* tail_dep;
    const double* tail_val;
    const int* long_rows;   // rows with >= long_min remainder entries (a warp each)
    int width;
    int ld;
    int b_ordered;          // b already in reordered-row order (bidx ignored)
    int long_min;           // 0: every row thread-serial
};

struct WaveArgs {
    const unsigned char* blobs;  // all chunk blobs (16-byte aligned)
    const int4* spans;           // 2 per chunk: (blob offset / 16, blob bytes, region bytes, r0),
                                 //              (b area bytes, b copy bytes, 0, 0)
    const int* cta_chunk0;       // ctas + 1
    const double* bp;            // right-hand side in reordered-row order
    double* xs;
    double* out;
    unsigned long long* mbox;    // 2 words per exported row: {lo32|epoch<<32, hi32|epoch<<32}
    uint32_t* counters;          // [0] ticket, [1] CTAs finished, [2] this solve's mailbox epoch
                                 // (advanced by the last CTA out: graph-replay safe)
    int ctas;
    int inflight;                // descriptor slots (power of two <= 32)
    int inflight_log2;
    int lead;                    // (informational: 1, chunks complete in order)
    int ring;                    // x ring entries (power of two)
    int halo_ring;               // H: staged-halo ring entries, behind the x ring
    int ring_off;                // shared-memory byte offsets
    int buf_off;
    int buf_bytes;
    int spin_ns;                 // back-off between the waiters' mailbox polls (HEC_WAVE_SPIN_NS, 0 = off)
    unsigned long long watchdog_cycles;  // SM cycles after the CTA started: past them a wait traps (HEC_WAVE_WATCHDOG_MS)
    unsigned long long* trace;   // diagnostics: 16 words per chunk (TRACE kernel only)
};

// k_cols (cols_kernel.cu; layout: tri_plan.hpp COLUMNS)
struct ColArgs {
    const unsigned char* blocks;  // one block per (CTA, level): val[3][lanes], (diag, rcp)[lanes], code[lanes]
    const int4* cta;              // per CTA: first level, level count, first slot / lanes, first block
    const double* bp;             // right-hand side in slot order (bp_reversed: slot s reads bp[slots-1-s])
    double* xw;                   // solution in slot order
    unsigned long long* mbox;     // tile-edge mailboxes, 2 epoch-tagged words each
    uint32_t* counters;           // as WaveArgs::counters
    long long slots;
    long long mbox_top0;          // first top-edge mailbox (right-edge ones come first)
    int ctas, nx, ny, nz, WX, WY, PX, PY, ox, oy;
    int block_bytes, ring, bp_reversed;
    int order;                    // entry order shared by all rows (plan::ColLayout::order)
    unsigned long long watchdog_cycles;
    unsigned long long* trace;    // diagnostics (trace kernel): 4 words per CTA level (warp 0, lane 0)
};
void* cols_kernel(int warps, int rpl, bool unit, bool trace, int order);
constexpr int kColOrderZYX = 2 | 1 << 2 | 0 << 4;  // (z-1, y-1, x-1): natural-order 7-point factors

// one launch per level, arguments read from dev_args (capturable once, replayed for any vectors)
void launch_levels(const LevelArgs* dev_args, const int* level_starts_host, const int* long_starts_host, int nlev,
                   cudaStream_t st);
void set_level_args(const LevelArgs& a, LevelArgs* dev, cudaStream_t st);
// all levels in one cooperative launch with a grid barrier between them
void launch_levels_persist(const LevelArgs* dev_args, const int* level_starts_dev, int nlev, cudaStream_t st);
// kernel for sliced-ELL width W (one of 1-8, 10, 13, 16) and solver shape
// (group warps G x groups K x rpl rows per lane, see wave_inst.cuh); nullptr
// when that combination is not instantiated
void* wave_kernel(int width, int group, int groups, int rpl, bool trace);
// bp[r] = b[bidx[r]] for r < n (the reference's permute-in pass, coalesced writes)
void permute_in(const double* b, const int* bidx, double* bp, int n, cudaStream_t st);
// bp[wpos[o]] = b[o], o in [0, n)
void scatter_rows(const double* b, const int* wpos, double* bp, int n, cudaStream_t st);
constexpr int kWaveSolverWarps = 16;
// producer / waiter warps of k_wave: 2 + 5 in general (3 waiters could not keep
// up with 27-point halos); the narrow-row shapes with more groups (z-pencils:
// few halo values per chunk) keep the thread count, hence the register budget,
// with 1 + 2
__host__ __device__ constexpr bool wave_lean_roles(int group, int groups, int rpl) {
    return groups == 3 && group * rpl > 0;
}
__host__ __device__ constexpr int wave_producers(int group, int groups, int rpl) {
    return wave_lean_roles(group, groups, rpl) ? 1 : 2;
}
__host__ __device__ constexpr int wave_waiters(int group, int groups, int rpl) {
    return wave_lean_roles(group, groups, rpl) ? 2 : 5;
}
__host__ __device__ constexpr int wave_role_threads(int group, int groups, int rpl) {
    return 32 * (wave_producers(group, groups, rpl) + wave_waiters(group, groups, rpl));
}
constexpr int kWaveCtrlBytes = 1536;                   // control block at the start of shared memory

}  // namespace hec::dev
