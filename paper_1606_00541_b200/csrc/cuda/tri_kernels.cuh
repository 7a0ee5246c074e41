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
    int width;
    int ld;
};

struct PipeArgs {
    const unsigned char* blobs;  // all chunk blobs (16-byte aligned)
    const int2* spans;           // per chunk (offset / 16, bytes)
    const int* cta_chunk0;       // ctas + 1
    const double* b;
    double* xs;
    double* out;
    unsigned long long* mbox;    // cross-CTA mailbox words (sentinel = empty)
    uint32_t* counters;          // [0] ticket, [1] CTAs finished
    int ctas;
    int nslots;
    int lag;
    int slot_bytes;
    int b_bytes;                 // gathered-b area at the start of each slot
    int halo_bytes;              // staged halo values after it
    int ring;                    // ring entries (power of two)
    int ring_off;                // shared-memory byte offsets
    int slot_off;
    unsigned long long* trace;   // diagnostics: 16 words per chunk (TRACE kernel only)
};

void launch_levels(const LevelArgs& a, const int* level_starts_host, int nlev, cudaStream_t st);
void* pipeline_kernel(int nsolve, bool trace);
void fill_mailboxes(unsigned long long* p, long long n, cudaStream_t st);
constexpr int kPipelineRoleThreads = 64;  // producer warp + waiter warp

}  // namespace hec::dev
