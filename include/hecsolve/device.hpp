#pragma once
// Device-side state attached to the drop-in types, and the B200 knobs.
// Nothing here exists in the reference; it only adds to PreparedTriangular and
// BlockPreconditioner (never to CsrMatrix / EllMatrix / HecMatrix, whose
// defaulted operator== the reference tests use).

#include <memory>
#include <mutex>

#include "hecsolve_c.h"

namespace hec::device {

// Process-wide defaults used when a mirror is first built.
struct Options {
    int strategy = HEC_STRATEGY_AUTO;  // HEC_STRATEGY_LEVELS | HEC_STRATEGY_PIPELINE
    int ctas = 0;                      // 0 = one persistent CTA per SM
    int threads = 0;                   // 0 = auto
};
void set_options(const Options& o);
Options options();

// Lazily built device copy of one prepared triangle; shared by copies of the
// PreparedTriangular that owns it.
struct TriMirror {
    std::mutex mu;
    hec_tri_t handle = nullptr;
    const void* source = nullptr;  // data() of the arrays the handle was built from
    TriMirror() = default;
    TriMirror(const TriMirror&) = delete;
    TriMirror& operator=(const TriMirror&) = delete;
    ~TriMirror();
};

struct PrecondMirror {
    std::mutex mu;
    hec_precond_t handle = nullptr;
    const void* source = nullptr;
    PrecondMirror() = default;
    PrecondMirror(const PrecondMirror&) = delete;
    PrecondMirror& operator=(const PrecondMirror&) = delete;
    ~PrecondMirror();
};

}  // namespace hec::device

namespace hec {
struct PreparedTriangular;
struct BlockPreconditioner;
// The device handles behind the drop-in objects (built on first use).
hec_tri_t device_handle(const PreparedTriangular& p);
hec_precond_t device_handle(const BlockPreconditioner& m);
}  // namespace hec
