#pragma once
// Hybrid ELL + CSR ("HEC") storage, the paper's format (arXiv 1606.00541 §2.1).
// Drop-in for reference proj/include/hecsolve/hec.hpp:13-57.
//
// Host-side layout is the reference's: the ELL block is column-major (slot k of
// row i at k * n_rows + i), unused slots hold value 0 and column min(i, n_cols-1);
// in triangular mode the diagonal is always the last entry of the CSR part.
// The device copy (see hecsolve/device.hpp) re-slices this per (CTA, level)
// chunk; the arithmetic order per row is unchanged.

#include <vector>

#include "hecsolve/csr.hpp"

namespace hec {

struct EllMatrix {
    int n_rows = 0;
    int width = 0;
    std::vector<int> col_indices;  // width * n_rows, column-major
    std::vector<double> values;    // width * n_rows, column-major

    bool operator==(const EllMatrix&) const = default;
};

struct WidthPolicy {
    enum class Mode { fixed, automatic };

    Mode mode = Mode::automatic;
    int width = 0;

    static WidthPolicy fixed(int w) { return {Mode::fixed, w}; }
    static WidthPolicy automatic() { return {}; }
};

struct HecMatrix {
    int n_rows = 0;
    int n_cols = 0;
    EllMatrix ell;
    CsrMatrix csr;

    bool operator==(const HecMatrix&) const = default;
};

// Splits every row: its first min(w, eligible) entries go to ELL, the rest to
// CSR. `triangular` reserves the diagonal (which must close each row) for CSR.
// Automatic width = median eligible count, clamped to [0, max count].
HecMatrix hec_from_csr(const CsrMatrix& a, bool triangular, WidthPolicy policy = {});

// y = A x over the hybrid form; bitwise equal to spmv_csr on the source.
std::vector<double> spmv_hec(const HecMatrix& a, const std::vector<double>& x, int workers = 1);

// Inverse of hec_from_csr (slots holding (pad column, 0.0) are dropped).
CsrMatrix csr_from_hec(const HecMatrix& h);

}  // namespace hec
