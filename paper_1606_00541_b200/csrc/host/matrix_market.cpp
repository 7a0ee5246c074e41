// MatrixMarket coordinate reader / writer (host setup; drop-in for reference
// proj/src/matrix_market.cpp:27-81). The reader scans the whole file once
// with a small cursor over a byte buffer instead of iostream extraction.

#include "hecsolve/matrix_market.hpp"

#include <cctype>
#include <cerrno>
#include <cstdio>
#include <cstdlib>
#include <fstream>
#include <iterator>
#include <stdexcept>
#include <string>
#include <vector>

namespace hec {

namespace {

struct Cursor {
    const std::string& path;
    std::string text;
    std::size_t at = 0;

    [[noreturn]] void bad(const std::string& what) const {
        throw std::runtime_error("read_matrix_market: " + what + " in " + path);
    }
    bool eof() const { return at >= text.size(); }
    std::string line() {  // next line without its terminator
        const std::size_t end = text.find('\n', at);
        std::string s = text.substr(at, end == std::string::npos ? std::string::npos : end - at);
        at = end == std::string::npos ? text.size() : end + 1;
        if (!s.empty() && s.back() == '\r') s.pop_back();
        return s;
    }
    void skip_space() {
        while (at < text.size() && std::isspace(static_cast<unsigned char>(text[at]))) ++at;
    }
    // one whitespace-delimited token as an integer / a double; false at end of input or on junk
    bool integer(long long& v) {
        skip_space();
        if (eof()) return false;
        char* end = nullptr;
        errno = 0;
        v = std::strtoll(text.c_str() + at, &end, 10);
        if (end == text.c_str() + at || errno) return false;
        at = static_cast<std::size_t>(end - text.c_str());
        return true;
    }
    bool real(double& v) {
        skip_space();
        if (eof()) return false;
        char* end = nullptr;
        v = std::strtod(text.c_str() + at, &end);
        if (end == text.c_str() + at) return false;
        at = static_cast<std::size_t>(end - text.c_str());
        return true;
    }
};

std::vector<std::string> words(const std::string& s) {
    std::vector<std::string> w;
    std::size_t i = 0;
    while (i < s.size()) {
        while (i < s.size() && std::isspace(static_cast<unsigned char>(s[i]))) ++i;
        std::size_t j = i;
        while (j < s.size() && !std::isspace(static_cast<unsigned char>(s[j]))) ++j;
        if (j > i) w.push_back(s.substr(i, j - i));
        i = j;
    }
    return w;
}

bool same_nocase(const std::string& a, const char* b) {
    std::size_t k = 0;
    for (; k < a.size() && b[k]; ++k)
        if (std::tolower(static_cast<unsigned char>(a[k])) != b[k]) return false;
    return k == a.size() && !b[k];
}

}  // namespace

CsrMatrix read_matrix_market(const std::string& path) {
    std::ifstream in(path, std::ios::binary);
    if (!in) throw std::runtime_error("read_matrix_market: cannot open " + path);
    Cursor c{path, std::string(std::istreambuf_iterator<char>(in), std::istreambuf_iterator<char>())};
    if (c.eof()) c.bad("missing header");
    const std::string head = c.line();
    const std::vector<std::string> h = words(head);
    if (h.size() < 4 || !same_nocase(h[0], "%%matrixmarket") || !same_nocase(h[1], "matrix") ||
        !same_nocase(h[2], "coordinate") || !same_nocase(h[3], "real"))
        c.bad("malformed header '" + head + "'");
    const std::string sym = h.size() > 4 ? h[4] : "";
    const bool symmetric = same_nocase(sym, "symmetric");
    if (!symmetric && !same_nocase(sym, "general")) c.bad("unsupported symmetry '" + sym + "'");

    std::string size_line;
    do {  // comment and blank lines may precede the size line
        if (c.eof()) c.bad("missing size line");
        size_line = c.line();
    } while (size_line.empty() || size_line[0] == '%');
    long long dims[3];
    Cursor sc{path, size_line};
    for (long long& d : dims)
        if (!sc.integer(d) || d < 0) c.bad("malformed size line '" + size_line + "'");
    const long long rows = dims[0], cols = dims[1], count = dims[2];
    if (symmetric && rows != cols) c.bad("symmetric header on a non-square size line");

    std::vector<Triplet> t;
    t.reserve(static_cast<std::size_t>(symmetric ? 2 * count : count));
    for (long long k = 0; k < count; ++k) {
        long long i = 0, j = 0;
        double v = 0.0;
        if (!c.integer(i) || !c.integer(j) || !c.real(v)) c.bad("unexpected end of entries");
        if (i < 1 || i > rows || j < 1 || j > cols)
            c.bad("entry index out of bounds at line " + std::to_string(k + 1));
        t.push_back({static_cast<int>(i - 1), static_cast<int>(j - 1), v});
        if (symmetric && i != j) t.push_back({static_cast<int>(j - 1), static_cast<int>(i - 1), v});
    }
    // duplicates (e.g. a symmetric file storing both halves) are rejected here
    return csr_from_triples(static_cast<int>(rows), static_cast<int>(cols), std::move(t));
}

void write_matrix_market(const CsrMatrix& a, const std::string& path) {
    std::FILE* f = std::fopen(path.c_str(), "w");
    if (!f) throw std::runtime_error("write_matrix_market: cannot open " + path);
    bool ok = std::fprintf(f, "%%%%MatrixMarket matrix coordinate real general\n%d %d %lld\n", a.n_rows,
                           a.n_cols, static_cast<long long>(a.nnz())) > 0;
    for (int i = 0; ok && i < a.n_rows; ++i)
        for (int k = a.row_offsets[i]; ok && k < a.row_offsets[i + 1]; ++k)
            ok = std::fprintf(f, "%d %d %.17g\n", i + 1, a.col_indices[k] + 1, a.values[k]) > 0;
    ok = (std::fclose(f) == 0) && ok;
    if (!ok) throw std::runtime_error("write_matrix_market: write failed for " + path);
}

}  // namespace hec
