// Matrix Market text reader / writer on the host.
//
// Follows load_matrix_market (matrix_market.cpp:117-165) and its helpers
// parse_header (:38-70) and next_data_line (:73-83): same accepted headers,
// same ParseError line numbers and messages, same UnsupportedFormat cases, the
// same symmetric / skew-symmetric expansion and zero filtering. The reference
// reads each line through an std::istringstream; the scanners below restate
// the C-locale extraction rules it relies on (libstdc++ num_get: optional
// sign, decimal digits, optional fraction and exponent, failure on an
// incomplete exponent or on overflow, the value itself converted by strtod, so
// the parsed doubles are the same bits) over one buffered read of the file.
#include "mtx.hpp"

#include <cerrno>
#include <cinttypes>
#include <cmath>
#include <cstdio>
#include <cstdlib>
#include <cstring>

#include "../../include/dashsvd_b200.h"

namespace dsvd {

namespace {

struct Cursor {
    const char* p;
    const char* end;
};

inline bool is_space(char ch) {
    return ch == ' ' || ch == '\t' || ch == '\n' || ch == '\v' || ch == '\f' || ch == '\r';
}

inline void skip_ws(Cursor& s) {
    while (s.p < s.end && is_space(*s.p)) ++s.p;
}

// `ss >> std::string`
bool read_token(Cursor& s, std::string& tok) {
    skip_ws(s);
    if (s.p == s.end) return false;
    const char* b = s.p;
    while (s.p < s.end && !is_space(*s.p)) ++s.p;
    tok.assign(b, s.p);
    return true;
}

// `ss >> int64_t`: [+-]digits, failure on no digits or overflow
bool read_int(Cursor& s, int64_t& out) {
    skip_ws(s);
    const char* q = s.p;
    bool neg = false;
    if (q < s.end && (*q == '+' || *q == '-')) neg = (*q++ == '-');
    const char* d0 = q;
    uint64_t mag = 0;
    bool overflow = false;
    const uint64_t lim = neg ? (uint64_t(INT64_MAX) + 1) : uint64_t(INT64_MAX);
    while (q < s.end && *q >= '0' && *q <= '9') {
        const unsigned dgt = static_cast<unsigned>(*q - '0');
        if (mag > (lim - dgt) / 10) overflow = true;
        else mag = mag * 10 + dgt;
        ++q;
    }
    if (q == d0 || overflow) return false;
    s.p = q;
    out = neg ? static_cast<int64_t>(0 - mag) : static_cast<int64_t>(mag);
    return true;
}

// `ss >> double`: accumulate [+-]digits[.digits][(e|E)[+-]digits] (an
// exponent only after a mantissa digit), convert with strtod; failure when
// the accumulated text is not a complete number or the value overflows.
bool read_double(Cursor& s, double& out) {
    skip_ws(s);
    const char* q = s.p;
    std::string acc;
    if (q < s.end && (*q == '+' || *q == '-')) acc.push_back(*q++);
    bool mant = false, dot = false;
    while (q < s.end) {
        const char ch = *q;
        if (ch >= '0' && ch <= '9') {
            mant = true;
        } else if (ch == '.' && !dot) {
            dot = true;
        } else {
            break;
        }
        acc.push_back(ch);
        ++q;
    }
    if (mant && q < s.end && (*q == 'e' || *q == 'E')) {
        acc.push_back(*q++);
        if (q < s.end && (*q == '+' || *q == '-')) acc.push_back(*q++);
        while (q < s.end && *q >= '0' && *q <= '9') acc.push_back(*q++);
    }
    s.p = q;
    if (acc.empty()) return false;
    char* stop = nullptr;
    const double v = std::strtod(acc.c_str(), &stop);
    if (stop == acc.c_str() || *stop != '\0') return false;
    if (v == HUGE_VAL || v == -HUGE_VAL) return false;
    out = v;
    return true;
}

std::string lower(std::string x) {
    for (char& ch : x)
        if (ch >= 'A' && ch <= 'Z') ch = static_cast<char>(ch - 'A' + 'a');
    return x;
}

struct Lines {
    const char* p;
    const char* end;
    int64_t lineno = 0;
    // std::getline: the next '\n'-terminated line; false at end of input
    bool getline(Cursor& line) {
        if (p >= end) return false;
        const char* nl = static_cast<const char*>(std::memchr(p, '\n', static_cast<size_t>(end - p)));
        const char* e = nl ? nl : end;
        line = Cursor{p, e};
        p = nl ? nl + 1 : end;
        return true;
    }
    // next_data_line: skip blank (" \t\r" only) and '%' comment lines
    bool next_data(Cursor& line) {
        while (getline(line)) {
            ++lineno;
            const char* q = line.p;
            while (q < line.end && (*q == ' ' || *q == '\t' || *q == '\r')) ++q;
            if (q == line.end || *q == '%') continue;
            return true;
        }
        return false;
    }
};

MtxStatus parse_error(int64_t line, std::string what) { return MtxStatus{DSVD_PARSE, line, std::move(what)}; }
MtxStatus format_error(std::string what) { return MtxStatus{DSVD_FORMAT, 0, std::move(what)}; }

enum Field { kReal, kInteger, kPattern };
enum Symmetry { kGeneral, kSymmetric, kSkew };
struct Header {
    bool coordinate = true;
    Field field = kReal;
    Symmetry sym = kGeneral;
};

// parse_header (matrix_market.cpp:38-70)
MtxStatus parse_header(const Cursor& line, Header& h) {
    std::string banner, object, format, fld, symmetry;
    Cursor c = line;
    read_token(c, banner) && read_token(c, object) && read_token(c, format) && read_token(c, fld) &&
        read_token(c, symmetry);
    if (banner != "%%MatrixMarket") return parse_error(1, "missing %%MatrixMarket banner");
    if (lower(object) != "matrix") return format_error("unsupported object: " + object);
    const std::string fm = lower(format);
    if (fm == "coordinate") h.coordinate = true;
    else if (fm == "array") h.coordinate = false;
    else return format_error("unsupported format: " + format);
    const std::string fl = lower(fld);
    if (fl == "real") h.field = kReal;
    else if (fl == "integer") h.field = kInteger;
    else if (fl == "pattern") h.field = kPattern;
    else return format_error("unsupported field: " + fld);
    const std::string sy = lower(symmetry);
    if (sy == "general") h.sym = kGeneral;
    else if (sy == "symmetric") h.sym = kSymmetric;
    else if (sy == "skew-symmetric") h.sym = kSkew;
    else return format_error("unsupported symmetry: " + symmetry);
    return MtxStatus{};
}

bool read_file(const char* path, std::string& buf) {
    std::FILE* f = std::fopen(path, "rb");
    if (!f) return false;
    char chunk[1 << 16];
    size_t got;
    while ((got = std::fread(chunk, 1, sizeof(chunk), f)) > 0) buf.append(chunk, got);
    std::fclose(f);
    return true;
}

}  // namespace

MtxStatus mtx_read(const char* path, MtxTriplets& out) {
    std::string buf;
    if (!read_file(path, buf)) return MtxStatus{DSVD_OTHER, 0, std::string("cannot open ") + path};
    Lines in{buf.data(), buf.data() + buf.size()};
    Cursor line{};
    if (!in.getline(line)) return parse_error(1, "empty file");
    in.lineno = 1;
    // parse_header (:38-70)
    Header hd;
    {
        const MtxStatus hs = parse_header(line, hd);
        if (hs.code != DSVD_OK) return hs;
        if (!hd.coordinate) return format_error("array format holds a dense matrix; use load_dense_array");
    }
    const auto field = hd.field;
    const auto sym = hd.sym;
    if (!in.next_data(line)) return parse_error(in.lineno + 1, "missing size line");
    int64_t rows, cols, nnz;
    {
        Cursor s = line;
        if (!(read_int(s, rows) && read_int(s, cols) && read_int(s, nnz)) || rows < 0 || cols < 0 || nnz < 0)
            return parse_error(in.lineno, "size line must be 'rows cols nnz'");
        std::string extra;
        if (read_token(s, extra)) return parse_error(in.lineno, "trailing token on size line");
    }
    out.rows = rows;
    out.cols = cols;
    const size_t cap = static_cast<size_t>(sym == kGeneral ? nnz : 2 * nnz);
    out.r.clear();
    out.c.clear();
    out.v.clear();
    out.r.reserve(cap);
    out.c.reserve(cap);
    out.v.reserve(cap);
    auto push = [&](int64_t i, int64_t j, double v) {
        out.r.push_back(i);
        out.c.push_back(j);
        out.v.push_back(v);
    };
    std::string extra;
    for (int64_t e = 0; e < nnz; ++e) {
        if (!in.next_data(line))
            return parse_error(in.lineno + 1, "expected " + std::to_string(nnz) + " entries, file ended after " +
                                                  std::to_string(e));
        Cursor s = line;
        int64_t i, j;
        if (!(read_int(s, i) && read_int(s, j))) return parse_error(in.lineno, "entry must start with two indices");
        double v = 1.0;
        if (field != kPattern && !read_double(s, v)) return parse_error(in.lineno, "entry is missing its value");
        if (read_token(s, extra)) return parse_error(in.lineno, "trailing token on entry line");
        if (i < 1 || i > rows || j < 1 || j > cols) return parse_error(in.lineno, "index out of declared bounds");
        if (!std::isfinite(v)) return parse_error(in.lineno, "non-finite value");
        --i, --j;
        if (sym == kSkew && i == j && v != 0.0)
            return parse_error(in.lineno, "nonzero diagonal in skew-symmetric matrix");
        if (v != 0.0) push(i, j, v);
        if (i != j) {
            if (sym == kSymmetric) push(j, i, v);
            if (sym == kSkew && v != 0.0) push(j, i, -v);
        }
    }
    return MtxStatus{};
}

MtxStatus mtx_write(const char* path, int64_t rows, int64_t cols, const int64_t* offsets,
                    const int64_t* col_indices, const double* values) {
    std::FILE* f = std::fopen(path, "w");
    if (!f) return MtxStatus{DSVD_OTHER, 0, std::string("cannot open ") + path + " for writing"};
    const int64_t nnz = offsets[rows];
    std::fprintf(f, "%%%%MatrixMarket matrix coordinate real general\n");
    std::fprintf(f, "%" PRId64 " %" PRId64 " %" PRId64 "\n", rows, cols, nnz);
    for (int64_t i = 0; i < rows; ++i)
        for (int64_t p = offsets[i]; p < offsets[i + 1]; ++p)
            std::fprintf(f, "%" PRId64 " %" PRId64 " %.17g\n", i + 1, col_indices[p] + 1, values[p]);
    if (std::fclose(f) != 0) return MtxStatus{DSVD_OTHER, 0, std::string("failed writing ") + path};
    return MtxStatus{};
}

MtxStatus dense_read(const char* path, DenseArray& out) {
    std::string buf;
    if (!read_file(path, buf)) return MtxStatus{DSVD_OTHER, 0, std::string("cannot open ") + path};
    Lines in{buf.data(), buf.data() + buf.size()};
    Cursor line{};
    if (!in.getline(line)) return parse_error(1, "empty file");
    in.lineno = 1;
    Header hd;
    {
        const MtxStatus hs = parse_header(line, hd);
        if (hs.code != DSVD_OK) return hs;
    }
    if (hd.coordinate) return format_error("coordinate file; use load_matrix_market");
    if (hd.field == kPattern) return format_error("pattern array is not a matrix");
    if (!in.next_data(line)) return parse_error(in.lineno + 1, "missing size line");
    int64_t rows, cols;
    {
        Cursor s = line;
        if (!(read_int(s, rows) && read_int(s, cols)) || rows < 0 || cols < 0)
            return parse_error(in.lineno, "size line must be 'rows cols'");
    }
    const int64_t total = rows * cols;
    out.rows = rows;
    out.cols = cols;
    out.data.clear();
    out.data.reserve(static_cast<size_t>(total));
    while (static_cast<int64_t>(out.data.size()) < total) {
        if (!in.next_data(line)) return parse_error(in.lineno + 1, "file ended before all entries were read");
        Cursor s = line;
        double v;
        // `while (ss >> v) push; if (!ss.eof()) malformed`: a failed extraction is
        // fine only when it ran into the end of the line
        while (read_double(s, v)) out.data.push_back(v);
        if (s.p != s.end) return parse_error(in.lineno, "malformed value");
    }
    if (static_cast<int64_t>(out.data.size()) != total) return parse_error(in.lineno, "more entries than rows*cols");
    for (double v : out.data)
        if (!std::isfinite(v)) return parse_error(in.lineno, "non-finite value in array");
    return MtxStatus{};
}

MtxStatus dense_write(const char* path, int64_t rows, int64_t cols, const double* colmajor) {
    std::FILE* f = std::fopen(path, "w");
    if (!f) return MtxStatus{DSVD_OTHER, 0, std::string("cannot open ") + path + " for writing"};
    std::fprintf(f, "%%%%MatrixMarket matrix array real general\n");
    std::fprintf(f, "%" PRId64 " %" PRId64 "\n", rows, cols);
    for (int64_t e = 0; e < rows * cols; ++e) std::fprintf(f, "%.17g\n", colmajor[e]);
    if (std::fclose(f) != 0) return MtxStatus{DSVD_OTHER, 0, std::string("failed writing ") + path};
    return MtxStatus{};
}

MtxStatus spectrum_read(const char* path, std::vector<double>& out) {
    std::string buf;
    if (!read_file(path, buf)) return MtxStatus{DSVD_OTHER, 0, std::string("cannot open ") + path};
    Lines in{buf.data(), buf.data() + buf.size()};
    Cursor line{};
    out.clear();
    while (in.getline(line)) {
        ++in.lineno;
        const char* q = line.p;
        while (q < line.end && (*q == ' ' || *q == '\t' || *q == '\r')) ++q;
        if (q == line.end || *q == '#') continue;
        Cursor s = line;
        double v;
        if (!read_double(s, v) || !std::isfinite(v) || v < 0.0)
            return parse_error(in.lineno, "expected a non-negative singular value");
        if (!out.empty() && v > out.back() * (1.0 + 1e-12) + 1e-300)
            return parse_error(in.lineno, "singular values must be non-increasing");
        out.push_back(v);
    }
    if (out.empty()) return parse_error(in.lineno, "no singular values in file");
    return MtxStatus{};
}

MtxStatus spectrum_write(const char* path, const double* sigmas, int64_t n) {
    std::FILE* f = std::fopen(path, "w");
    if (!f) return MtxStatus{DSVD_OTHER, 0, std::string("cannot open ") + path + " for writing"};
    for (int64_t i = 0; i < n; ++i) std::fprintf(f, "%.17g\n", sigmas[i]);
    if (std::fclose(f) != 0) return MtxStatus{DSVD_OTHER, 0, std::string("failed writing ") + path};
    return MtxStatus{};
}

}  // namespace dsvd
