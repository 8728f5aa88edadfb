// mtx.cpp -- Matrix Market ingestion into host CSR (SURVEY.md §8f "next" #2).
//
// The reference reads .mtx files for statistics only (matrix_market.cpp:126-201:
// banner, size line, per-entry validation, symmetric expansion) and feeds
// them to the CSR model (stats_to_report, matrix_market.cpp:203-216).  This
// restates that parser with the same error kinds and messages' meaning, and
// extends it to materialise the CSR arrays the sm_100a SpMV consumes:
// 0-based int32 indices, columns sorted within each row, symmetric /
// skew-symmetric storage expanded (mirror entries; skew mirrors negate),
// pattern entries stored as 1.0.  Complex and array formats are rejected.
#include <algorithm>
#include <cctype>
#include <cerrno>
#include <cstdlib>
#include <cstring>
#include <fstream>
#include <numeric>
#include <string>
#include <vector>

#include "../../include/rooflens_b200.hpp"

namespace rooflens::b200 {
namespace {

enum class Field { Real, Integer, Pattern, Complex };
enum class Symm { General, Symmetric, Skew, Hermitian };

struct Banner {
    bool coordinate = true;
    Field field = Field::Real;
    Symm symm = Symm::General;
};

std::string lower(std::string s) {
    for (char& ch : s) ch = static_cast<char>(std::tolower(static_cast<unsigned char>(ch)));
    return s;
}

std::vector<std::string> tokens_of(const std::string& line) {
    std::vector<std::string> out;
    size_t i = 0;
    while (i < line.size()) {
        while (i < line.size() && std::isspace(static_cast<unsigned char>(line[i]))) ++i;
        const size_t b = i;
        while (i < line.size() && !std::isspace(static_cast<unsigned char>(line[i]))) ++i;
        if (i > b) out.emplace_back(line.substr(b, i - b));
    }
    return out;
}

Banner banner_of(const std::string& line) {
    const auto t = tokens_of(line);
    if (t.size() < 5 || lower(t[0]) != "%%matrixmarket")
        throw Error(ErrorKind::BadBanner, "expected '%%MatrixMarket object format field symmetry'");
    if (lower(t[1]) != "matrix") throw Error(ErrorKind::BadBanner, "unsupported object '" + lower(t[1]) + "'");
    Banner b;
    const std::string fmt = lower(t[2]), fld = lower(t[3]), sym = lower(t[4]);
    if (fmt == "coordinate") b.coordinate = true;
    else if (fmt == "array") b.coordinate = false;
    else throw Error(ErrorKind::BadBanner, "unknown format '" + fmt + "'");
    if (fld == "real") b.field = Field::Real;
    else if (fld == "integer") b.field = Field::Integer;
    else if (fld == "pattern") b.field = Field::Pattern;
    else if (fld == "complex") b.field = Field::Complex;
    else throw Error(ErrorKind::BadBanner, "unknown field '" + fld + "'");
    if (sym == "general") b.symm = Symm::General;
    else if (sym == "symmetric") b.symm = Symm::Symmetric;
    else if (sym == "skew-symmetric") b.symm = Symm::Skew;
    else if (sym == "hermitian") b.symm = Symm::Hermitian;
    else throw Error(ErrorKind::BadBanner, "unknown symmetry '" + sym + "'");
    return b;
}

bool data_line(std::istream& in, std::string& line) {
    while (std::getline(in, line)) {
        if (!line.empty() && line.back() == '\r') line.pop_back();
        if (line.empty() || line[0] == '%') continue;
        if (std::all_of(line.begin(), line.end(), [](unsigned char ch) { return std::isspace(ch); })) continue;
        return true;
    }
    return false;
}

std::uint64_t count_of(const std::string& tok, const char* what) {
    errno = 0;
    char* end = nullptr;
    const long long v = std::strtoll(tok.c_str(), &end, 10);
    if (end != tok.c_str() + tok.size() || errno == ERANGE || v < 0)
        throw Error(ErrorKind::MalformedEntry, std::string("bad ") + what + " '" + tok + "' in size line");
    return static_cast<std::uint64_t>(v);
}

std::uint64_t index_of(const std::string& tok, std::uint64_t limit, const char* axis, std::uint64_t e) {
    errno = 0;
    char* end = nullptr;
    const long long v = std::strtoll(tok.c_str(), &end, 10);
    if (end != tok.c_str() + tok.size() || errno == ERANGE)
        throw Error(ErrorKind::MalformedEntry,
                    "entry " + std::to_string(e) + ": bad " + axis + " index '" + tok + "'");
    if (v < 1 || static_cast<std::uint64_t>(v) > limit)
        throw Error(ErrorKind::IndexOutOfRange, "entry " + std::to_string(e) + ": " + axis + " index " +
                                                    std::to_string(v) + " outside [1, " +
                                                    std::to_string(limit) + "]");
    return static_cast<std::uint64_t>(v);
}

double value_of(const std::string& tok, std::uint64_t e) {
    char* end = nullptr;
    const double v = std::strtod(tok.c_str(), &end);
    if (end != tok.c_str() + tok.size())
        throw Error(ErrorKind::MalformedEntry, "entry " + std::to_string(e) + ": bad value '" + tok + "'");
    return v;
}

struct Entry {
    std::uint64_t i, j;
    double v;
};

// One pass over the file.  With `sink` null only the statistics are formed.
SparseMatrixStats scan(const std::string& path, std::vector<Entry>* sink) {
    std::ifstream in(path);
    if (!in) throw Error(ErrorKind::IoError, "cannot open '" + path + "'");
    std::string line;
    if (!std::getline(in, line)) throw Error(ErrorKind::BadBanner, "empty stream");
    const Banner b = banner_of(line);
    if (!b.coordinate) throw Error(ErrorKind::UnsupportedFormat, "array format carries no nnz; coordinate only");
    if (!data_line(in, line)) throw Error(ErrorKind::TruncatedFile, "missing size line");
    const auto st = tokens_of(line);
    if (st.size() != 3) throw Error(ErrorKind::MalformedEntry, "size line must be 'rows cols nnz'");
    const std::uint64_t rows = count_of(st[0], "row count");
    const std::uint64_t cols = count_of(st[1], "column count");
    const std::uint64_t declared = count_of(st[2], "entry count");
    const size_t want = b.field == Field::Pattern ? 2 : (b.field == Field::Complex ? 4 : 3);
    const bool expand = b.symm != Symm::General, skew = b.symm == Symm::Skew;
    if (sink && b.field == Field::Complex)
        throw Error(ErrorKind::UnsupportedFormat, "complex values cannot feed the FP64 SpMV");
    std::uint64_t nnz = 0;
    for (std::uint64_t e = 1; e <= declared; ++e) {
        if (!data_line(in, line))
            throw Error(ErrorKind::TruncatedFile, "declared " + std::to_string(declared) + " entries, found " +
                                                      std::to_string(e - 1));
        const auto t = tokens_of(line);
        if (t.size() != want)
            throw Error(ErrorKind::MalformedEntry, "entry " + std::to_string(e) + ": expected " +
                                                       std::to_string(want) + " tokens, got " +
                                                       std::to_string(t.size()));
        const std::uint64_t i = index_of(t[0], rows, "row", e);
        const std::uint64_t j = index_of(t[1], cols, "column", e);
        double v = 1.0;
        for (size_t k = 2; k < want; ++k) {
            const double x = value_of(t[k], e);
            if (k == 2) v = x;
        }
        if (!expand) {
            nnz += 1;
        } else if (i == j) {
            if (skew)
                throw Error(ErrorKind::MalformedEntry,
                            "entry " + std::to_string(e) + ": skew-symmetric matrices have zero diagonal");
            nnz += 1;
        } else {
            nnz += 2;
        }
        if (sink) {
            sink->push_back({i - 1, j - 1, v});
            if (expand && i != j) sink->push_back({j - 1, i - 1, skew ? -v : v});
        }
    }
    if (data_line(in, line))
        throw Error(ErrorKind::MalformedEntry, "more entries than the declared " + std::to_string(declared));
    SparseMatrixStats s{rows, cols, nnz};
    s.validate();
    return s;
}

}  // namespace

SparseMatrixStats mtx_stats(const std::string& path) { return scan(path, nullptr); }

SparseMatrixStats mtx_read_csr(const std::string& path, std::vector<std::int32_t>& row_ptr,
                               std::vector<std::int32_t>& col, std::vector<double>& val) {
    std::vector<Entry> es;
    const SparseMatrixStats s = scan(path, &es);
    if (s.rows > 0x7fffffffull || s.cols > 0x7fffffffull || s.nnz > 0x7fffffffull)
        throw Error(ErrorKind::InvalidRange, "int32 CSR indices cannot address this matrix");
    std::stable_sort(es.begin(), es.end(), [](const Entry& a, const Entry& b) {
        return a.i != b.i ? a.i < b.i : a.j < b.j;
    });
    row_ptr.assign(s.rows + 1, 0);
    col.resize(es.size());
    val.resize(es.size());
    for (size_t k = 0; k < es.size(); ++k) {
        row_ptr[es[k].i + 1] += 1;
        col[k] = static_cast<std::int32_t>(es[k].j);
        val[k] = es[k].v;
    }
    std::partial_sum(row_ptr.begin(), row_ptr.end(), row_ptr.begin());
    return s;
}

}  // namespace rooflens::b200
