// sngb/io.hpp -- SNGD binary datasets and label files for the C++ mirror
// (the data formats on either side of the hot path).
//
// The byte layout, function names, exception types and messages are the
// reference's compatibility contract and are kept:
//   layout              proj/include/sng/io.hpp:28-31 -- "SNGD", version byte 1,
//                       little-endian u64 n and dim, n*dim little-endian doubles
//   save/load_binary    proj/include/sng/io.hpp:30-31
//   load_points         proj/include/sng/io.hpp:34 (binary by magic; the CSV
//                       reader is outside this package's scope)
//   save/load_labels    proj/include/sng/io.hpp:37-42 -- one integer per line,
//                       noise "-1"
//   ParseError/IoError  proj/include/sng/errors.hpp
// The implementation is this package's own: whole-buffer stdio I/O with an
// explicit little-endian codec, and a reader that hands the rows to
// sng::Dataset, which keeps them as fp32 when fp32 holds every value (the
// fp32 entry points) and as fp64 otherwise (the exact fp64 entry points).
#pragma once

#include <algorithm>
#include <array>
#include <charconv>
#include <cstdint>
#include <cstdio>
#include <cstring>
#include <memory>
#include <span>
#include <stdexcept>
#include <string>
#include <string_view>
#include <vector>

#include "sngb/sng.hpp"

namespace sng {

// Malformed input; carries the 1-based line number when one applies.
class ParseError : public std::runtime_error {
public:
    explicit ParseError(const std::string& message, std::size_t line = 0)
        : std::runtime_error(with_line(message, line)), line_(line) {}
    std::size_t line() const { return line_; }

private:
    static std::string with_line(const std::string& m, std::size_t line) {
        return line == 0 ? m : "line " + std::to_string(line) + ": " + m;
    }
    std::size_t line_;
};

// Filesystem-level failure (missing file, unwritable path, short write).
class IoError : public std::runtime_error {
public:
    explicit IoError(const std::string& message) : std::runtime_error(message) {}
};

namespace sngd {

inline constexpr std::array<unsigned char, 4> kMagic{'S', 'N', 'G', 'D'};
inline constexpr int kVersion = 1;
inline constexpr std::size_t kHeaderBytes = 4 + 1 + 8 + 8;

struct FileCloser {
    void operator()(std::FILE* f) const {
        if (f) std::fclose(f);
    }
};
using File = std::unique_ptr<std::FILE, FileCloser>;

inline File open_or_throw(const std::string& path, const char* mode, const char* what) {
    File f(std::fopen(path.c_str(), mode));
    if (!f) throw IoError("cannot open '" + path + "' for " + what);
    return f;
}

inline void put_u64le(unsigned char* p, std::uint64_t v) {
    for (int i = 0; i < 8; ++i) p[i] = static_cast<unsigned char>(v >> (8 * i));
}
inline std::uint64_t get_u64le(const unsigned char* p) {
    std::uint64_t v = 0;
    for (int i = 7; i >= 0; --i) v = (v << 8) | p[i];
    return v;
}
inline void put_f64le(unsigned char* p, double x) {
    std::uint64_t bits;
    std::memcpy(&bits, &x, 8);
    put_u64le(p, bits);
}
inline double get_f64le(const unsigned char* p) {
    const std::uint64_t bits = get_u64le(p);
    double x;
    std::memcpy(&x, &bits, 8);
    return x;
}

// Closes f, reporting a failed flush as the reference does.
inline void close_written(File f, const std::string& path) {
    if (std::fclose(f.release()) != 0) throw IoError("error while writing '" + path + "'");
}

}  // namespace sngd

inline void save_binary(const Dataset& data, const std::string& path) {
    sngd::File f = sngd::open_or_throw(path, "wb", "writing");
    std::array<unsigned char, sngd::kHeaderBytes> head{};
    std::memcpy(head.data(), sngd::kMagic.data(), 4);
    head[4] = static_cast<unsigned char>(sngd::kVersion);
    sngd::put_u64le(head.data() + 5, data.size());
    sngd::put_u64le(head.data() + 13, data.dim());
    bool ok = std::fwrite(head.data(), 1, head.size(), f.get()) == head.size();
    // the payload in 64 KiB blocks of little-endian doubles
    const std::vector<double> v = data.values();
    std::vector<unsigned char> block(8 * 8192);
    for (std::size_t i = 0; ok && i < v.size(); i += 8192) {
        const std::size_t k = std::min<std::size_t>(8192, v.size() - i);
        for (std::size_t j = 0; j < k; ++j) sngd::put_f64le(block.data() + 8 * j, v[i + j]);
        ok = std::fwrite(block.data(), 8, k, f.get()) == k;
    }
    if (!ok) throw IoError("error while writing '" + path + "'");
    sngd::close_written(std::move(f), path);
}

inline Dataset load_binary(const std::string& path) {
    sngd::File f = sngd::open_or_throw(path, "rb", "reading");
    std::array<unsigned char, sngd::kHeaderBytes> head{};
    const std::size_t got = std::fread(head.data(), 1, head.size(), f.get());
    if (got < 4 || std::memcmp(head.data(), sngd::kMagic.data(), 4) != 0)
        throw ParseError("file '" + path + "' is not an SNGD binary dataset");
    const int version = got > 4 ? head[4] : -1;  // a missing byte reads as EOF (-1)
    if (version != sngd::kVersion)
        throw ParseError("unsupported SNGD version " + std::to_string(version));
    const std::uint64_t n = got == head.size() ? sngd::get_u64le(head.data() + 5) : 0;
    const std::uint64_t dim = got == head.size() ? sngd::get_u64le(head.data() + 13) : 0;
    if (n == 0 || dim == 0) throw ParseError("corrupt SNGD header in '" + path + "'");
    std::vector<double> values(n * dim);
    std::vector<unsigned char> block(8 * 8192);
    for (std::size_t i = 0; i < values.size(); i += 8192) {
        const std::size_t k = std::min<std::size_t>(8192, values.size() - i);
        if (std::fread(block.data(), 8, k, f.get()) != k)
            throw ParseError("truncated SNGD payload in '" + path + "'");
        for (std::size_t j = 0; j < k; ++j) values[i + j] = sngd::get_f64le(block.data() + 8 * j);
    }
    return Dataset(std::move(values), static_cast<std::size_t>(dim));
}

// The binary format, recognised by its magic (a CSV reader is not part of this
// package: such a file raises IoError).
inline Dataset load_points(const std::string& path) {
    {
        sngd::File f = sngd::open_or_throw(path, "rb", "reading");
        std::array<unsigned char, 4> m{};
        if (std::fread(m.data(), 1, 4, f.get()) == 4 && m == sngd::kMagic) {
            f.reset();
            return load_binary(path);
        }
    }
    throw IoError("'" + path + "' is not an SNGD dataset (CSV input is outside the GPU package)");
}

inline void save_labels(std::span<const std::int32_t> labels, const std::string& path) {
    sngd::File f = sngd::open_or_throw(path, "w", "writing");
    std::string text;
    text.reserve(labels.size() * 4);
    char num[16];
    for (std::int32_t v : labels) {
        const auto r = std::to_chars(num, num + sizeof(num), v);
        text.append(num, r.ptr);
        text.push_back('\n');
    }
    if (std::fwrite(text.data(), 1, text.size(), f.get()) != text.size())
        throw IoError("error while writing '" + path + "'");
    sngd::close_written(std::move(f), path);
}

inline std::vector<std::int32_t> load_labels(const std::string& path) {
    sngd::File f = sngd::open_or_throw(path, "r", "reading");
    std::string text;
    char buf[1 << 16];
    for (std::size_t k; (k = std::fread(buf, 1, sizeof(buf), f.get())) > 0;) text.append(buf, k);
    std::vector<std::int32_t> labels;
    std::size_t line_no = 0;
    for (std::size_t pos = 0; pos < text.size();) {
        std::size_t end = text.find('\n', pos);
        if (end == std::string::npos) end = text.size();
        ++line_no;
        std::string_view line(text.data() + pos, end - pos);
        pos = end + 1;
        if (!line.empty() && line.back() == '\r') line.remove_suffix(1);
        if (line.empty()) continue;
        std::int32_t value = 0;
        const auto r = std::from_chars(line.data(), line.data() + line.size(), value);
        if (r.ec != std::errc{} || r.ptr != line.data() + line.size())
            throw ParseError("label '" + std::string(line) + "' is not an integer", line_no);
        labels.push_back(value);
    }
    return labels;
}

inline void save_clustering(const Clustering& c, const std::string& path) {
    save_labels(c.assignment, path);
}

}  // namespace sng
