// sngb/io.hpp -- SNGD binary datasets and label files for the C++ mirror
// (SURVEY.md section 8(f)), same layout, names, messages and error types as the
// reference:
//   layout            proj/include/sng/io.hpp:28-31 -- "SNGD", version byte 1,
//                     little-endian u64 n and dim, n*dim little-endian doubles
//   save/load_binary  proj/src/io.cpp:123-155
//   save/load_labels  proj/src/io.cpp:168-193 -- one integer per line, noise "-1"
//   ParseError/IoError proj/include/sng/errors.hpp
// A loaded file is an sng::Dataset of fp64 rows, so it runs the exact fp64
// entry points unless fp32 holds every value.
#pragma once

#include <charconv>
#include <cstdint>
#include <cstdio>
#include <cstring>
#include <fstream>
#include <span>
#include <stdexcept>
#include <string>
#include <vector>

#include "sngb/sng.hpp"

namespace sng {

class ParseError : public std::runtime_error {
public:
    ParseError(const std::string& message, std::size_t line = 0)
        : std::runtime_error(line > 0 ? "line " + std::to_string(line) + ": " + message : message),
          line_(line) {}
    std::size_t line() const { return line_; }

private:
    std::size_t line_;
};

class IoError : public std::runtime_error {
public:
    explicit IoError(const std::string& message) : std::runtime_error(message) {}
};

namespace sngd {
inline constexpr char kMagic[4] = {'S', 'N', 'G', 'D'};
inline constexpr std::uint8_t kVersion = 1;
}  // namespace sngd

inline void save_binary(const Dataset& data, const std::string& path) {
    std::ofstream out(path, std::ios::binary);
    if (!out) throw IoError("cannot open '" + path + "' for writing");
    const std::vector<double> v = data.values();
    const std::uint64_t n = data.size(), dim = data.dim();
    out.write(sngd::kMagic, 4);
    out.put(static_cast<char>(sngd::kVersion));
    out.write(reinterpret_cast<const char*>(&n), sizeof(n));  // little-endian hosts
    out.write(reinterpret_cast<const char*>(&dim), sizeof(dim));
    out.write(reinterpret_cast<const char*>(v.data()),
              static_cast<std::streamsize>(v.size() * sizeof(double)));
    if (!out) throw IoError("error while writing '" + path + "'");
}

inline Dataset load_binary(const std::string& path) {
    std::ifstream in(path, std::ios::binary);
    if (!in) throw IoError("cannot open '" + path + "' for reading");
    char magic[4];
    in.read(magic, 4);
    if (!in || std::memcmp(magic, sngd::kMagic, 4) != 0)
        throw ParseError("file '" + path + "' is not an SNGD binary dataset");
    const int version = in.get();
    if (version != sngd::kVersion)
        throw ParseError("unsupported SNGD version " + std::to_string(version));
    std::uint64_t n = 0, dim = 0;
    in.read(reinterpret_cast<char*>(&n), sizeof(n));
    in.read(reinterpret_cast<char*>(&dim), sizeof(dim));
    if (!in || n == 0 || dim == 0) throw ParseError("corrupt SNGD header in '" + path + "'");
    std::vector<double> values(n * dim);
    in.read(reinterpret_cast<char*>(values.data()),
            static_cast<std::streamsize>(values.size() * sizeof(double)));
    if (!in) throw ParseError("truncated SNGD payload in '" + path + "'");
    return Dataset(std::move(values), dim);
}

inline void save_labels(std::span<const std::int32_t> labels, const std::string& path) {
    std::FILE* f = std::fopen(path.c_str(), "w");
    if (!f) throw IoError("cannot open '" + path + "' for writing");
    for (std::int32_t v : labels) std::fprintf(f, "%d\n", v);
    if (std::fclose(f) != 0) throw IoError("error while writing '" + path + "'");
}

inline std::vector<std::int32_t> load_labels(const std::string& path) {
    std::ifstream in(path);
    if (!in) throw IoError("cannot open '" + path + "' for reading");
    std::vector<std::int32_t> labels;
    std::string line;
    std::size_t line_no = 0;
    while (std::getline(in, line)) {
        ++line_no;
        if (!line.empty() && line.back() == '\r') line.pop_back();
        if (line.empty()) continue;
        std::int32_t value = 0;
        const auto [ptr, ec] = std::from_chars(line.data(), line.data() + line.size(), value);
        if (ec != std::errc{} || ptr != line.data() + line.size())
            throw ParseError("label '" + line + "' is not an integer", line_no);
        labels.push_back(value);
    }
    return labels;
}

inline void save_clustering(const Clustering& c, const std::string& path) {
    save_labels(c.assignment, path);
}

}  // namespace sng
