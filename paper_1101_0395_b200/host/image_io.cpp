// image_io.cpp -- host file I/O of image.hpp and histogram.hpp (reference
// src/image.cpp:53-73,181-191,237-247; src/histogram.cpp:106-119): binary PPM,
// the palette text file and the histogram CSV. PNG needs libpng, which this
// build does not link.
#include <cctype>
#include <cerrno>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <fstream>

#include "context.hpp"

namespace quant {

namespace {
[[noreturn]] void io_fail(const std::string &path, const std::string &what) {
    throw std::runtime_error(path + ": " + what);
}

// next whitespace-delimited header token; '#' comments run to end of line.
// The delimiter after the token is consumed (so after maxval exactly one
// whitespace byte separates the header from the raster).
bool ppm_token(std::istream &in, std::string &tok) {
    tok.clear();
    for (int c = in.get(); c != EOF; c = in.get()) {
        if (c == '#') {
            while (c != EOF && c != '\n') c = in.get();
            if (c == EOF) break;
            continue;
        }
        if (std::isspace(c)) {
            if (tok.empty()) continue;
            return true;
        }
        tok.push_back(static_cast<char>(c));
    }
    return !tok.empty();
}

long ppm_field(std::istream &in, const std::string &path, const char *field) {
    std::string tok;
    if (!ppm_token(in, tok)) io_fail(path, std::string("truncated PPM header (missing ") + field + ")");
    char *end = nullptr;
    errno = 0;
    const long v = std::strtol(tok.c_str(), &end, 10);
    if (tok.empty() || *end != '\0' || errno != 0 || std::isspace(static_cast<unsigned char>(tok[0])))
        io_fail(path, std::string("malformed PPM ") + field + " '" + tok + "'");
    return v;
}

bool ends_with_ci(const std::string &s, const char *suffix) {
    const std::size_t n = std::strlen(suffix);
    if (s.size() < n) return false;
    for (std::size_t i = 0; i < n; ++i)
        if (std::tolower(static_cast<unsigned char>(s[s.size() - n + i])) != suffix[i]) return false;
    return true;
}
} // namespace

LoadedImage load_image(const std::string &path) {
    std::ifstream in(path, std::ios::binary);
    if (!in) io_fail(path, "cannot open file");
    char magic[2] = {0, 0};
    in.read(magic, 2);
    if (in.gcount() < 2) io_fail(path, "file too short to identify");
    if (magic[0] == '\x89' && magic[1] == 'P') io_fail(path, "PNG input needs libpng, which this build does not link");
    if (!(magic[0] == 'P' && magic[1] == '6'))
        io_fail(path, "unsupported format (expected binary PPM 'P6' or PNG)");
    const long w = ppm_field(in, path, "width");
    const long h = ppm_field(in, path, "height");
    const long maxval = ppm_field(in, path, "maxval");
    if (w <= 0 || h <= 0) io_fail(path, "non-positive PPM dimensions");
    if (maxval != 255) io_fail(path, "unsupported PPM maxval " + std::to_string(maxval) + " (only 255)");
    LoadedImage out;
    out.image.width = static_cast<int>(w);
    out.image.height = static_cast<int>(h);
    const std::size_t bytes = static_cast<std::size_t>(w) * static_cast<std::size_t>(h) * 3;
    out.image.pixels.resize(bytes / 3);
    in.read(reinterpret_cast<char *>(out.image.pixels.data()), static_cast<std::streamsize>(bytes));
    if (static_cast<std::size_t>(in.gcount()) != bytes)
        io_fail(path, "truncated PPM pixel data (expected " + std::to_string(bytes) + " bytes, got " +
                          std::to_string(in.gcount()) + ")");
    return out;
}

void save_ppm(const RawImage &image, const std::string &path) {
    if (image.width <= 0 || image.height <= 0 ||
        image.pixels.size() != static_cast<std::size_t>(image.width) * static_cast<std::size_t>(image.height))
        throw std::invalid_argument("save_ppm: inconsistent image dimensions");
    std::ofstream out(path, std::ios::binary);
    if (!out) io_fail(path, "cannot open file for writing");
    const std::string head = "P6\n" + std::to_string(image.width) + " " + std::to_string(image.height) + "\n255\n";
    out.write(head.data(), static_cast<std::streamsize>(head.size()));
    out.write(reinterpret_cast<const char *>(image.pixels.data()),
              static_cast<std::streamsize>(image.pixels.size() * 3));
    if (!out) io_fail(path, "write failed");
}

void save_image(const RawImage &image, const std::string &path) {
    if (ends_with_ci(path, ".ppm")) return save_ppm(image, path);
    if (ends_with_ci(path, ".png")) io_fail(path, "PNG output needs libpng, which this build does not link");
    io_fail(path, "unknown output extension (use .ppm or .png)");
}


void save_png(const RawImage &, const std::string &path) {
    io_fail(path, "PNG output needs libpng, which this build does not link");
}

void save_palette_text(const Palette &palette, const std::string &path) {
    if (palette.colors.empty()) throw std::invalid_argument("save_palette_text: empty palette");
    std::ofstream out(path);
    if (!out) io_fail(path, "cannot open file for writing");
    for (const ColorPoint &c : palette.colors) {
        const Rgb8 q = to_rgb8(c);
        out << int(q.r) << ' ' << int(q.g) << ' ' << int(q.b) << '\n';
    }
    if (!out) io_fail(path, "write failed");
}

void dump_histogram_csv(const WeightedHistogram &hist, const std::string &path) {
    std::ofstream out(path);
    if (!out) io_fail(path, "cannot open file for writing");
    out << "r,g,b,count,weight\n";
    char row[96];
    for (std::size_t i = 0; i < hist.size(); ++i) {
        std::snprintf(row, sizeof row, "%d,%d,%d,%u,%.9f\n", int(hist.colors[i].r), int(hist.colors[i].g),
                      int(hist.colors[i].b), hist.counts[i], hist.weights[i]);
        out << row;
    }
    if (!out) io_fail(path, "write failed");
}

} // namespace quant
