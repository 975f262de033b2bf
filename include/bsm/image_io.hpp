// bsm/image_io.hpp -- the reference's image and disparity file layer
// (image_io.hpp:238-382), host-side: PGM/PPM (P2/P3/P5/P6, 8/16-bit), PFM and
// PNG readers; 16-bit PGM / PFM disparity writers; 8-bit PGM and PPM writers.
// Same outcomes and messages as the reference.  PNG: 8-bit gray, RGB and
// palette images, non-interlaced, inflated with zlib (link with -lz); other
// PNG variants raise FormatError.
#pragma once

#include <zlib.h>

#include <bit>
#include <cctype>
#include <cmath>
#include <cstdint>
#include <cstring>
#include <fstream>
#include <iterator>
#include <limits>
#include <string>
#include <vector>

#include "bsm/errors.hpp"
#include "bsm/image.hpp"

namespace bsm {
namespace io_detail {

inline std::vector<uint8_t> slurp(const std::string& path) {
    std::ifstream f(path, std::ios::binary);
    if (!f) throw IoError("cannot open " + path);
    std::vector<uint8_t> bytes((std::istreambuf_iterator<char>(f)), std::istreambuf_iterator<char>());
    if (f.bad()) throw IoError("read failed on " + path);
    return bytes;
}

inline void spill(const std::string& path, const std::string& head, const void* body, std::size_t n) {
    std::ofstream f(path, std::ios::binary);
    if (!f) throw IoError("cannot open " + path + " for writing");
    f.write(head.data(), std::streamsize(head.size()));
    f.write(static_cast<const char*>(body), std::streamsize(n));
    if (!f) throw IoError("write failed on " + path);
}

// Header tokens: whitespace separated, '#' comments to end of line.
struct Tokens {
    const std::vector<uint8_t>& b;
    std::size_t at = 0;

    static bool ws(uint8_t c) { return std::isspace(c) != 0; }
    std::string next(const char* what) {
        for (;;) {
            while (at < b.size() && ws(b[at])) ++at;
            if (at < b.size() && b[at] == '#') {
                while (at < b.size() && b[at] != '\n') ++at;
                continue;
            }
            break;
        }
        const std::size_t s = at;
        while (at < b.size() && !ws(b[at]) && b[at] != '#') ++at;
        if (at == s) throw FormatError(std::string("missing ") + what + " in PNM header");
        return std::string(reinterpret_cast<const char*>(b.data()) + s, at - s);
    }
    long integer(const char* what) {
        const std::string t = next(what);
        std::size_t used = 0;
        long v = 0;
        try {
            v = std::stol(t, &used);
        } catch (const std::exception&) {
            throw FormatError(std::string("bad ") + what + " '" + t + "' in PNM header");
        }
        if (used != t.size()) throw FormatError(std::string("bad ") + what + " in PNM header");
        return v;
    }
    void one_space() {
        if (at >= b.size() || !ws(b[at])) throw FormatError("missing separator before PNM payload");
        ++at;
    }
};

struct Pnm {
    char kind;  // '2', '3', '5', '6'
    int w, h;
    long maxval;
    std::vector<uint16_t> samples;
};

inline Pnm read_pnm(const std::vector<uint8_t>& b, bool allow_colour, const std::string& path) {
    Tokens t{b};
    const std::string magic = t.next("magic");
    if (magic.size() != 2 || magic[0] != 'P' || std::strchr("2356", magic[1]) == nullptr)
        throw FormatError("unsupported PNM magic '" + magic + "'");
    Pnm p{magic[1], 0, 0, 0, {}};
    const long w = t.integer("width"), h = t.integer("height");
    p.maxval = t.integer("maxval");
    if (w < 1 || h < 1 || w > (1L << 20) || h > (1L << 20)) throw FormatError("bad PNM dimensions");
    if (p.maxval < 1 || p.maxval > 65535) throw FormatError("bad PNM maxval");
    p.w = int(w);
    p.h = int(h);
    const bool colour = p.kind == '3' || p.kind == '6';
    if (colour && !allow_colour) throw FormatError("disparity PGM must be grayscale: " + path);
    const std::size_t count = std::size_t(p.w) * std::size_t(p.h) * (colour ? 3 : 1);
    p.samples.resize(count);
    if (p.kind == '2' || p.kind == '3') {
        for (std::size_t i = 0; i < count; ++i) {
            const long v = t.integer("sample");
            if (v < 0 || v > p.maxval) throw FormatError("PNM sample out of range");
            p.samples[i] = uint16_t(v);
        }
        return p;
    }
    t.one_space();
    const std::size_t bps = p.maxval > 255 ? 2 : 1;
    if (b.size() - t.at < count * bps) throw FormatError("truncated PNM payload");
    const uint8_t* s = b.data() + t.at;
    for (std::size_t i = 0; i < count; ++i)
        p.samples[i] = bps == 1 ? s[i] : uint16_t((unsigned(s[2 * i]) << 8) | s[2 * i + 1]);  // big-endian
    return p;
}

inline uint8_t to8(uint16_t v, long maxval) {
    return maxval == 255 ? uint8_t(v) : uint8_t((long(v) * 255 + maxval / 2) / maxval);
}

inline bool is_png(const std::vector<uint8_t>& b) {
    static const uint8_t sig[8] = {0x89, 'P', 'N', 'G', '\r', '\n', 0x1a, '\n'};
    return b.size() >= 8 && std::memcmp(b.data(), sig, 8) == 0;
}

// 8-bit gray / RGB / palette PNG -> rows of 1 or 3 channels (channels = 3
// expands gray; channels = 1 rejects colour).
inline std::vector<uint8_t> read_png(const std::vector<uint8_t>& b, const std::string& path, int channels,
                                     int& w, int& h) {
    auto bad = [&](const std::string& m) { return FormatError("bad PNG " + path + ": " + m); };
    auto be32 = [&](std::size_t o) {
        return (uint32_t(b[o]) << 24) | (uint32_t(b[o + 1]) << 16) | (uint32_t(b[o + 2]) << 8) | b[o + 3];
    };
    std::size_t o = 8;
    bool have_hdr = false;
    uint8_t depth = 0, ctype = 0, interlace = 0;
    std::vector<uint8_t> plte, z;
    while (o + 8 <= b.size()) {
        const uint32_t len = be32(o);
        if (o + 12 + std::size_t(len) > b.size()) throw bad("truncated chunk");
        const uint8_t* type = &b[o + 4];
        const uint8_t* body = &b[o + 8];
        if (uint32_t(crc32(crc32(0L, type, 4), body, len)) != be32(o + 8 + len)) throw bad("CRC error");
        if (!std::memcmp(type, "IHDR", 4) && len >= 13) {
            w = int(be32(o + 8));
            h = int(be32(o + 12));
            depth = body[8];
            ctype = body[9];
            if (body[10] != 0 || body[11] != 0 || w < 1 || h < 1) throw bad("invalid IHDR");
            interlace = body[12];
            have_hdr = true;
        } else if (!std::memcmp(type, "PLTE", 4)) {
            plte.assign(body, body + len);
        } else if (!std::memcmp(type, "IDAT", 4)) {
            z.insert(z.end(), body, body + len);
        } else if (!std::memcmp(type, "IEND", 4)) {
            break;
        }
        o += 12 + len;
    }
    if (!have_hdr || z.empty()) throw bad("missing IHDR/IDAT");
    if (depth != 8 || (ctype != 0 && ctype != 2 && ctype != 3) || interlace != 0)
        throw bad("unsupported PNG variant (this build reads 8-bit gray/RGB/palette, non-interlaced)");
    if (ctype == 3 && plte.empty()) throw bad("palette image without PLTE");
    const int bpp = ctype == 2 ? 3 : 1;
    const std::size_t stride = std::size_t(w) * bpp;
    std::vector<uint8_t> raw((stride + 1) * std::size_t(h));
    uLongf got = uLongf(raw.size());
    if (uncompress(raw.data(), &got, z.data(), uLong(z.size())) != Z_OK || got < raw.size())
        throw bad("corrupt or truncated image data");
    std::vector<uint8_t> img(stride * std::size_t(h));
    for (int y = 0; y < h; ++y) {
        const uint8_t f = raw[std::size_t(y) * (stride + 1)];
        const uint8_t* in = &raw[std::size_t(y) * (stride + 1) + 1];
        uint8_t* cur = &img[std::size_t(y) * stride];
        const uint8_t* up = y ? cur - stride : nullptr;
        for (std::size_t x = 0; x < stride; ++x) {
            const int a = x >= std::size_t(bpp) ? cur[x - bpp] : 0, u = up ? up[x] : 0;
            const int c = (up && x >= std::size_t(bpp)) ? up[x - bpp] : 0;
            int pred = 0;
            switch (f) {
                case 0: break;
                case 1: pred = a; break;
                case 2: pred = u; break;
                case 3: pred = (a + u) >> 1; break;
                case 4: {
                    const int pa = std::abs(u - c), pb = std::abs(a - c), pc = std::abs(a + u - 2 * c);
                    pred = (pa <= pb && pa <= pc) ? a : (pb <= pc ? u : c);
                    break;
                }
                default: throw bad("bad filter type");
            }
            cur[x] = uint8_t(in[x] + pred);
        }
    }
    if (ctype == 3) {
        if (channels != 3) throw bad("colour-to-gray conversion is not supported by this build");
        std::vector<uint8_t> rgb(std::size_t(w) * h * 3);
        for (std::size_t i = 0; i < img.size(); ++i) {
            if (3u * img[i] + 2 >= plte.size()) throw bad("palette index out of range");
            std::memcpy(&rgb[3 * i], &plte[3u * img[i]], 3);
        }
        return rgb;
    }
    if (ctype == 2) {
        if (channels != 3) throw bad("colour-to-gray conversion is not supported by this build");
        return img;
    }
    if (channels == 1) return img;
    std::vector<uint8_t> rgb(img.size() * 3);
    for (std::size_t i = 0; i < img.size(); ++i) rgb[3 * i] = rgb[3 * i + 1] = rgb[3 * i + 2] = img[i];
    return rgb;
}

inline long round_half_away(double v) { return std::lround(v); }

}  // namespace io_detail

// Decodes a PGM (P2/P5), PPM (P3/P6) or PNG; gray sources expand to r = g = b,
// 16-bit samples rescale to 8 bits.
inline RgbImage load_image(const std::string& path) {
    const std::vector<uint8_t> b = io_detail::slurp(path);
    if (b.empty()) throw FormatError("empty file " + path);
    if (io_detail::is_png(b)) {
        int w = 0, h = 0;
        const std::vector<uint8_t> rgb = io_detail::read_png(b, path, 3, w, h);
        RgbImage out(w, h);
        std::memcpy(out.pixels.data(), rgb.data(), rgb.size());
        return out;
    }
    const io_detail::Pnm p = io_detail::read_pnm(b, true, path);
    RgbImage out(p.w, p.h);
    const bool colour = p.kind == '3' || p.kind == '6';
    for (std::size_t i = 0; i < out.pixels.size(); ++i) {
        if (colour) {
            out.pixels[i] = {io_detail::to8(p.samples[3 * i], p.maxval), io_detail::to8(p.samples[3 * i + 1], p.maxval),
                             io_detail::to8(p.samples[3 * i + 2], p.maxval)};
        } else {
            const uint8_t g = io_detail::to8(p.samples[i], p.maxval);
            out.pixels[i] = {g, g, g};
        }
    }
    return out;
}

// Stored value / scale; PGM 0 and non-finite PFM values are unknown pixels.
inline DisparityMap load_gt_disparity(const std::string& path, double scale) {
    if (scale <= 0) throw InvalidArgument("disparity scale must be > 0");
    const std::vector<uint8_t> b = io_detail::slurp(path);
    if (b.empty()) throw FormatError("empty file " + path);
    if (b.size() >= 2 && b[0] == 'P' && (b[1] == 'f' || b[1] == 'F')) {
        io_detail::Tokens t{b};
        const std::string magic = t.next("magic");
        if (magic != "Pf" && magic != "PF") throw FormatError("bad PFM magic in " + path);
        const long w = t.integer("width"), h = t.integer("height");
        if (w < 1 || h < 1 || w > (1L << 20) || h > (1L << 20)) throw FormatError("bad PFM dimensions in " + path);
        const std::string st = t.next("scale");
        double fs = 0;
        try {
            fs = std::stod(st);
        } catch (const std::exception&) {
            throw FormatError("bad PFM scale in " + path);
        }
        if (fs == 0) throw FormatError("bad PFM scale in " + path);
        t.one_space();
        const std::size_t ch = magic == "PF" ? 3 : 1;
        const std::size_t count = std::size_t(w) * std::size_t(h) * ch;
        if (b.size() - t.at < count * 4) throw FormatError("truncated PFM payload in " + path);
        if (ch != 1) throw FormatError("disparity PFM must be grayscale: " + path);
        const bool swap = (fs > 0) != (std::endian::native == std::endian::big);
        DisparityMap out(static_cast<int>(w), static_cast<int>(h));
        for (long fy = 0; fy < h; ++fy) {  // rows are stored bottom-up
            for (long x = 0; x < w; ++x) {
                uint32_t u;
                std::memcpy(&u, &b[t.at + (std::size_t(fy) * std::size_t(w) + std::size_t(x)) * 4], 4);
                if (swap) u = __builtin_bswap32(u);
                float v;
                std::memcpy(&v, &u, 4);
                const std::size_t i = std::size_t(h - 1 - fy) * std::size_t(w) + std::size_t(x);
                out.disparity[i] = std::isfinite(v) ? float(v / scale) : 0.0f;
                out.valid[i] = std::isfinite(v) ? 1 : 0;
            }
        }
        return out;
    }
    int w = 0, h = 0;
    std::vector<uint16_t> stored;
    if (io_detail::is_png(b)) {
        const std::vector<uint8_t> g = io_detail::read_png(b, path, 1, w, h);
        stored.assign(g.begin(), g.end());
    } else {
        io_detail::Pnm p = io_detail::read_pnm(b, false, path);
        w = p.w;
        h = p.h;
        stored = std::move(p.samples);
    }
    DisparityMap out(w, h);
    for (std::size_t i = 0; i < stored.size(); ++i) {
        out.valid[i] = stored[i] != 0;
        out.disparity[i] = stored[i] ? float(stored[i] / scale) : 0.0f;
    }
    return out;
}

// 16-bit PGM of round(d * scale) clamped to [0, 65535]; invalid pixels store 0.
inline void save_disparity(const DisparityMap& m, const std::string& path, double scale) {
    if (scale <= 0) throw InvalidArgument("disparity scale must be > 0");
    std::vector<uint8_t> px(m.disparity.size() * 2);
    for (std::size_t i = 0; i < m.disparity.size(); ++i) {
        long v = m.valid[i] ? io_detail::round_half_away(double(m.disparity[i]) * scale) : 0;
        v = v < 0 ? 0 : (v > 65535 ? 65535 : v);
        px[2 * i] = uint8_t(v >> 8);
        px[2 * i + 1] = uint8_t(v & 0xff);
    }
    io_detail::spill(path, "P5\n" + std::to_string(m.width) + " " + std::to_string(m.height) + "\n65535\n",
                     px.data(), px.size());
}

// Grayscale PFM, host byte order, bottom-up rows, +inf for invalid pixels.
inline void save_disparity_pfm(const DisparityMap& m, const std::string& path) {
    std::vector<float> rows(m.disparity.size());
    const float inf = std::numeric_limits<float>::infinity();
    for (int y = 0; y < m.height; ++y)
        for (int x = 0; x < m.width; ++x) {
            const std::size_t i = std::size_t(y) * m.width + x;
            rows[std::size_t(m.height - 1 - y) * m.width + x] = m.valid[i] ? m.disparity[i] : inf;
        }
    const char* order = std::endian::native == std::endian::big ? "1.0" : "-1.0";
    io_detail::spill(path, "Pf\n" + std::to_string(m.width) + " " + std::to_string(m.height) + "\n" + order + "\n",
                     rows.data(), rows.size() * 4);
}

// 8-bit PGM of round(v) clamped to [0, 255] (stage visualisations, fixtures).
inline void save_gray_pgm(const GrayImage& g, const std::string& path) {
    std::vector<uint8_t> px(g.values.size());
    for (std::size_t i = 0; i < px.size(); ++i) {
        const float r = std::round(g.values[i]);
        px[i] = uint8_t(r < 0 ? 0 : (r > 255 ? 255 : r));
    }
    io_detail::spill(path, "P5\n" + std::to_string(g.width) + " " + std::to_string(g.height) + "\n255\n", px.data(),
                     px.size());
}

inline void save_ppm(const RgbImage& img, const std::string& path) {
    io_detail::spill(path, "P6\n" + std::to_string(img.width) + " " + std::to_string(img.height) + "\n255\n",
                     img.pixels.data(), img.pixels.size() * 3);
}

}  // namespace bsm
