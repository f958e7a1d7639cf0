// Voxel colours, the dense test grid and dense primitives.
//
// voxel_color follows reference proj/src/ingest.cpp:24-29 (SplitMix64
// finaliser over x<<42 | y<<21 | z) and :67-85 (mode switch). The primitive
// occupancy rules follow ingest.cpp:193-266; the sphere rule is also the one
// the sparse procedural builder (procedural.cpp) evaluates per cube.
#include "voxanim/ingest.hpp"

#include <algorithm>
#include <bit>
#include <charconv>
#include <cmath>
#include <string>
#include <string_view>
#include <vector>

namespace voxanim {

namespace {

constexpr std::uint32_t kDenseDepthCap = 10; // reference ingest.cpp:15

std::uint64_t splitmix_finalize(std::uint64_t k) {
    k += 0x9e3779b97f4a7c15ull;
    k = (k ^ (k >> 30)) * 0xbf58476d1ce4e5b9ull;
    k = (k ^ (k >> 27)) * 0x94d049bb133111ebull;
    return k ^ (k >> 31);
}

std::uint8_t ramp8(double from, double to, double f) {
    return static_cast<std::uint8_t>(std::lround(from + (to - from) * f));
}

bool pow2(std::uint32_t v) { return v != 0 && (v & (v - 1)) == 0; }

} // namespace

VoxelAttribute voxel_color(const ColorSpec& spec, std::uint32_t resolution, std::uint32_t x, std::uint32_t y,
                           std::uint32_t z) {
    if (spec.mode == ColorMode::Constant) return spec.constant;
    if (spec.mode == ColorMode::ByHeight) {
        const double f = resolution > 1 ? static_cast<double>(y) / (resolution - 1) : 0.0;
        return {ramp8(40, 235, f), ramp8(90, 170, f), ramp8(200, 60, f), 255};
    }
    const std::uint64_t h = splitmix_finalize((std::uint64_t{x} << 42) | (std::uint64_t{y} << 21) | z);
    return {static_cast<std::uint8_t>(64 + (h & 0xbf)), static_cast<std::uint8_t>(64 + ((h >> 8) & 0xbf)),
            static_cast<std::uint8_t>(64 + ((h >> 16) & 0xbf)), 255};
}

VoxelGrid::VoxelGrid(std::uint32_t resolution, ColorSpec colors) : n_(resolution), colors_(colors) {
    if (!pow2(resolution))
        throw ValidationError("grid resolution must be a power of two, got " + std::to_string(resolution));
    if (resolution > (1u << kDenseDepthCap))
        throw ValidationError("grid resolution " + std::to_string(resolution) +
                              " exceeds the dense-grid cap of 2^" + std::to_string(kDenseDepthCap));
    const std::uint64_t cells = std::uint64_t{n_} * n_ * n_;
    words_.assign((cells + 63) / 64, 0);
}

std::uint32_t VoxelGrid::depth() const { return static_cast<std::uint32_t>(std::countr_zero(n_)); }

void VoxelGrid::set(std::uint32_t x, std::uint32_t y, std::uint32_t z, bool on) {
    const std::uint64_t i = linear(x, y, z);
    const std::uint64_t bit = std::uint64_t{1} << (i & 63);
    if (on)
        words_[i >> 6] |= bit;
    else
        words_[i >> 6] &= ~bit;
}

std::uint64_t VoxelGrid::set_count() const {
    std::uint64_t total = 0;
    for (const std::uint64_t w : words_) total += static_cast<std::uint64_t>(std::popcount(w));
    return total;
}

namespace {

template <class Pred> void fill_where(VoxelGrid& g, std::uint32_t side, Pred keep) {
    for (std::uint32_t x = 0; x < side; ++x)
        for (std::uint32_t y = 0; y < side; ++y)
            for (std::uint32_t z = 0; z < side; ++z)
                if (keep(x, y, z)) g.set(x, y, z);
}

bool in_menger(std::uint32_t x, std::uint32_t y, std::uint32_t z, std::uint32_t level) {
    for (; level > 0; --level, x /= 3, y /= 3, z /= 3)
        if ((x % 3 == 1) + (y % 3 == 1) + (z % 3 == 1) >= 2) return false;
    return true;
}

} // namespace

VoxelGrid gen_primitive(PrimitiveKind kind, std::uint32_t depth, ColorSpec colors) {
    if (depth < 1 || depth > kDenseDepthCap)
        throw ValidationError("primitive depth must be in [1, 10], got " + std::to_string(depth));
    if (kind == PrimitiveKind::Menger) {
        std::uint32_t side = 1;
        for (std::uint32_t i = 0; i < depth; ++i) side *= 3;
        VoxelGrid g(std::bit_ceil(side), colors);
        fill_where(g, side, [&](auto x, auto y, auto z) { return in_menger(x, y, z, depth); });
        return g;
    }
    const std::uint32_t n = 1u << depth;
    VoxelGrid g(n, colors);
    switch (kind) {
    case PrimitiveKind::Sphere: {
        // (x+.5-c)^2 + (y+.5-c)^2 + (z+.5-c)^2 <= c^2, c = n/2 (exact in FP64).
        const double c = n * 0.5;
        fill_where(g, n, [&](auto x, auto y, auto z) {
            const double dx = x + 0.5 - c, dy = y + 0.5 - c, dz = z + 0.5 - c;
            return dx * dx + dy * dy + dz * dz <= c * c;
        });
        break;
    }
    case PrimitiveKind::BoxShell:
        fill_where(g, n, [&](auto x, auto y, auto z) {
            return x == 0 || y == 0 || z == 0 || x == n - 1 || y == n - 1 || z == n - 1;
        });
        break;
    case PrimitiveKind::Checker:
        fill_where(g, n, [](auto x, auto y, auto z) { return ((x + y + z) & 1u) == 0; });
        break;
    default:
        throw ValidationError("unknown primitive kind");
    }
    return g;
}

PrimitiveKind primitive_kind_from_name(const std::string& name) {
    if (name == "sphere") return PrimitiveKind::Sphere;
    if (name == "box_shell") return PrimitiveKind::BoxShell;
    if (name == "menger") return PrimitiveKind::Menger;
    if (name == "checker") return PrimitiveKind::Checker;
    throw ValidationError("unknown shape \"" + name + "\"; expected sphere, box_shell, menger, or checker");
}

namespace {

// Whitespace-separated fields of one header line.
std::vector<std::string_view> fields_of(std::string_view line) {
    std::vector<std::string_view> out;
    std::size_t i = 0;
    while (i < line.size()) {
        while (i < line.size() && (line[i] == ' ' || line[i] == '\t')) ++i;
        std::size_t j = i;
        while (j < line.size() && line[j] != ' ' && line[j] != '\t') ++j;
        if (j > i) out.push_back(line.substr(i, j - i));
        i = j;
    }
    return out;
}

// leading integer of a field, as `istream >> long long` reads it
bool integer_field(std::string_view f, long long& v) {
    if (!f.empty() && f[0] == '+') f.remove_prefix(1);
    const auto [end, ec] = std::from_chars(f.data(), f.data() + f.size(), v);
    return ec == std::errc{};
}

} // namespace

VoxelGrid parse_binvox(std::span<const std::uint8_t> bytes) {
    const std::string_view text(reinterpret_cast<const char*>(bytes.data()), bytes.size());
    std::size_t pos = 0;
    // one header line ('\n'-terminated, a trailing '\r' dropped)
    const auto line = [&]() {
        if (pos >= text.size()) throw ParseError("binvox: truncated header");
        std::size_t eol = text.find('\n', pos);
        if (eol == std::string_view::npos) eol = text.size();
        std::string_view l = text.substr(pos, eol - pos);
        pos = std::min(text.size(), eol + 1);
        if (!l.empty() && l.back() == '\r') l.remove_suffix(1);
        return l;
    };
    {
        const auto f = fields_of(line());
        long long version = -1;
        if (f.size() < 2 || f[0] != "#binvox" || !integer_field(f[1], version) || version != 1)
            throw ParseError("binvox: bad header, expected \"#binvox 1\"");
    }
    // dim lists depth, height, width: the x, z and y extents
    std::uint64_t nx = 0, nz = 0, ny = 0;
    bool dims = false;
    for (bool data = false; !data;) {
        const auto f = fields_of(line());
        if (f.empty()) continue;
        if (f[0] == "data") {
            data = true;
        } else if (f[0] == "dim") {
            long long d[3] = {-1, -1, -1};
            for (int k = 0; k < 3; ++k)
                if (f.size() > static_cast<std::size_t>(k + 1) && !integer_field(f[k + 1], d[k])) d[k] = -1;
            if (d[0] <= 0 || d[1] <= 0 || d[2] <= 0) throw ParseError("binvox: bad dim line");
            nx = static_cast<std::uint64_t>(d[0]);
            nz = static_cast<std::uint64_t>(d[1]);
            ny = static_cast<std::uint64_t>(d[2]);
            dims = true;
        } // translate, scale and unknown keywords carry no voxels
    }
    if (!dims) throw ParseError("binvox: missing dim line");
    const std::uint64_t extent = std::max({nx, ny, nz});
    if (extent > (std::uint64_t{1} << kDenseDepthCap))
        throw ParseError("binvox: dimensions too large for the dense-grid cap");
    VoxelGrid grid(std::bit_ceil(static_cast<std::uint32_t>(extent)));

    const std::uint64_t total = nx * ny * nz, slab = ny * nz;
    std::uint64_t done = 0;
    for (; pos < text.size(); pos += 2) {
        if (pos + 1 >= text.size()) throw ParseError("binvox: truncated RLE stream (dangling value byte)");
        const std::uint8_t value = bytes[pos], count = bytes[pos + 1];
        if (value > 1 || count == 0) throw ParseError("binvox: invalid RLE pair");
        if (done + count > total) throw ParseError("binvox: RLE run count exceeds dim product");
        if (value)
            for (std::uint64_t i = done; i < done + count; ++i)
                grid.set(static_cast<std::uint32_t>(i / slab), static_cast<std::uint32_t>(i % ny),
                         static_cast<std::uint32_t>((i % slab) / ny));
        done += count;
    }
    if (done != total)
        throw ParseError("binvox: RLE decodes " + std::to_string(done) + " voxels, dim product is " +
                         std::to_string(total));
    return grid;
}

} // namespace voxanim
