// latch_b200.hpp — C++ host face of the B200 CLATCH paths (header-only, over clatch.h).
//
// Mirrors the slice of the reference's C++ API that sits on the two hot paths, with the
// same names, argument meaning and error behaviour, so host code written against
// "latchkit" keeps compiling when it includes this header instead of
// latch/descriptor.hpp + latch/match.hpp (paths relative to /root/reference/proj):
//
//   describe_all / describe / keypoint_in_margin   include/latch/descriptor.hpp:48-67
//   match_brute_force / knn2 / hamming             include/latch/match.hpp:13-45
//   Image, Keypoint, Descriptor, TripletPattern,
//   WeightMask, Triplet, MatchOptions, MatchPair   image.hpp:12-29, detect.hpp:11-16,
//                                                  descriptor.hpp:31-42, pattern.hpp:19-52
//   Error / ErrorCode                              errors.hpp:10-56
//   parse_pattern / default_pattern                pattern.hpp:100-108
//   fast_detect / detect_and_orient                detect.hpp:18-40 (the step before the path)
//
// Everything per-sample / per-pair runs on the GPU through the C ABI; this header only
// converts containers, keeps the reference's early-outs and re-raises status codes as
// latch::Error. There is no CPU arithmetic path here: without a B200 every compute call
// throws. In a real integration the reference keeps its own type definitions and only the
// bodies of the functions below move (INTEGRATION.md shows the patch).
#pragma once

#include <algorithm>
#include <cctype>
#include <cmath>
#include <cstdint>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <exception>
#include <fstream>
#include <memory>
#include <mutex>
#include <optional>
#include <sstream>
#include <stdexcept>
#include <string>
#include <thread>
#include <utility>
#include <vector>

#include "clatch.h"

namespace latch {

// ---- errors (errors.hpp:10-56) ----------------------------------------------------
enum class ErrorCode {
    NotPGM, UnsupportedDepth, Truncated, Malformed, OutOfBounds, BadScale,
    ImageTooSmall, TooCloseToBorder,
    BadHeader, BadTripletCount, CoordinateOutOfRange, DegenerateTriplet, MissingInfo,
    GridSizeMismatch, LabelParse, NoPositives, NoNegatives, EmptyPairs, InsufficientCandidates,
    LengthMismatch, EmptyGallery,
    NoKeypoints,
    DeviceUnavailable   // extension: the GPU path could not run (no CPU fallback exists)
};

inline const char* error_code_name(ErrorCode code) {
    static const char* const names[] = {
        "NotPGM", "UnsupportedDepth", "Truncated", "Malformed", "OutOfBounds", "BadScale",
        "ImageTooSmall", "TooCloseToBorder", "BadHeader", "BadTripletCount", "CoordinateOutOfRange",
        "DegenerateTriplet", "MissingInfo", "GridSizeMismatch", "LabelParse", "NoPositives",
        "NoNegatives", "EmptyPairs", "InsufficientCandidates", "LengthMismatch", "EmptyGallery",
        "NoKeypoints", "DeviceUnavailable"};
    return names[static_cast<int>(code)];
}

class Error : public std::runtime_error {
public:
    Error(ErrorCode code, const std::string& message)
        : std::runtime_error(prefixed(code, message)), code_(code) {}
    ErrorCode code() const noexcept { return code_; }

private:
    static std::string prefixed(ErrorCode code, const std::string& m) {
        const std::string name = error_code_name(code);
        return m.compare(0, name.size(), name) == 0 ? m : name + ": " + m;
    }
    ErrorCode code_;
};

[[noreturn]] inline void raise(ErrorCode code, const std::string& message) { throw Error(code, message); }

// ---- data types ---------------------------------------------------------------------
inline constexpr int kWindowSize = 64;
inline constexpr int kDefaultPatchSize = 8;
inline constexpr int kDefaultBitCount = 512;
inline constexpr int kWindowMargin = 46;

struct Image {   // image.hpp:12-29: row-major doubles, pixel centres at integers
    int width = 0, height = 0;
    std::vector<double> data;
    Image() = default;
    Image(int w, int h) : width(w), height(h), data(static_cast<std::size_t>(w) * h, 0.0) {}
    Image(int w, int h, std::vector<double> v) : width(w), height(h), data(std::move(v)) {}
    double at(int x, int y) const { return data[static_cast<std::size_t>(y) * width + x]; }
    double& at(int x, int y) { return data[static_cast<std::size_t>(y) * width + x]; }
};

struct Keypoint { double x = 0, y = 0, theta = 0, score = 0; };   // detect.hpp:11-16

struct Descriptor {   // descriptor.hpp:31-42: bit t in byte t/8, position t%8
    std::vector<std::uint8_t> bytes;
    bool bit(std::size_t t) const { return (bytes[t >> 3] >> (t & 7)) & 1u; }
    void set_bit(std::size_t t, bool v) {
        const auto b = static_cast<std::uint8_t>(1u << (t & 7));
        if (v) bytes[t >> 3] |= b; else bytes[t >> 3] &= static_cast<std::uint8_t>(~b);
    }
    std::size_t bit_count() const { return bytes.size() * 8; }
    bool operator==(const Descriptor& o) const { return bytes == o.bytes; }
};

struct Triplet { int ax = 0, ay = 0, bx = 0, by = 0, cx = 0, cy = 0; };   // pattern.hpp:19-25

struct WeightMask {   // pattern.hpp:30-42
    int size = kDefaultPatchSize;
    std::vector<double> weights;
    static WeightMask ones(int size = kDefaultPatchSize) {
        WeightMask m; m.size = size; m.weights.assign(static_cast<std::size_t>(size) * size, 1.0); return m;
    }
    static WeightMask seven_by_seven() {
        WeightMask m = ones(kDefaultPatchSize);
        for (int i = 0; i < 8; ++i) m.weights[7 * 8 + i] = m.weights[i * 8 + 7] = 0.0;
        return m;
    }
};

struct TripletPattern {   // pattern.hpp:46-52
    int bit_count = kDefaultBitCount;
    int patch_size = kDefaultPatchSize;
    std::vector<Triplet> triplets;
    WeightMask mask;
};

struct MatchPair { int probe_index = 0, gallery_index = 0, distance = 0, second_distance = 0; };

struct MatchOptions {   // match.hpp:20-25
    std::optional<double> ratio;
    bool cross_check = false;
    std::optional<int> max_distance;
    int workers = 0;   // accepted for source compatibility; the GPU grid replaces the thread fan-out
};

struct Knn2Result { int best_index = -1, best_distance = 0, second_distance = 0; };

// ---- the shared GPU context -----------------------------------------------------------
namespace b200 {

[[noreturn]] inline void rethrow(int rc) {
    const std::string msg = clatch_last_error();
    if (rc >= 100 && rc <= 121) throw Error(static_cast<ErrorCode>(rc - 100), msg);   // 100 + ErrorCode
    if (rc == CLATCH_ERR_NONFINITE) throw Error(ErrorCode::OutOfBounds, msg);
    if (rc == CLATCH_ERR_INVALID) throw std::invalid_argument(msg);
    throw Error(ErrorCode::DeviceUnavailable, msg);
}

inline void check(int rc) { if (rc != CLATCH_OK) rethrow(rc); }

struct Context {
    clatch_ctx* ctx = nullptr;
    std::mutex mutex;                 // one ctx: calls are serialised (clatch.h threading note)
    const void* pattern_tag = nullptr;
    std::vector<std::int16_t> pattern_coords;
    std::vector<double> pattern_weights;
    int pattern_t = 0, pattern_k = 0;
    ~Context() { if (ctx) clatch_ctx_destroy(ctx); }
};

inline Context& context() {
    static Context c;
    if (!c.ctx) {
        const char* dev = std::getenv("CLATCH_DEVICE");
        check(clatch_ctx_create(dev ? std::atoi(dev) : 0, &c.ctx));
    }
    return c;
}

// One context per entry of a device list (the same device may appear more than once: each entry gets its
// own context, stream and scratch). Used by the sharded helpers at the end of this header, which run one
// host thread per entry — the C++ counterpart of paper_1609_03986_b200/sharded.py's one process per GPU.
struct ContextPool {
    std::vector<std::unique_ptr<Context>> slots;
    explicit ContextPool(const std::vector<int>& devices) {
        for (int d : devices) {
            slots.emplace_back(new Context);
            check(clatch_ctx_create(d, &slots.back()->ctx));
        }
    }
};

// Installs `pattern` unless the very same table is already on the device.
inline void use_pattern(Context& c, const TripletPattern& pattern) {
    std::vector<std::int16_t> coords;
    coords.reserve(pattern.triplets.size() * 6);
    for (const Triplet& t : pattern.triplets)
        for (int v : {t.ax, t.ay, t.bx, t.by, t.cx, t.cy}) coords.push_back(static_cast<std::int16_t>(v));
    if (c.pattern_t == pattern.bit_count && c.pattern_k == pattern.patch_size && c.pattern_coords == coords &&
        c.pattern_weights == pattern.mask.weights)
        return;
    if (static_cast<int>(pattern.triplets.size()) != pattern.bit_count ||
        static_cast<int>(pattern.mask.weights.size()) != pattern.patch_size * pattern.patch_size)
        raise(ErrorCode::BadTripletCount, "pattern tables do not match T / K");
    check(clatch_set_pattern(c.ctx, coords.data(), pattern.bit_count, pattern.patch_size,
                             pattern.mask.weights.data()));
    c.pattern_t = pattern.bit_count;
    c.pattern_k = pattern.patch_size;
    c.pattern_coords = std::move(coords);
    c.pattern_weights = pattern.mask.weights;
}

inline std::vector<std::uint8_t> flatten(const std::vector<Descriptor>& set, std::size_t bytes) {
    std::vector<std::uint8_t> flat(set.size() * bytes);
    for (std::size_t i = 0; i < set.size(); ++i) {
        if (set[i].bytes.size() != bytes)   // hamming's check, src/match.cpp:15-18
            raise(ErrorCode::LengthMismatch, "descriptor lengths differ: " + std::to_string(bytes) + " vs " +
                                                 std::to_string(set[i].bytes.size()));
        std::memcpy(flat.data() + i * bytes, set[i].bytes.data(), bytes);
    }
    return flat;
}

} // namespace b200

// ---- pattern text (pattern.hpp:100-108; src/pattern.cpp:68-131) ---------------------------
inline TripletPattern parse_pattern(const std::string& text) {
    std::istringstream in(text);
    std::string line;
    if (!std::getline(in, line)) raise(ErrorCode::BadHeader, "empty pattern file");
    int T = 0, K = 0;
    if (std::sscanf(line.c_str(), "LATCHPAT v1 T=%d K=%d", &T, &K) != 2)
        raise(ErrorCode::BadHeader, "bad header line '" + line + "'");
    if (T <= 0 || T % 8 != 0) raise(ErrorCode::BadHeader, "T must be a positive multiple of 8, got " + std::to_string(T));
    if (K < 1 || K > kWindowSize) raise(ErrorCode::BadHeader, "K out of range: " + std::to_string(K));
    TripletPattern p;
    p.bit_count = T;
    p.patch_size = K;
    bool weights = false;
    while (std::getline(in, line)) {
        if (line.empty()) continue;
        if (line == "WEIGHTS") { weights = true; break; }
        if (static_cast<int>(p.triplets.size()) == T)
            raise(ErrorCode::BadTripletCount, "more than T=" + std::to_string(T) + " triplet lines");
        Triplet t;
        if (std::sscanf(line.c_str(), "%d %d %d %d %d %d", &t.ax, &t.ay, &t.bx, &t.by, &t.cx, &t.cy) != 6)
            raise(ErrorCode::BadTripletCount, "bad triplet line '" + line + "'");
        for (int c : {t.ax, t.ay, t.bx, t.by, t.cx, t.cy})
            if (c < 0 || c > kWindowSize - K)
                raise(ErrorCode::CoordinateOutOfRange, "coordinate " + std::to_string(c) + " outside [0, " +
                                                           std::to_string(kWindowSize - K) + "]");
        if (t.bx == t.cx && t.by == t.cy)
            raise(ErrorCode::DegenerateTriplet, "companion patches coincide at (" + std::to_string(t.bx) + ", " +
                                                    std::to_string(t.by) + ")");
        p.triplets.push_back(t);
    }
    if (static_cast<int>(p.triplets.size()) != T)
        raise(ErrorCode::BadTripletCount, "expected " + std::to_string(T) + " triplets, got " +
                                              std::to_string(p.triplets.size()));
    if (!weights) { p.mask = WeightMask::ones(K); return p; }
    p.mask.size = K;
    bool any = false;
    for (int row = 0; row < K; ++row) {
        if (!std::getline(in, line)) raise(ErrorCode::BadHeader, "truncated WEIGHTS section");
        std::istringstream ls(line);
        for (int col = 0; col < K; ++col) {
            double w;
            if (!(ls >> w) || !std::isfinite(w) || w < 0.0)
                raise(ErrorCode::BadHeader, "bad weight in row " + std::to_string(row));
            p.mask.weights.push_back(w);
            any = any || w > 0.0;
        }
    }
    if (!any) raise(ErrorCode::BadHeader, "weight mask is all zeros");
    return p;
}

inline TripletPattern load_pattern_file(const std::string& path) {
    std::ifstream f(path, std::ios::binary);
    if (!f) raise(ErrorCode::BadHeader, "cannot open pattern file '" + path + "'");
    std::ostringstream buf;
    buf << f.rdbuf();
    return parse_pattern(buf.str());
}

/// The shipped 512-triplet table (pattern_default.cpp:527-539), read once from the LATCHPAT
/// file named by CLATCH_DEFAULT_PATTERN (default: paper_1609_03986_b200/data/default_pattern.latchpat
/// relative to the working directory). A reference build keeps its compiled-in table instead.
inline const TripletPattern& default_pattern() {
    static const TripletPattern p = [] {
        const char* env = std::getenv("CLATCH_DEFAULT_PATTERN");
        return load_pattern_file(env ? env : "paper_1609_03986_b200/data/default_pattern.latchpat");
    }();
    return p;
}

// ---- detection (detect.hpp:18-40; the step before the path) ----------------------------------
inline constexpr int kFastBorder = 3;
inline constexpr int kDefaultFastThreshold = 20;
inline constexpr int kOrientationRadius = 15;

namespace b200 {
inline std::vector<Keypoint> run_detect(const Image& image, double threshold, bool do_nms, bool orient, int radius) {
    Context& c = context();
    std::lock_guard<std::mutex> lock(c.mutex);
    std::size_t cap = std::max<std::size_t>(1024, static_cast<std::size_t>(image.width) * image.height / 64), count = 0;
    std::vector<double> rows;
    for (;;) {
        rows.resize(cap * 4);
        const int rc = clatch_detect_f64(c.ctx, image.data.data(), image.width, image.height,
                                         static_cast<std::size_t>(image.width), threshold, do_nms, orient, radius,
                                         rows.data(), cap, &count);
        if (rc == CLATCH_ERR_INVALID && count > cap) {   // buffer too small: *count holds the need
            cap = count;
            continue;
        }
        check(rc);
        break;
    }
    std::vector<Keypoint> out(count);
    for (std::size_t i = 0; i < count; ++i) out[i] = {rows[4 * i], rows[4 * i + 1], rows[4 * i + 2], rows[4 * i + 3]};
    return out;
}
} // namespace b200

/// FAST-9 segment test (+ 3x3 NMS, ties keep the smallest (y, x)); output sorted by (y, x), theta 0.
inline std::vector<Keypoint> fast_detect(const Image& image, double threshold, bool do_nms) {
    return b200::run_detect(image, threshold, do_nms, false, kOrientationRadius);
}

/// fast_detect followed by the intensity-centroid orientation; detections whose disc does not
/// fit in the image are dropped.
inline std::vector<Keypoint> detect_and_orient(const Image& image, double threshold, bool do_nms,
                                               int radius = kOrientationRadius) {
    return b200::run_detect(image, threshold, do_nms, true, radius);
}

// ---- extraction (descriptor.hpp:48-67) ------------------------------------------------------
inline bool keypoint_in_margin(const Image& image, const Keypoint& k) {   // src/descriptor.cpp:23-27
    return k.x - kWindowMargin >= 0.0 && k.y - kWindowMargin >= 0.0 && k.x + kWindowMargin <= image.width - 1 &&
           k.y + kWindowMargin <= image.height - 1;
}

/// Batch extraction: margin violators are silently dropped, the rest keep their input
/// order; output is identical for any `workers` (it only sizes the host-side trig pass).
inline std::vector<std::pair<Keypoint, Descriptor>> describe_all(const Image& image,
                                                                 const std::vector<Keypoint>& keypoints,
                                                                 const TripletPattern& pattern, int workers = 0) {
    static_assert(sizeof(Keypoint) == 4 * sizeof(double), "Keypoint must be 4 packed doubles");
    b200::Context& c = b200::context();
    std::lock_guard<std::mutex> lock(c.mutex);
    b200::use_pattern(c, pattern);
    const std::size_t n = keypoints.size(), bytes = static_cast<std::size_t>(pattern.bit_count) / 8;
    std::vector<std::int64_t> kept(n);
    std::vector<std::uint8_t> flat(n * bytes);
    std::size_t m = 0;
    b200::check(clatch_describe_all_f64(c.ctx, image.data.data(), image.width, image.height,
                                        static_cast<std::size_t>(image.width),
                                        reinterpret_cast<const double*>(keypoints.data()), n, 4, workers,
                                        kept.data(), flat.data(), &m));
    std::vector<std::pair<Keypoint, Descriptor>> out(m);
    for (std::size_t j = 0; j < m; ++j) {
        out[j].first = keypoints[static_cast<std::size_t>(kept[j])];
        out[j].second.bytes.assign(flat.begin() + static_cast<std::ptrdiff_t>(j * bytes),
                                   flat.begin() + static_cast<std::ptrdiff_t>((j + 1) * bytes));
    }
    return out;
}

/// Full descriptor for one keypoint. Throws TooCloseToBorder outside the margin.
inline Descriptor describe(const Image& image, const Keypoint& keypoint, const TripletPattern& pattern) {
    if (!keypoint_in_margin(image, keypoint))   // src/descriptor.cpp:30-33
        raise(ErrorCode::TooCloseToBorder, "keypoint (" + std::to_string(keypoint.x) + ", " +
                                               std::to_string(keypoint.y) + ") violates the " +
                                               std::to_string(kWindowMargin) + "-pixel margin");
    return describe_all(image, {keypoint}, pattern, 1).at(0).second;
}

// ---- LTCH descriptor container (descriptor.hpp:69-79, src/descriptor.cpp:110-211) --------------
// Host-side, byte for byte the reference's format: "LTCH", u32 version 1, u32 count, u32 descriptor
// bytes, u32 0, then per record four little-endian float32 (x, y, theta, score) + the descriptor.
namespace b200 {
inline void append_u32(std::string& out, std::uint32_t v) {
    for (int shift = 0; shift < 32; shift += 8) out.push_back(static_cast<char>((v >> shift) & 0xffu));
}
inline std::uint32_t read_u32(const std::string& in, std::size_t& pos) {
    if (in.size() < pos + 4) raise(ErrorCode::Truncated, "descriptor file ends mid-field");
    std::uint32_t v = 0;
    for (int i = 0; i < 4; ++i) v |= static_cast<std::uint32_t>(static_cast<unsigned char>(in[pos + i])) << (8 * i);
    pos += 4;
    return v;
}
} // namespace b200

inline std::string format_descriptor_file(const std::vector<std::pair<Keypoint, Descriptor>>& records) {
    const std::size_t bytes = records.empty() ? 0 : records.front().second.bytes.size();
    std::string out = "LTCH";
    b200::append_u32(out, 1u);
    b200::append_u32(out, static_cast<std::uint32_t>(records.size()));
    b200::append_u32(out, static_cast<std::uint32_t>(bytes));
    b200::append_u32(out, 0u);
    for (const auto& record : records) {
        const double fields[4] = {record.first.x, record.first.y, record.first.theta, record.first.score};
        for (double field : fields) {
            const float narrow = static_cast<float>(field);
            std::uint32_t bits;
            std::memcpy(&bits, &narrow, sizeof bits);
            b200::append_u32(out, bits);
        }
        out.append(reinterpret_cast<const char*>(record.second.bytes.data()), record.second.bytes.size());
    }
    return out;
}

inline std::vector<std::pair<Keypoint, Descriptor>> parse_descriptor_file(const std::string& data) {
    if (data.size() < 4 || data.compare(0, 4, "LTCH") != 0) raise(ErrorCode::BadHeader, "not a descriptor file (bad magic)");
    std::size_t pos = 4;
    const std::uint32_t version = b200::read_u32(data, pos);
    if (version != 1u) raise(ErrorCode::BadHeader, "unsupported descriptor file version " + std::to_string(version));
    const std::uint32_t count = b200::read_u32(data, pos), bytes = b200::read_u32(data, pos);
    b200::read_u32(data, pos);   // reserved
    std::vector<std::pair<Keypoint, Descriptor>> records;
    records.reserve(count);
    for (std::uint32_t i = 0; i < count; ++i) {
        double fields[4];
        for (double& field : fields) {
            const std::uint32_t bits = b200::read_u32(data, pos);
            float narrow;
            std::memcpy(&narrow, &bits, sizeof narrow);
            field = narrow;
        }
        if (data.size() < pos + bytes) raise(ErrorCode::Truncated, "descriptor file ends mid-record");
        Descriptor d;
        d.bytes.assign(data.begin() + static_cast<std::ptrdiff_t>(pos), data.begin() + static_cast<std::ptrdiff_t>(pos + bytes));
        pos += bytes;
        records.emplace_back(Keypoint{fields[0], fields[1], fields[2], fields[3]}, std::move(d));
    }
    return records;
}

inline void save_descriptor_file(const std::vector<std::pair<Keypoint, Descriptor>>& records, const std::string& path) {
    std::ofstream f(path, std::ios::binary);
    if (!f) raise(ErrorCode::Malformed, "cannot open '" + path + "' for writing");
    const std::string data = format_descriptor_file(records);
    f.write(data.data(), static_cast<std::streamsize>(data.size()));
}

inline std::vector<std::pair<Keypoint, Descriptor>> load_descriptor_file(const std::string& path) {
    std::ifstream f(path, std::ios::binary);
    if (!f) raise(ErrorCode::Malformed, "cannot open '" + path + "'");
    std::ostringstream buffer;
    buffer << f.rdbuf();
    return parse_descriptor_file(buffer.str());
}

// ---- matching (match.hpp:27-45) ---------------------------------------------------------------
/// Best and second-best gallery distances for one probe; ties go to the smallest index.
inline Knn2Result knn2(const Descriptor& probe, const std::vector<Descriptor>& gallery) {
    if (gallery.empty()) raise(ErrorCode::EmptyGallery, "knn2 needs a nonempty gallery");
    const std::size_t bytes = probe.bytes.size();
    const std::vector<std::uint8_t> g = b200::flatten(gallery, bytes);
    b200::Context& c = b200::context();
    std::lock_guard<std::mutex> lock(c.mutex);
    std::int32_t r[3];
    b200::check(clatch_match_top2(c.ctx, probe.bytes.data(), 1, g.data(), gallery.size(), static_cast<int>(bytes),
                                  &r[0], &r[1], &r[2]));
    return {r[0], r[1], r[2]};
}

/// Number of differing bits. Lengths must match (LengthMismatch otherwise).
inline int hamming(const Descriptor& a, const Descriptor& b) {
    if (a.bytes.size() != b.bytes.size())
        raise(ErrorCode::LengthMismatch, "descriptor lengths differ: " + std::to_string(a.bytes.size()) + " vs " +
                                             std::to_string(b.bytes.size()));
    if (a.bytes.empty()) return 0;
    return knn2(a, {b}).best_distance;
}

/// Brute-force matcher with optional ratio, cross-check and distance-cutoff filters.
/// Output sorted by probe index.
inline std::vector<MatchPair> match_brute_force(const std::vector<Descriptor>& probes,
                                                const std::vector<Descriptor>& gallery,
                                                const MatchOptions& options = {}) {
    if (gallery.empty()) raise(ErrorCode::EmptyGallery, "matching needs a nonempty gallery");   // src/match.cpp:55
    if (probes.empty()) return {};                                                              // :56
    const std::size_t bytes = probes[0].bytes.size();
    const std::vector<std::uint8_t> p = b200::flatten(probes, bytes), g = b200::flatten(gallery, bytes);
    std::vector<std::int32_t> rows(probes.size() * 4);
    std::size_t count = 0;
    b200::Context& c = b200::context();
    std::lock_guard<std::mutex> lock(c.mutex);
    b200::check(clatch_match_brute_force(c.ctx, p.data(), probes.size(), g.data(), gallery.size(),
                                         static_cast<int>(bytes), options.ratio.has_value(),
                                         options.ratio.value_or(0.0), options.cross_check,
                                         options.max_distance.has_value(), options.max_distance.value_or(0),
                                         rows.data(), &count));
    std::vector<MatchPair> out(count);
    for (std::size_t i = 0; i < count; ++i)
        out[i] = {rows[4 * i], rows[4 * i + 1], rows[4 * i + 2], rows[4 * i + 3]};
    return out;
}

// ---- text / image files around the path (src/image.cpp:52-78, src/detect.cpp:158-185, src/match.cpp:83-92) ----
// Host-side restatements of the reference's file formats so that a `latch detect | describe | match` pipeline can
// run on this library with the same files (tools: paper_1609_03986_b200/csrc/latch_cli.cpp).
namespace b200 {
inline std::string read_file(const std::string& path) {
    std::ifstream f(path, std::ios::binary);
    if (!f) raise(ErrorCode::Malformed, "cannot open '" + path + "'");
    std::ostringstream buf;
    buf << f.rdbuf();
    return buf.str();
}
inline void write_file(const std::string& path, const std::string& bytes) {
    std::ofstream f(path, std::ios::binary);
    if (!f) raise(ErrorCode::Malformed, "cannot open '" + path + "' for writing");
    f.write(bytes.data(), static_cast<std::streamsize>(bytes.size()));
    if (!f) raise(ErrorCode::Malformed, "write failed for '" + path + "'");
}
// One header token of a binary PGM: whitespace and '#' comments (to end of line) are skipped first.
inline std::string pgm_token(const std::string& b, std::size_t& pos) {
    for (;;) {
        while (pos < b.size() && std::isspace(static_cast<unsigned char>(b[pos]))) ++pos;
        if (pos < b.size() && b[pos] == '#') {
            while (pos < b.size() && b[pos] != '\n') ++pos;
            continue;
        }
        break;
    }
    const std::size_t start = pos;
    while (pos < b.size() && !std::isspace(static_cast<unsigned char>(b[pos])) && b[pos] != '#') ++pos;
    return b.substr(start, pos - start);
}
inline int pgm_number(const std::string& tok, const char* what) {
    if (tok.empty()) raise(ErrorCode::Malformed, std::string("missing ") + what);
    for (char ch : tok)
        if (!std::isdigit(static_cast<unsigned char>(ch)))
            raise(ErrorCode::Malformed, std::string("non-numeric ") + what + " '" + tok + "'");
    if (tok.size() > 9) raise(ErrorCode::Malformed, std::string("unparsable ") + what + " '" + tok + "'");
    return std::atoi(tok.c_str());
}
} // namespace b200

/// Binary PGM (P5, maxval <= 255) -> Image with integer-valued pixels (src/image.cpp:52-78).
inline Image load_pgm(const std::string& bytes) {
    std::size_t pos = 0;
    const std::string magic = b200::pgm_token(bytes, pos);
    if (magic != "P5") raise(ErrorCode::NotPGM, "expected magic 'P5', got '" + magic + "'");
    const int w = b200::pgm_number(b200::pgm_token(bytes, pos), "width");
    const int h = b200::pgm_number(b200::pgm_token(bytes, pos), "height");
    const int maxval = b200::pgm_number(b200::pgm_token(bytes, pos), "maxval");
    if (w < 1 || h < 1) raise(ErrorCode::Malformed, "non-positive dimensions");
    if (maxval < 1) raise(ErrorCode::Malformed, "maxval must be >= 1");
    if (maxval > 255) raise(ErrorCode::UnsupportedDepth, "maxval > 255 not supported");
    if (pos >= bytes.size() || !std::isspace(static_cast<unsigned char>(bytes[pos])))
        raise(ErrorCode::Malformed, "missing separator before payload");
    ++pos;   // exactly one whitespace byte before the pixels
    const std::size_t count = static_cast<std::size_t>(w) * h;
    if (bytes.size() - pos < count)
        raise(ErrorCode::Truncated, "payload has " + std::to_string(bytes.size() - pos) + " bytes, need " +
                                        std::to_string(count));
    Image image(w, h);
    for (std::size_t i = 0; i < count; ++i) image.data[i] = static_cast<unsigned char>(bytes[pos + i]);
    return image;
}
inline Image load_pgm_file(const std::string& path) { return load_pgm(b200::read_file(path)); }

/// Keypoint TSV: header line "x\ty\ttheta\tscore", then one "%.9g" row per keypoint (src/detect.cpp:158-185).
inline std::string format_keypoints(const std::vector<Keypoint>& keypoints) {
    std::string out = "x\ty\ttheta\tscore\n";
    char line[128];
    for (const Keypoint& k : keypoints) {
        std::snprintf(line, sizeof(line), "%.9g\t%.9g\t%.9g\t%.9g\n", k.x, k.y, k.theta, k.score);
        out += line;
    }
    return out;
}
inline std::vector<Keypoint> parse_keypoints(const std::string& text) {
    std::vector<Keypoint> out;
    std::istringstream in(text);
    std::string line;
    for (bool header = true; std::getline(in, line); header = false) {
        if (header || line.empty()) continue;
        Keypoint k;
        if (std::sscanf(line.c_str(), "%lf\t%lf\t%lf\t%lf", &k.x, &k.y, &k.theta, &k.score) != 4)
            raise(ErrorCode::Malformed, "bad keypoint line '" + line + "'");
        out.push_back(k);
    }
    return out;
}
inline void save_keypoints_file(const std::vector<Keypoint>& k, const std::string& path) { b200::write_file(path, format_keypoints(k)); }
inline std::vector<Keypoint> load_keypoints_file(const std::string& path) { return parse_keypoints(b200::read_file(path)); }

/// Match TSV: "probe\tgallery\tdistance\tsecond_distance" rows, no header (src/match.cpp:83-92).
inline std::string format_matches(const std::vector<MatchPair>& matches) {
    std::string out;
    char line[96];
    for (const MatchPair& m : matches) {
        std::snprintf(line, sizeof(line), "%d\t%d\t%d\t%d\n", m.probe_index, m.gallery_index, m.distance, m.second_distance);
        out += line;
    }
    return out;
}
inline void save_matches_file(const std::vector<MatchPair>& m, const std::string& path) { b200::write_file(path, format_matches(m)); }

// ---- sharding over several GPUs from C++ (the reference fans out over std::thread, src/parallel.hpp:17-38) ----
// One host thread and one context per entry of `devices`; units are dealt round-robin exactly as
// paper_1609_03986_b200/sharded.py deals them across processes (image i -> entry i mod D; pair k of the row-major
// (i < j) list -> entry k mod D), no data-path collective. Results do not depend on the device list.
namespace b200 {
template <class Fn>
inline void run_sharded(const std::vector<int>& devices, Fn&& per_slot) {
    if (devices.empty()) throw std::invalid_argument("device list is empty");
    ContextPool pool(devices);
    std::vector<std::thread> threads;
    std::vector<std::exception_ptr> errors(devices.size());
    for (std::size_t d = 0; d < devices.size(); ++d)
        threads.emplace_back([&, d] {
            try {
                per_slot(*pool.slots[d], d, devices.size());
            } catch (...) {
                errors[d] = std::current_exception();
            }
        });
    for (std::thread& t : threads) t.join();
    for (const std::exception_ptr& e : errors)
        if (e) std::rethrow_exception(e);
}
} // namespace b200

/// describe_all over many images, images dealt across `devices` (cfg3's partition). out[i] == describe_all(images[i], ...).
inline std::vector<std::vector<std::pair<Keypoint, Descriptor>>> describe_all_images(
    const std::vector<Image>& images, const std::vector<std::vector<Keypoint>>& keypoints, const TripletPattern& pattern,
    const std::vector<int>& devices = {0}, int workers = 0) {
    if (images.size() != keypoints.size()) throw std::invalid_argument("one keypoint list per image");
    std::vector<std::vector<std::pair<Keypoint, Descriptor>>> out(images.size());
    const std::size_t bytes = static_cast<std::size_t>(pattern.bit_count) / 8;
    b200::run_sharded(devices, [&](b200::Context& c, std::size_t slot, std::size_t slots) {
        b200::use_pattern(c, pattern);
        std::vector<const double*> img, kps;
        std::vector<int> w, h;
        std::vector<std::size_t> pitch, count, m;
        std::vector<std::vector<std::int64_t>> kept;
        std::vector<std::vector<std::uint8_t>> flat;
        std::vector<std::int64_t*> kept_p;
        std::vector<std::uint8_t*> flat_p;
        std::vector<std::size_t> mine;
        for (std::size_t i = slot; i < images.size(); i += slots) mine.push_back(i);
        if (mine.empty()) return;
        for (std::size_t i : mine) {
            img.push_back(images[i].data.data());
            w.push_back(images[i].width);
            h.push_back(images[i].height);
            pitch.push_back(static_cast<std::size_t>(images[i].width));
            kps.push_back(reinterpret_cast<const double*>(keypoints[i].data()));
            count.push_back(keypoints[i].size());
            kept.emplace_back(keypoints[i].size());
            flat.emplace_back(keypoints[i].size() * bytes);
        }
        for (std::size_t k = 0; k < mine.size(); ++k) {
            kept_p.push_back(kept[k].data());
            flat_p.push_back(flat[k].data());
        }
        m.assign(mine.size(), 0);
        b200::check(clatch_describe_batch_f64(c.ctx, img.data(), w.data(), h.data(), pitch.data(), kps.data(), count.data(), 4,
                                              mine.size(), workers, kept_p.data(), flat_p.data(), m.data()));
        for (std::size_t k = 0; k < mine.size(); ++k) {
            auto& rec = out[mine[k]];
            rec.resize(m[k]);
            for (std::size_t j = 0; j < m[k]; ++j) {
                rec[j].first = keypoints[mine[k]][static_cast<std::size_t>(kept[k][j])];
                rec[j].second.bytes.assign(flat[k].begin() + static_cast<std::ptrdiff_t>(j * bytes),
                                           flat[k].begin() + static_cast<std::ptrdiff_t>((j + 1) * bytes));
            }
        }
    });
    return out;
}

/// match_brute_force over every (i < j) pair of descriptor sets (cfg5's partition), pairs dealt across `devices`;
/// each entry uploads the sets its pairs touch once and runs them as resident sets. Returned in row-major pair order:
/// result[k] is the pair (i, j) at position k of {(0,1), (0,2), ..., (n-2,n-1)} and equals
/// match_brute_force(sets[i], sets[j], options). 64-byte descriptors.
inline std::vector<std::vector<MatchPair>> match_all_pairs(const std::vector<std::vector<Descriptor>>& sets,
                                                           const MatchOptions& options = {},
                                                           const std::vector<int>& devices = {0}) {
    std::vector<std::pair<int, int>> pairs;
    for (std::size_t i = 0; i < sets.size(); ++i)
        for (std::size_t j = i + 1; j < sets.size(); ++j) pairs.emplace_back(static_cast<int>(i), static_cast<int>(j));
    for (const auto& set : sets)
        if (set.empty()) raise(ErrorCode::EmptyGallery, "matching needs nonempty descriptor sets");
    std::vector<std::vector<MatchPair>> out(pairs.size());
    b200::run_sharded(devices, [&](b200::Context& c, std::size_t slot, std::size_t slots) {
        std::vector<std::size_t> mine;
        for (std::size_t k = slot; k < pairs.size(); k += slots) mine.push_back(k);
        if (mine.empty()) return;
        std::vector<int> local(sets.size(), -1);
        std::vector<clatch_set*> handles;
        struct Guard {
            std::vector<clatch_set*>& h;
            ~Guard() { for (clatch_set* s : h) clatch_set_destroy(s); }
        } guard{handles};
        std::vector<std::int32_t> idx;
        std::size_t cap = 0;
        for (std::size_t k : mine) {
            for (int side : {pairs[k].first, pairs[k].second})
                if (local[static_cast<std::size_t>(side)] < 0) {
                    const std::vector<std::uint8_t> flat = b200::flatten(sets[static_cast<std::size_t>(side)], 64);
                    clatch_set* s = nullptr;
                    b200::check(clatch_set_create(c.ctx, flat.data(), sets[static_cast<std::size_t>(side)].size(), 0, &s));
                    local[static_cast<std::size_t>(side)] = static_cast<int>(handles.size());
                    handles.push_back(s);
                }
            idx.push_back(local[static_cast<std::size_t>(pairs[k].first)]);
            idx.push_back(local[static_cast<std::size_t>(pairs[k].second)]);
            cap += sets[static_cast<std::size_t>(pairs[k].first)].size();
        }
        std::vector<std::int32_t> rows(std::max<std::size_t>(cap, 1) * 4);
        std::vector<std::size_t> offsets(mine.size() + 1, 0);
        b200::check(clatch_match_set_pairs(c.ctx, handles.data(), handles.size(), idx.data(), mine.size(),
                                           options.ratio.has_value(), options.ratio.value_or(0.0), options.cross_check,
                                           options.max_distance.has_value(), options.max_distance.value_or(0), rows.data(),
                                           cap, offsets.data()));
        for (std::size_t q = 0; q < mine.size(); ++q) {
            auto& dst = out[mine[q]];
            dst.resize(offsets[q + 1] - offsets[q]);
            for (std::size_t r = 0; r < dst.size(); ++r) {
                const std::int32_t* row = rows.data() + 4 * (offsets[q] + r);
                dst[r] = {row[0], row[1], row[2], row[3]};
            }
        }
    });
    return out;
}

} // namespace latch
