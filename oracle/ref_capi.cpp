// TEST INFRASTRUCTURE — not part of the product.
//
// Thin extern "C" surface over the UNMODIFIED reference ("latchkit") so that
// Python tests and bench.py's cpu_baseline / --impl reference leg can call the
// reference's own describe_all / match_brute_force / knn2 / hamming and its
// test generators through ctypes. This file contains no algorithm of its own:
// every call forwards into headers/sources that stay under /root/reference and
// are compiled from there by oracle/build_ref.sh into oracle/_ref/ (git-ignored).
//
// Reference entry points wrapped (paths relative to /root/reference/proj):
//   describe_all            src/descriptor.cpp:90-105
//   describe                src/descriptor.cpp:79-88
//   extract_window          src/descriptor.cpp:29-49
//   match_brute_force       src/match.cpp:52-81
//   knn2                    src/match.cpp:33-50
//   hamming                 src/match.cpp:14-31
//   detect_and_orient       src/detect.cpp
//   default_pattern         src/pattern_default.cpp:527-539
//   parse/format_pattern    src/pattern.cpp:68-160
//   testutil::random_image / structured_image / random_descriptor   tests/test_util.hpp:38-83
//   oracle::describe / oracle::reference_match                      tests/oracles.hpp:153-209
//   latch::Rng              include/latch/rng.hpp:13-38

#include <algorithm>
#include <cstdint>
#include <cstring>
#include <optional>
#include <string>
#include <vector>

#include "latch/descriptor.hpp"
#include "latch/detect.hpp"
#include "latch/errors.hpp"
#include "latch/image.hpp"
#include "latch/match.hpp"
#include "latch/pattern.hpp"
#include "latch/rng.hpp"
#define LATCH_TEST_DATA_DIR "."
#include "oracles.hpp"
#include "test_util.hpp"

namespace {

thread_local std::string g_error;

latch::Image make_image(const double* data, int w, int h) {
    latch::Image im(w, h);
    std::memcpy(im.data.data(), data, sizeof(double) * im.data.size());
    return im;
}

std::vector<latch::Keypoint> make_keypoints(const double* kps, std::size_t n) {
    std::vector<latch::Keypoint> out(n);
    for (std::size_t i = 0; i < n; ++i)
        out[i] = {kps[4 * i + 0], kps[4 * i + 1], kps[4 * i + 2], kps[4 * i + 3]};
    return out;
}

std::vector<latch::Descriptor> make_descriptors(const std::uint8_t* d, std::size_t n, int bytes) {
    std::vector<latch::Descriptor> out(n);
    for (std::size_t i = 0; i < n; ++i)
        out[i].bytes.assign(d + i * bytes, d + (i + 1) * bytes);
    return out;
}

latch::TripletPattern pattern_of(const char* text) {
    return text ? latch::parse_pattern(text) : latch::default_pattern();
}

template <typename Fn>
int guarded(Fn&& fn) {
    try {
        fn();
        return 0;
    } catch (const latch::Error& e) {
        g_error = e.what();
        return 100 + static_cast<int>(e.code());
    } catch (const std::exception& e) {
        g_error = e.what();
        return 99;
    }
}

} // namespace

extern "C" {

const char* ref_last_error() { return g_error.c_str(); }

// ---- generators (latch::Rng streams shared with the C++ tests) -------------

void ref_rng_units(std::uint64_t seed, std::size_t n, double* out) {
    latch::Rng rng(seed);
    for (std::size_t i = 0; i < n; ++i) out[i] = rng.unit();
}

void ref_rng_next(std::uint64_t seed, std::size_t n, std::uint64_t* out) {
    latch::Rng rng(seed);
    for (std::size_t i = 0; i < n; ++i) out[i] = rng.next();
}

void ref_random_image(std::uint64_t seed, int w, int h, double* out) {
    latch::Rng rng(seed);
    const latch::Image im = testutil::random_image(rng, w, h);
    std::memcpy(out, im.data.data(), sizeof(double) * im.data.size());
}

void ref_structured_image(std::uint64_t seed, int w, int h, double* out) {
    latch::Rng rng(seed);
    const latch::Image im = testutil::structured_image(rng, w, h);
    std::memcpy(out, im.data.data(), sizeof(double) * im.data.size());
}

void ref_random_descriptors(std::uint64_t seed, std::size_t n, int bytes, std::uint8_t* out) {
    latch::Rng rng(seed);
    for (std::size_t i = 0; i < n; ++i) {
        const latch::Descriptor d = testutil::random_descriptor(rng, bytes);
        std::memcpy(out + i * bytes, d.bytes.data(), bytes);
    }
}

// ---- pattern ------------------------------------------------------------

// Writes format_pattern(default_pattern()) into buf (NUL-terminated); returns
// the length needed (excluding NUL).
std::size_t ref_default_pattern_text(char* buf, std::size_t cap) {
    const std::string text = latch::format_pattern(latch::default_pattern());
    if (buf && cap > text.size()) std::memcpy(buf, text.c_str(), text.size() + 1);
    return text.size();
}

// Parses pattern text; fills T, K, triplets (T*6 ints, cap_t entries) and
// weights (K*K doubles, cap_w entries).
int ref_parse_pattern(const char* text, int* T, int* K, int* triplets, std::size_t cap_t,
                      double* weights, std::size_t cap_w) {
    return guarded([&] {
        const latch::TripletPattern p = latch::parse_pattern(text);
        *T = p.bit_count;
        *K = p.patch_size;
        for (std::size_t i = 0; i < p.triplets.size() && 6 * i + 5 < cap_t; ++i) {
            const latch::Triplet& t = p.triplets[i];
            const int v[6] = {t.ax, t.ay, t.bx, t.by, t.cx, t.cy};
            std::memcpy(triplets + 6 * i, v, sizeof(v));
        }
        for (std::size_t i = 0; i < p.mask.weights.size() && i < cap_w; ++i)
            weights[i] = p.mask.weights[i];
    });
}

// ---- detection (only used to regenerate the golden keypoints) ---------------

int ref_detect_and_orient(const double* img, int w, int h, double threshold, int nms,
                          double* out_kps, std::size_t cap, std::size_t* count) {
    return guarded([&] {
        const auto kps = latch::detect_and_orient(make_image(img, w, h), threshold, nms != 0);
        *count = kps.size();
        for (std::size_t i = 0; i < kps.size() && i < cap; ++i) {
            out_kps[4 * i + 0] = kps[i].x;
            out_kps[4 * i + 1] = kps[i].y;
            out_kps[4 * i + 2] = kps[i].theta;
            out_kps[4 * i + 3] = kps[i].score;
        }
    });
}

// triplet_bits (src/pattern.cpp:352-360) for C candidates over n 64x64 patches -> C rows of
// row_bytes bytes, BitVector layout (bit i of row c, LSB first).
int ref_triplet_bits(const double* windows, std::size_t n, const int* candidates, std::size_t C, int K,
                     const double* weights, std::uint8_t* out, std::size_t row_bytes) {
    return guarded([&] {
        latch::PatchDataset dataset;
        for (std::size_t i = 0; i < n; ++i) {
            dataset.patches.push_back(make_image(windows + i * 4096, 64, 64));
            dataset.labels.push_back(static_cast<long>(i));
        }
        latch::WeightMask mask;
        mask.size = K;
        mask.weights.assign(weights, weights + static_cast<std::size_t>(K) * K);
        std::memset(out, 0, C * row_bytes);
        for (std::size_t c = 0; c < C; ++c) {
            const int* t = candidates + 6 * c;
            const latch::BitVector bits = latch::triplet_bits({t[0], t[1], t[2], t[3], t[4], t[5]}, mask, dataset);
            for (std::size_t i = 0; i < n; ++i)
                if (bits.get(i)) out[c * row_bytes + (i >> 3)] |= static_cast<std::uint8_t>(1u << (i & 7));
        }
    });
}

// sample_candidates (src/pattern.cpp) -> count x 6 ints.
int ref_sample_candidates(std::size_t count, int K, std::uint64_t seed, int* out) {
    return guarded([&] {
        const auto cand = latch::sample_candidates(count, K, seed);
        for (std::size_t i = 0; i < cand.size(); ++i) {
            const int v[6] = {cand[i].ax, cand[i].ay, cand[i].bx, cand[i].by, cand[i].cx, cand[i].cy};
            std::memcpy(out + 6 * i, v, sizeof(v));
        }
    });
}

int ref_fast_detect(const double* img, int w, int h, double threshold, int nms, double* out_kps,
                    std::size_t cap, std::size_t* count) {
    return guarded([&] {
        const auto kps = latch::fast_detect(make_image(img, w, h), threshold, nms != 0);
        *count = kps.size();
        for (std::size_t i = 0; i < kps.size() && i < cap; ++i) {
            out_kps[4 * i + 0] = kps[i].x;
            out_kps[4 * i + 1] = kps[i].y;
            out_kps[4 * i + 2] = kps[i].theta;
            out_kps[4 * i + 3] = kps[i].score;
        }
    });
}

int ref_load_pgm(const char* path, double* out, std::size_t cap, int* w, int* h) {
    return guarded([&] {
        const latch::Image im = latch::load_pgm_file(path);
        *w = im.width;
        *h = im.height;
        if (out && cap >= im.data.size())
            std::memcpy(out, im.data.data(), sizeof(double) * im.data.size());
    });
}

// ---- extraction ------------------------------------------------------------

int ref_keypoint_in_margin(int w, int h, double x, double y) {
    const latch::Image im(w, h);
    return latch::keypoint_in_margin(im, {x, y, 0.0, 0.0}) ? 1 : 0;
}

int ref_extract_window(const double* img, int w, int h, const double* kp4, double* out4096) {
    return guarded([&] {
        const latch::Window64 win =
            latch::extract_window(make_image(img, w, h), {kp4[0], kp4[1], kp4[2], kp4[3]});
        std::memcpy(out4096, win.data.data(), sizeof(double) * 4096);
    });
}

// The test-suite oracle window (tests/oracles.hpp:117-130).
void ref_oracle_window(const double* img, int w, int h, const double* kp4, double* out4096) {
    const auto win = oracle::window(make_image(img, w, h), {kp4[0], kp4[1], kp4[2], kp4[3]});
    std::memcpy(out4096, win.data(), sizeof(double) * 4096);
}

int ref_triplet_bit(const double* win4096, const int* trip6, int K, const double* weights) {
    latch::Window64 w;
    std::memcpy(w.data.data(), win4096, sizeof(double) * 4096);
    latch::WeightMask mask;
    mask.size = K;
    mask.weights.assign(weights, weights + static_cast<std::size_t>(K) * K);
    const latch::Triplet t{trip6[0], trip6[1], trip6[2], trip6[3], trip6[4], trip6[5]};
    return latch::triplet_bit(w, t, mask) ? 1 : 0;
}

int ref_describe(const double* img, int w, int h, const double* kp4, const char* pattern_text,
                 std::uint8_t* out) {
    return guarded([&] {
        const latch::TripletPattern pat = pattern_of(pattern_text);
        const latch::Descriptor d =
            latch::describe(make_image(img, w, h), {kp4[0], kp4[1], kp4[2], kp4[3]}, pat);
        std::memcpy(out, d.bytes.data(), d.bytes.size());
    });
}

// Scalar test-suite oracle (tests/oracles.hpp:153-163).
int ref_oracle_describe(const double* img, int w, int h, const double* kp4,
                        const char* pattern_text, std::uint8_t* out) {
    return guarded([&] {
        const latch::TripletPattern pat = pattern_of(pattern_text);
        const auto bytes =
            oracle::describe(make_image(img, w, h), {kp4[0], kp4[1], kp4[2], kp4[3]}, pat);
        std::memcpy(out, bytes.data(), bytes.size());
    });
}

// describe_all: out_kept receives the input indices of the kept keypoints,
// out_desc kept*T/8 bytes (both sized for n by the caller).
int ref_describe_all(const double* img, int w, int h, const double* kps, std::size_t n,
                     const char* pattern_text, int workers, std::int64_t* out_kept,
                     std::uint8_t* out_desc, std::size_t* out_count) {
    return guarded([&] {
        const latch::Image im = make_image(img, w, h);
        const latch::TripletPattern pat = pattern_of(pattern_text);
        const auto keypoints = make_keypoints(kps, n);
        const auto records = latch::describe_all(im, keypoints, pat, workers);
        const std::size_t bytes = static_cast<std::size_t>(pat.bit_count) / 8;
        std::size_t slot = 0;
        for (std::size_t i = 0; i < n && slot < records.size(); ++i) {
            if (!latch::keypoint_in_margin(im, keypoints[i])) continue;
            out_kept[slot] = static_cast<std::int64_t>(i);
            std::memcpy(out_desc + slot * bytes, records[slot].second.bytes.data(), bytes);
            ++slot;
        }
        *out_count = records.size();
    });
}

// Serialises describe_all(...) with the reference's LTCH container
// (src/descriptor.cpp:146-162) — used to regenerate golden_descriptors.bin.
int ref_describe_all_file(const double* img, int w, int h, const double* kps, std::size_t n,
                          char* out, std::size_t cap, std::size_t* out_len) {
    return guarded([&] {
        const latch::Image im = make_image(img, w, h);
        const std::string bytes = latch::format_descriptor_file(
            latch::describe_all(im, make_keypoints(kps, n), latch::default_pattern(), 1));
        *out_len = bytes.size();
        if (out && cap >= bytes.size()) std::memcpy(out, bytes.data(), bytes.size());
    });
}

// ---- matching --------------------------------------------------------------

int ref_hamming(const std::uint8_t* a, std::size_t na, const std::uint8_t* b, std::size_t nb,
                int* out) {
    return guarded([&] {
        latch::Descriptor da, db;
        da.bytes.assign(a, a + na);
        db.bytes.assign(b, b + nb);
        *out = latch::hamming(da, db);
    });
}

int ref_knn2(const std::uint8_t* probe, const std::uint8_t* gallery, std::size_t n, int bytes,
             int* out3) {
    return guarded([&] {
        latch::Descriptor p;
        p.bytes.assign(probe, probe + bytes);
        const latch::Knn2Result r = latch::knn2(p, make_descriptors(gallery, n, bytes));
        out3[0] = r.best_index;
        out3[1] = r.best_distance;
        out3[2] = r.second_distance;
    });
}

// Forward top-2 for every probe (knn2 loop under the reference's parallel_for
// semantics is what match_brute_force does; exposed raw for parity on the
// unfiltered triples). out is Q*3 ints.
int ref_knn2_all(const std::uint8_t* probes, std::size_t q, const std::uint8_t* gallery,
                 std::size_t n, int bytes, int* out) {
    return guarded([&] {
        const auto g = make_descriptors(gallery, n, bytes);
        for (std::size_t i = 0; i < q; ++i) {
            latch::Descriptor p;
            p.bytes.assign(probes + i * bytes, probes + (i + 1) * bytes);
            const latch::Knn2Result r = latch::knn2(p, g);
            out[3 * i + 0] = r.best_index;
            out[3 * i + 1] = r.best_distance;
            out[3 * i + 2] = r.second_distance;
        }
    });
}

// match_brute_force. has_ratio / has_max select the optionals. out is up to
// q rows of 4 ints.
int ref_match(const std::uint8_t* probes, std::size_t q, const std::uint8_t* gallery,
              std::size_t n, int bytes, int has_ratio, double ratio, int cross_check, int has_max,
              int max_distance, int workers, int* out, std::size_t* out_count) {
    return guarded([&] {
        latch::MatchOptions opt;
        if (has_ratio) opt.ratio = ratio;
        opt.cross_check = cross_check != 0;
        if (has_max) opt.max_distance = max_distance;
        opt.workers = workers;
        const auto m = latch::match_brute_force(make_descriptors(probes, q, bytes),
                                                make_descriptors(gallery, n, bytes), opt);
        *out_count = m.size();
        for (std::size_t i = 0; i < m.size(); ++i) {
            out[4 * i + 0] = m[i].probe_index;
            out[4 * i + 1] = m[i].gallery_index;
            out[4 * i + 2] = m[i].distance;
            out[4 * i + 3] = m[i].second_distance;
        }
    });
}

// The test-suite's scalar matcher (tests/oracles.hpp:175-209).
int ref_oracle_match(const std::uint8_t* probes, std::size_t q, const std::uint8_t* gallery,
                     std::size_t n, int bytes, int has_ratio, double ratio, int cross_check,
                     int has_max, int max_distance, int* out, std::size_t* out_count) {
    return guarded([&] {
        latch::MatchOptions opt;
        if (has_ratio) opt.ratio = ratio;
        opt.cross_check = cross_check != 0;
        if (has_max) opt.max_distance = max_distance;
        const auto m = oracle::reference_match(make_descriptors(probes, q, bytes),
                                               make_descriptors(gallery, n, bytes), opt);
        *out_count = m.size();
        for (std::size_t i = 0; i < m.size(); ++i) {
            out[4 * i + 0] = m[i].probe_index;
            out[4 * i + 1] = m[i].gallery_index;
            out[4 * i + 2] = m[i].distance;
            out[4 * i + 3] = m[i].second_distance;
        }
    });
}

// ---- timed legs for bench.py (--impl reference / cpu_baseline) ---------------
// Pre-built objects so the timed region holds only the reference's hot path.

struct RefBenchState {
    latch::Image image;
    std::vector<latch::Keypoint> keypoints;
    std::vector<latch::Descriptor> probes, gallery;
};

void* ref_bench_create(const double* img, int w, int h, const double* kps, std::size_t n) {
    auto* s = new RefBenchState;
    s->image = make_image(img, w, h);
    s->keypoints = make_keypoints(kps, n);
    return s;
}

void ref_bench_destroy(void* state) { delete static_cast<RefBenchState*>(state); }

// describe_all over the first `count` keypoints, result kept as the probe and
// gallery sets for the match leg. Returns the number of descriptors.
std::size_t ref_bench_describe(void* state, std::size_t count, int workers) {
    auto* s = static_cast<RefBenchState*>(state);
    std::vector<latch::Keypoint> sub(s->keypoints.begin(),
                                     s->keypoints.begin() + static_cast<std::ptrdiff_t>(count));
    const auto records = latch::describe_all(s->image, sub, latch::default_pattern(), workers);
    s->probes.clear();
    for (const auto& r : records) s->probes.push_back(r.second);
    return records.size();
}

void ref_bench_set_gallery(void* state, const std::uint8_t* gallery, std::size_t n, int bytes) {
    static_cast<RefBenchState*>(state)->gallery = make_descriptors(gallery, n, bytes);
}

void ref_bench_gallery_from_probes(void* state) {
    auto* s = static_cast<RefBenchState*>(state);
    s->gallery = s->probes;
}

void ref_bench_set_probes(void* state, const std::uint8_t* probes, std::size_t n, int bytes) {
    static_cast<RefBenchState*>(state)->probes = make_descriptors(probes, n, bytes);
}

// match_brute_force(first `count` probes, gallery), no filters. Returns the
// number of matches; checksum accumulates indices/distances so the work
// cannot be elided.
std::size_t ref_bench_match(void* state, std::size_t count, int workers, std::uint64_t* checksum) {
    auto* s = static_cast<RefBenchState*>(state);
    std::vector<latch::Descriptor> sub(s->probes.begin(),
                                       s->probes.begin() + static_cast<std::ptrdiff_t>(count));
    latch::MatchOptions opt;
    opt.workers = workers;
    const auto m = latch::match_brute_force(sub, s->gallery, opt);
    std::uint64_t c = 0;
    for (const auto& p : m)
        c = c * 1000003u + static_cast<std::uint64_t>(p.gallery_index) * 1024u +
            static_cast<std::uint64_t>(p.distance) + static_cast<std::uint64_t>(p.second_distance);
    if (checksum) *checksum = c;
    return m.size();
}

} // extern "C"
