// C++ parity tests of the latch:: host API in include/latch_b200.hpp (GPU path through the
// C ABI) — written the way the reference's own doctest suites read
// (proj/tests/test_descriptor.cpp, test_match.cpp, acceptance.cpp), with the plain-C oracle
// (oracle/latch_oracle.c, linked directly) and the golden fixtures as the expected values.
// Run on a B200 box:  tests/cpp/test_latch_host <repo root>
#include <cstdio>
#include <cstdlib>
#include <fstream>
#include <iterator>
#include <string>
#include <vector>

#include "latch_b200.hpp"

extern "C" {   // oracle/latch_oracle.c — test infrastructure
size_t oracle_detect_and_orient(const double* img, int w, int h, double threshold, int do_nms, int radius,
                                double* out, size_t cap);
size_t oracle_fast_detect(const double* img, int w, int h, double threshold, int do_nms, double* out, size_t cap);
void oracle_structured_image(uint64_t seed, int w, int h, double* out);
void oracle_random_image(uint64_t seed, int w, int h, double* out);
void oracle_random_descriptors(uint64_t seed, size_t n, int bytes, uint8_t* out);
void oracle_random_keypoints(uint64_t seed, int w, int h, size_t n, double* out);
int oracle_describe(const double* img, int w, int h, const double* kp, const int* triplets, int T, int K,
                    const double* weights, uint8_t* out);
int oracle_hamming(const uint8_t* a, const uint8_t* b, size_t n);
void oracle_knn2(const uint8_t* probe, const uint8_t* gallery, size_t n, int bytes, int* out);
size_t oracle_match(const uint8_t* probes, size_t q, const uint8_t* gallery, size_t n, int bytes, int has_ratio,
                    double ratio, int cross_check, int has_max, int max_distance, int* out);
}

using latch::Descriptor;
using latch::Error;
using latch::ErrorCode;
using latch::Image;
using latch::Keypoint;
using latch::MatchOptions;
using latch::MatchPair;

static int g_checks = 0, g_failures = 0;
#define CHECK(cond)                                                              \
    do {                                                                         \
        ++g_checks;                                                              \
        if (!(cond)) { ++g_failures; std::printf("FAIL %s:%d  %s\n", __FILE__, __LINE__, #cond); } \
    } while (0)
#define CHECK_THROWS_CODE(expr, want)                                            \
    do {                                                                         \
        ++g_checks;                                                              \
        bool ok = false;                                                         \
        try { (void)(expr); } catch (const Error& e) { ok = e.code() == (want); } \
        if (!ok) { ++g_failures; std::printf("FAIL %s:%d  %s did not throw %s\n", __FILE__, __LINE__, #expr, #want); } \
    } while (0)

static Descriptor with_ones(int ones, int bytes = 64) {
    Descriptor d;
    d.bytes.assign(bytes, 0);
    for (int t = 0; t < ones; ++t) d.set_bit(static_cast<std::size_t>(t), true);
    return d;
}

static std::vector<Descriptor> random_descriptors(uint64_t seed, size_t n, int bytes = 64) {
    std::vector<uint8_t> flat(n * bytes);
    oracle_random_descriptors(seed, n, bytes, flat.data());
    std::vector<Descriptor> out(n);
    for (size_t i = 0; i < n; ++i) out[i].bytes.assign(flat.begin() + i * bytes, flat.begin() + (i + 1) * bytes);
    return out;
}

static std::vector<uint8_t> flat(const std::vector<Descriptor>& v) {
    std::vector<uint8_t> f;
    for (const Descriptor& d : v) f.insert(f.end(), d.bytes.begin(), d.bytes.end());
    return f;
}

static Image make_image(bool structured, uint64_t seed, int w, int h) {
    Image im(w, h);
    (structured ? oracle_structured_image : oracle_random_image)(seed, w, h, im.data.data());
    return im;
}

static std::vector<uint8_t> oracle_desc(const Image& im, const Keypoint& k, const latch::TripletPattern& p) {
    std::vector<int> trip;
    for (const latch::Triplet& t : p.triplets) trip.insert(trip.end(), {t.ax, t.ay, t.bx, t.by, t.cx, t.cy});
    std::vector<uint8_t> out(p.bit_count / 8);
    const double kp[3] = {k.x, k.y, k.theta};
    oracle_describe(im.data.data(), im.width, im.height, kp, trip.data(), p.bit_count, p.patch_size,
                    p.mask.weights.data(), out.data());
    return out;
}

static bool same(const std::vector<MatchPair>& got, const std::vector<int>& want, size_t count) {
    if (got.size() != count) return false;
    for (size_t i = 0; i < count; ++i)
        if (got[i].probe_index != want[4 * i] || got[i].gallery_index != want[4 * i + 1] ||
            got[i].distance != want[4 * i + 2] || got[i].second_distance != want[4 * i + 3])
            return false;
    return true;
}

static std::string read_file(const std::string& path) {
    std::ifstream f(path, std::ios::binary);
    return std::string(std::istreambuf_iterator<char>(f), std::istreambuf_iterator<char>());
}

int main(int argc, char** argv) {
    const std::string root = argc > 1 ? argv[1] : ".";
    setenv("CLATCH_DEFAULT_PATTERN", (root + "/paper_1609_03986_b200/data/default_pattern.latchpat").c_str(), 0);
    const latch::TripletPattern& pattern = latch::default_pattern();
    CHECK(pattern.bit_count == 512 && pattern.patch_size == 8 && pattern.triplets.size() == 512);

    // ---- hamming counts differing bits (test_match.cpp:41-66) ----
    {
        Descriptor a, b;
        a.bytes = {0x0f, 0xf0}; b.bytes = {0x00, 0xf0};
        CHECK(latch::hamming(a, b) == 4);
        CHECK(latch::hamming(with_ones(512), with_ones(0)) == 512);
        CHECK(latch::hamming(with_ones(200), with_ones(137)) == 63);
        Descriptor one, two;
        one.bytes = {0}; two.bytes = {0, 0};
        CHECK_THROWS_CODE(latch::hamming(one, two), ErrorCode::LengthMismatch);
        const auto d = random_descriptors(109, 40);
        for (size_t i = 0; i + 1 < d.size(); i += 2) {
            CHECK(latch::hamming(d[i], d[i + 1]) == oracle_hamming(d[i].bytes.data(), d[i + 1].bytes.data(), 64));
            CHECK(latch::hamming(d[i], d[i]) == 0);
        }
        const auto t = random_descriptors(113, 20, 13);   // byte tail
        for (size_t i = 0; i + 1 < t.size(); i += 2)
            CHECK(latch::hamming(t[i], t[i + 1]) == oracle_hamming(t[i].bytes.data(), t[i + 1].bytes.data(), 13));
    }

    // ---- knn2: ties go down, runner-up may tie, singleton sentinel (test_match.cpp:68-103) ----
    {
        const std::vector<Descriptor> gallery = {with_ones(10), with_ones(3), with_ones(7), with_ones(3)};
        const auto r = latch::knn2(with_ones(0), gallery);
        CHECK(r.best_index == 1 && r.best_distance == 3 && r.second_distance == 3);
        const auto single = latch::knn2(with_ones(0), {with_ones(9)});
        CHECK(single.best_index == 0 && single.best_distance == 9 && single.second_distance == 513);
        CHECK_THROWS_CODE(latch::knn2(with_ones(0), {}), ErrorCode::EmptyGallery);
        const auto g = random_descriptors(127, 40);
        const auto gf = flat(g);
        for (const Descriptor& p : random_descriptors(128, 50)) {
            int want[3];
            oracle_knn2(p.bytes.data(), gf.data(), g.size(), 64, want);
            const auto got = latch::knn2(p, g);
            CHECK(got.best_index == want[0] && got.best_distance == want[1] && got.second_distance == want[2]);
        }
    }

    // ---- filters (test_match.cpp:105-158) ----
    {
        MatchOptions opt;
        opt.ratio = 1.0;
        CHECK(latch::match_brute_force({with_ones(0)}, {with_ones(4), with_ones(4)}, opt).empty());   // strict <
        const std::vector<Descriptor> spread = {with_ones(4), with_ones(9)};
        opt.ratio = 0.5;
        const auto kept = latch::match_brute_force({with_ones(0)}, spread, opt);
        CHECK(kept.size() == 1 && kept[0].gallery_index == 0 && kept[0].distance == 4 && kept[0].second_distance == 9);
        opt.ratio = 0.4;
        CHECK(latch::match_brute_force({with_ones(0)}, spread, opt).empty());
        opt.ratio = 0.8;
        CHECK(latch::match_brute_force({with_ones(0)}, {with_ones(400)}, opt).size() == 1);           // sentinel 513
        MatchOptions cut;
        cut.max_distance = 7;
        CHECK(latch::match_brute_force({with_ones(0)}, {with_ones(7)}, cut).size() == 1);             // inclusive
        cut.max_distance = 6;
        CHECK(latch::match_brute_force({with_ones(0)}, {with_ones(7)}, cut).empty());
        MatchOptions cross;
        cross.cross_check = true;
        const auto got = latch::match_brute_force({with_ones(1), with_ones(2)}, {with_ones(0), with_ones(30)}, cross);
        CHECK(got.size() == 1 && got[0].probe_index == 0 && got[0].gallery_index == 0 && got[0].distance == 1);
        CHECK(latch::match_brute_force({with_ones(1), with_ones(2)}, {with_ones(0), with_ones(30)}).size() == 2);
    }

    // ---- every filter combination against the oracle (test_match.cpp:160-188) ----
    {
        auto all = random_descriptors(131, 105);
        std::vector<Descriptor> probes(all.begin(), all.begin() + 60), gallery(all.begin() + 60, all.end());
        gallery[10] = gallery[3];
        gallery[44] = gallery[7];
        probes[5] = gallery[3];
        const auto pf = flat(probes), gf = flat(gallery);
        for (int combo = 0; combo < 8; ++combo) {
            MatchOptions opt;
            if (combo & 1) opt.ratio = 0.9;
            if (combo & 2) opt.cross_check = true;
            if (combo & 4) opt.max_distance = 250;
            std::vector<int> want(4 * probes.size());
            const size_t count = oracle_match(pf.data(), probes.size(), gf.data(), gallery.size(), 64, combo & 1, 0.9,
                                              (combo & 2) != 0, (combo & 4) != 0, 250, want.data());
            for (int workers : {1, 2, 8}) {
                opt.workers = workers;
                CHECK(same(latch::match_brute_force(probes, gallery, opt), want, count));
            }
        }
        CHECK(latch::match_brute_force({}, {with_ones(1)}).empty());                       // test_match.cpp:190-192
        CHECK_THROWS_CODE(latch::match_brute_force({with_ones(1)}, {}), ErrorCode::EmptyGallery);
        CHECK_THROWS_CODE(latch::match_brute_force({}, {}), ErrorCode::EmptyGallery);
    }

    // ---- margin and describe (test_descriptor.cpp:76-87, 130-143) ----
    {
        const Image small(93, 93);
        CHECK(latch::keypoint_in_margin(small, {46.0, 46.0, 0, 0}));
        CHECK(!latch::keypoint_in_margin(small, {45.999, 46.0, 0, 0}));
        CHECK(!latch::keypoint_in_margin(small, {46.0, 46.001, 0, 0}));
        CHECK_THROWS_CODE(latch::describe(small, {36.0, 46.0, 0.0, 0.0}, pattern), ErrorCode::TooCloseToBorder);
        const Image big(200, 100);
        CHECK(latch::keypoint_in_margin(big, {153.0, 53.0, 0, 0}));
        CHECK(!latch::keypoint_in_margin(big, {154.0, 53.0, 0, 0}));

        const Image img = make_image(true, 83, 160, 160);
        std::vector<double> k(4 * 10);
        oracle_random_keypoints(84, 160, 160, 10, k.data());
        for (int i = 0; i < 10; ++i) {
            const Keypoint kp{k[4 * i], k[4 * i + 1], k[4 * i + 2], 0.0};
            const Descriptor d = latch::describe(img, kp, pattern);
            CHECK(d.bytes.size() == 64);
            CHECK(d.bytes == oracle_desc(img, kp, pattern));
        }
    }

    // ---- describe_all drops margin violators, ignores workers (test_descriptor.cpp:178-201) ----
    {
        const Image img = make_image(true, 101, 140, 140);
        const std::vector<Keypoint> kps = {{50.0, 50.0, 0.5, 9.0}, {10.0, 70.0, 0.0, 8.0}, {70.0, 50.0, -0.5, 7.0},
                                           {70.0, 139.0, 0.0, 6.0}, {93.0, 93.0, 2.0, 5.0}};
        const auto batch = latch::describe_all(img, kps, pattern, 1);
        CHECK(batch.size() == 3);
        if (batch.size() == 3) {
            CHECK(batch[0].first.x == 50.0 && batch[1].first.x == 70.0 && batch[1].first.y == 50.0 &&
                  batch[2].first.x == 93.0 && batch[2].first.score == 5.0);
            for (const auto& [kp, d] : batch) CHECK(d.bytes == oracle_desc(img, kp, pattern));
            for (int workers : {2, 8}) {
                const auto again = latch::describe_all(img, kps, pattern, workers);
                CHECK(again.size() == 3);
                for (size_t i = 0; i < again.size() && i < 3; ++i) CHECK(again[i].second == batch[i].second);
            }
        }
        CHECK(latch::describe_all(img, {}, pattern).empty());
    }

    // ---- additive brightness invariance, exact (test_descriptor.cpp:145-161) ----
    {
        const Image img = make_image(true, 89, 128, 128);
        std::vector<double> k(4 * 6);
        oracle_random_keypoints(90, 128, 128, 6, k.data());
        for (double shift : {30.0, -50.0, 1.0}) {
            Image shifted = img;
            for (double& v : shifted.data) v += shift;
            for (int i = 0; i < 6; ++i) {
                const Keypoint kp{k[4 * i], k[4 * i + 1], k[4 * i + 2], 0.0};
                CHECK(latch::describe(img, kp, pattern).bytes == latch::describe(shifted, kp, pattern).bytes);
            }
        }
    }

    // ---- custom pattern through parse_pattern (python/test_smoke.py:105-123 shape: T=8) ----
    {
        const latch::TripletPattern small = latch::parse_pattern(read_file(root + "/tests/golden/pattern_t8k8.latchpat"));
        const latch::TripletPattern weighted = latch::parse_pattern(read_file(root + "/tests/golden/pattern_t64k5w.latchpat"));
        const Image img = make_image(true, 97, 140, 140);
        const Keypoint kp{60.25, 71.5, 0.7, 0.0};
        CHECK(latch::describe(img, kp, small).bytes == oracle_desc(img, kp, small));
        CHECK(latch::describe(img, kp, weighted).bytes == oracle_desc(img, kp, weighted));
        CHECK(latch::describe(img, kp, pattern).bytes == oracle_desc(img, kp, pattern));   // and back
        CHECK_THROWS_CODE(latch::parse_pattern("not a pattern"), ErrorCode::BadHeader);
    }

    // ---- golden vector (acceptance.cpp:96-118): kp (128,128,0.3) on the golden image ----
    {
        const std::string pgm = read_file(root + "/tests/golden/golden_image.pgm");
        const std::string bits = read_file(root + "/tests/golden/golden_bits.bin");
        CHECK(bits.size() == 64 && pgm.size() == 65551);
        Image golden(256, 256);
        const size_t header = pgm.size() - 65536;
        for (size_t i = 0; i < 65536; ++i) golden.data[i] = static_cast<unsigned char>(pgm[header + i]);
        const Descriptor d = latch::describe(golden, {128.0, 128.0, 0.3, 0.0}, pattern);
        CHECK(std::string(d.bytes.begin(), d.bytes.end()) == bits);
    }

    // ---- LTCH container: detect + describe the golden image, the file is the fixture byte for byte
    //      (acceptance.cpp:120-130); parse/format round trip; error categories ----
    {
        const std::string pgm = read_file(root + "/tests/golden/golden_image.pgm");
        const std::string fixture = read_file(root + "/tests/golden/golden_descriptors.bin");
        Image golden(256, 256);
        const size_t header = pgm.size() - 65536;
        for (size_t i = 0; i < 65536; ++i) golden.data[i] = static_cast<unsigned char>(pgm[header + i]);
        const auto records = latch::describe_all(golden, latch::detect_and_orient(golden, 20.0, true), pattern);
        CHECK(records.size() == 257);
        CHECK(latch::format_descriptor_file(records) == fixture);
        const auto parsed = latch::parse_descriptor_file(fixture);
        CHECK(parsed.size() == 257 && latch::format_descriptor_file(parsed) == fixture);
        CHECK(latch::format_descriptor_file({}).size() == 20);
        CHECK_THROWS_CODE(latch::parse_descriptor_file("LTCX" + fixture.substr(4)), ErrorCode::BadHeader);
        CHECK_THROWS_CODE(latch::parse_descriptor_file(fixture.substr(0, fixture.size() - 1)), ErrorCode::Truncated);
        CHECK_THROWS_CODE(latch::load_descriptor_file(root + "/tests/golden/no_such_file.ltch"), ErrorCode::Malformed);
    }

    // ---- detection (test_detect.cpp:34-41, 128-151; acceptance.cpp:120-123) ----
    {
        Image flat(32, 32);
        for (double& v : flat.data) v = 77.0;
        CHECK(latch::fast_detect(flat, 20.0, true).empty());
        CHECK_THROWS_CODE(latch::fast_detect(Image(6, 32), 20.0, true), ErrorCode::ImageTooSmall);
        for (int structured = 0; structured < 2; ++structured) {
            const Image img = make_image(structured != 0, 21 + structured, 320, 240);
            std::vector<double> want(4 * img.data.size());
            const size_t n = oracle_detect_and_orient(img.data.data(), img.width, img.height, 20.0, 1, 15, want.data(),
                                                      img.data.size());
            const auto got = latch::detect_and_orient(img, 20.0, true);
            CHECK(got.size() == n);
            bool same = got.size() == n;
            for (size_t i = 0; same && i < n; ++i)
                same = got[i].x == want[4 * i] && got[i].y == want[4 * i + 1] && got[i].theta == want[4 * i + 2] &&
                       got[i].score == want[4 * i + 3];
            CHECK(same);
            const size_t m = oracle_fast_detect(img.data.data(), img.width, img.height, 25.5, 0, want.data(),
                                                img.data.size());
            const auto raw = latch::fast_detect(img, 25.5, false);
            CHECK(raw.size() == m);
            for (size_t i = 1; i < raw.size(); ++i)   // sorted by (y, x)
                CHECK((raw[i - 1].y < raw[i].y || (raw[i - 1].y == raw[i].y && raw[i - 1].x < raw[i].x)));
        }
    }

    // ---- sharding from C++ (latch_b200.hpp: one host thread + context per device-list entry) ----
    //      describe_all_images / match_all_pairs must equal the per-call API whatever the device list;
    //      {0, 0} runs two contexts on this box's one GPU concurrently.
    {
        std::vector<Image> images;
        std::vector<std::vector<Keypoint>> kps;
        for (int i = 0; i < 5; ++i) {
            images.push_back(make_image(i % 2 == 0, 300 + i, 200 + 16 * i, 180));
            std::vector<double> k(4 * 120);
            oracle_random_keypoints(400 + i, images.back().width, 180, 120, k.data());
            std::vector<Keypoint> list;
            for (int j = 0; j < 120; ++j) list.push_back({k[4 * j], k[4 * j + 1], k[4 * j + 2], 0.0});
            list[7].x = 3.0;   // a margin violator
            kps.push_back(list);
        }
        std::vector<std::vector<std::pair<Keypoint, Descriptor>>> want;
        for (int i = 0; i < 5; ++i) want.push_back(latch::describe_all(images[i], kps[i], pattern));
        for (const std::vector<int>& devices : {std::vector<int>{0}, std::vector<int>{0, 0}, std::vector<int>{0, 0, 0}}) {
            const auto got = latch::describe_all_images(images, kps, pattern, devices);
            CHECK(got.size() == 5);
            for (int i = 0; i < 5 && got.size() == 5; ++i) {
                CHECK(got[i].size() == want[i].size() && got[i].size() == 119);
                bool same_desc = got[i].size() == want[i].size();
                for (size_t j = 0; same_desc && j < got[i].size(); ++j)
                    same_desc = got[i][j].second == want[i][j].second && got[i][j].first.x == want[i][j].first.x;
                CHECK(same_desc);
            }
            std::vector<std::vector<Descriptor>> sets;
            for (const auto& rec : got) {
                sets.emplace_back();
                for (const auto& r : rec) sets.back().push_back(r.second);
            }
            sets[3][5] = sets[0][9];        // cross-image duplicates -> real matches and ties
            sets[3][6] = sets[0][9];
            sets[1][2] = sets[0][9];
            latch::MatchOptions opt;
            opt.ratio = 0.95;
            opt.cross_check = true;
            const auto all = latch::match_all_pairs(sets, opt, devices);
            CHECK(all.size() == 10);
            size_t k = 0, rows = 0;
            for (size_t i = 0; i < sets.size(); ++i)
                for (size_t j = i + 1; j < sets.size(); ++j, ++k) {
                    const auto one = latch::match_brute_force(sets[i], sets[j], opt);
                    bool eq = k < all.size() && all[k].size() == one.size();
                    for (size_t r = 0; eq && r < one.size(); ++r)
                        eq = all[k][r].probe_index == one[r].probe_index && all[k][r].gallery_index == one[r].gallery_index &&
                             all[k][r].distance == one[r].distance && all[k][r].second_distance == one[r].second_distance;
                    CHECK(eq);
                    rows += one.size();
                }
            CHECK(rows > 0);
        }
        CHECK(latch::describe_all_images({}, {}, pattern).empty());
        CHECK(latch::match_all_pairs({}, {}).empty());
    }

    // ---- the file formats around the path: PGM in, keypoint TSV both ways, match TSV out ----
    {
        const latch::Image golden = latch::load_pgm_file(root + "/tests/golden/golden_image.pgm");
        CHECK(golden.width == 256 && golden.height == 256);
        CHECK(latch::load_pgm("P5\n# a comment\n2 1\n255\n\x07\xff").data == (std::vector<double>{7.0, 255.0}));
        CHECK_THROWS_CODE(latch::load_pgm("P2\n2 1\n255\n12"), ErrorCode::NotPGM);
        CHECK_THROWS_CODE(latch::load_pgm("P5\n2 2\n255\nabc"), ErrorCode::Truncated);
        CHECK_THROWS_CODE(latch::load_pgm("P5\n2 2\n65535\nabcdefgh"), ErrorCode::UnsupportedDepth);
        const std::vector<Keypoint> kp = {{10.5, 20.25, -0.5, 33.0}, {1e-3, 123456.789, 3.14159265358979, 0.0}};
        const std::string text = latch::format_keypoints(kp);
        CHECK(text.rfind("x\ty\ttheta\tscore\n", 0) == 0);
        const auto back = latch::parse_keypoints(text);
        CHECK(back.size() == 2 && back[0].x == 10.5 && back[0].theta == -0.5 && latch::format_keypoints(back) == text);
        CHECK_THROWS_CODE(latch::parse_keypoints("x\ty\ttheta\tscore\n1\t2\tthree\t4\n"), ErrorCode::Malformed);
        CHECK(latch::format_matches({{0, 5, 12, 40}, {3, 1, 0, 513}}) == "0\t5\t12\t40\n3\t1\t0\t513\n");
    }

    std::printf("%s: %d checks, %d failures\n", g_failures ? "FAILED" : "PASSED", g_checks, g_failures);
    return g_failures ? 1 : 0;
}
