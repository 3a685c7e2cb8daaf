/* TEST INFRASTRUCTURE — CPU restatement of the reference algorithm, NOT the product.
 *
 * Plain-C restatement of the two hot paths of the reference ("latchkit",
 * /root/reference/proj): LATCH descriptor extraction and brute-force Hamming
 * top-2 matching, plus the seeded generators the reference's tests draw their
 * inputs from. It exists so that tests/, __graft_entry__.smoke() and bench.py's
 * cpu_baseline leg have a checker that travels to the GPU box without the
 * reference tree. Nothing under paper_1609_03986_b200/ may call into this file.
 *
 * Parity is PINNED: tests/test_oracle.py checks every function below against
 *  (a) the golden fixtures regenerated from the reference's own tools
 *      (golden_bits.bin, golden_descriptors.bin; SHA-256s in SURVEY.md §4), and
 *  (b) the unmodified reference compiled into oracle/_ref/liblatch_ref.so
 *      whenever that library is present.
 *
 * Arithmetic contract (must match the reference build: x86-64 baseline, no
 * FMA contraction, glibc libm trig): compile with -O2 -ffp-contract=off and
 * no -ffast-math / -march flags (oracle/Makefile does).
 *
 * Every function cites the reference file:line it restates
 * (paths relative to /root/reference/proj).
 */
#include <math.h>
#include <stddef.h>
#include <stdint.h>
#include <stdlib.h>
#include <string.h>

#define ORACLE_WINDOW 64  /* include/latch/pattern.hpp:12 kWindowSize */
#define ORACLE_MARGIN 46  /* include/latch/descriptor.hpp:17 kWindowMargin */

/* ------------------------------------------------------------------------
 * RNG — include/latch/rng.hpp:13-38. std::mt19937_64 (Matsumoto/Nishimura
 * 2004 MT19937-64, the ISO C++ parameter set), seeded with a single value.
 * ---------------------------------------------------------------------- */
typedef struct {
    uint64_t mt[312];
    int idx;
} oracle_rng;

static void rng_seed(oracle_rng* r, uint64_t seed) {
    r->mt[0] = seed;
    for (int i = 1; i < 312; ++i)
        r->mt[i] = 6364136223846793005ULL * (r->mt[i - 1] ^ (r->mt[i - 1] >> 62)) + (uint64_t)i;
    r->idx = 312;
}

static uint64_t rng_next(oracle_rng* r) { /* rng.hpp:17 */
    if (r->idx >= 312) {
        for (int i = 0; i < 312; ++i) {
            const uint64_t x = (r->mt[i] & 0xFFFFFFFF80000000ULL) |
                               (r->mt[(i + 1) % 312] & 0x7FFFFFFFULL);
            uint64_t xa = x >> 1;
            if (x & 1ULL) xa ^= 0xB5026F5AA96619E9ULL;
            r->mt[i] = r->mt[(i + 156) % 312] ^ xa;
        }
        r->idx = 0;
    }
    uint64_t y = r->mt[r->idx++];
    y ^= (y >> 29) & 0x5555555555555555ULL;
    y ^= (y << 17) & 0x71D67FFFEDA60000ULL;
    y ^= (y << 37) & 0xFFF7EEE000000000ULL;
    y ^= (y >> 43);
    return y;
}

static uint32_t rng_bounded(oracle_rng* r, uint32_t n) { /* rng.hpp:21-23 */
    return (uint32_t)(rng_next(r) % n);
}

static double rng_unit(oracle_rng* r) { /* rng.hpp:26 */
    return (double)(rng_next(r) >> 11) * 0x1.0p-53;
}

void oracle_rng_next(uint64_t seed, size_t n, uint64_t* out) {
    oracle_rng r;
    rng_seed(&r, seed);
    for (size_t i = 0; i < n; ++i) out[i] = rng_next(&r);
}

void oracle_rng_units(uint64_t seed, size_t n, double* out) {
    oracle_rng r;
    rng_seed(&r, seed);
    for (size_t i = 0; i < n; ++i) out[i] = rng_unit(&r);
}

/* ------------------------------------------------------------------------
 * Generators — tests/test_util.hpp:38-83.
 * ---------------------------------------------------------------------- */

/* testutil::random_image (test_util.hpp:38-47), lo = 0, hi = 255. */
void oracle_random_image(uint64_t seed, int w, int h, double* out) {
    oracle_rng r;
    rng_seed(&r, seed);
    const size_t n = (size_t)w * (size_t)h;
    for (size_t i = 0; i < n; ++i) out[i] = 0 + (double)rng_bounded(&r, 256u);
}

/* Same stream, written straight to bytes (values are integers in [0,255]). */
void oracle_random_image_u8(uint64_t seed, int w, int h, uint8_t* out) {
    oracle_rng r;
    rng_seed(&r, seed);
    const size_t n = (size_t)w * (size_t)h;
    for (size_t i = 0; i < n; ++i) out[i] = (uint8_t)rng_bounded(&r, 256u);
}

static int imin(int a, int b) { return a < b ? a : b; }
static int imax(int a, int b) { return a > b ? a : b; }

/* testutil::structured_image (test_util.hpp:51-76). */
void oracle_structured_image(uint64_t seed, int w, int h, double* out) {
    oracle_rng r;
    rng_seed(&r, seed);
    for (int y = 0; y < h; ++y)
        for (int x = 0; x < w; ++x)
            out[(size_t)y * w + x] = 110.0 + 40.0 * sin(x * 0.05) * cos(y * 0.07);

    const int blobs = (w * h) / 800;
    for (int i = 0; i < blobs; ++i) {
        const double value = rng_bounded(&r, 2) == 0 ? 60.0 + 25.0 * rng_unit(&r)
                                                     : 190.0 + 30.0 * rng_unit(&r);
        const int cx = 8 + (int)rng_bounded(&r, (uint32_t)(w - 16));
        const int cy = 8 + (int)rng_bounded(&r, (uint32_t)(h - 16));
        const int rad = 2 + (int)rng_bounded(&r, 5);
        const int square = rng_bounded(&r, 2) == 0;
        for (int y = imax(0, cy - rad); y <= imin(h - 1, cy + rad); ++y)
            for (int x = imax(0, cx - rad); x <= imin(w - 1, cx + rad); ++x) {
                const int dx = x - cx, dy = y - cy;
                if (square || dx * dx + dy * dy <= rad * rad) out[(size_t)y * w + x] = value;
            }
    }
    const size_t n = (size_t)w * (size_t)h;
    for (size_t i = 0; i < n; ++i) {
        double p = round(out[i]);
        if (p < 55.0) p = 55.0;
        if (p > 225.0) p = 225.0;
        out[i] = p;
    }
}

/* testutil::random_descriptor (test_util.hpp:78-83), n descriptors back to
 * back from one stream. */
void oracle_random_descriptors(uint64_t seed, size_t n, int bytes, uint8_t* out) {
    oracle_rng r;
    rng_seed(&r, seed);
    const size_t total = n * (size_t)bytes;
    for (size_t i = 0; i < total; ++i) out[i] = (uint8_t)rng_bounded(&r, 256u);
}

/* Keypoint recipe of tests/acceptance.cpp:43-49 with the SURVEY §8(d) theta
 * range: x = 46 + unit*(W-93), y = 46 + unit*(H-93), theta = -pi + unit*2pi,
 * score 0. out is n x 4 doubles. */
void oracle_random_keypoints(uint64_t seed, int w, int h, size_t n, double* out) {
    oracle_rng r;
    rng_seed(&r, seed);
    for (size_t i = 0; i < n; ++i) {
        out[4 * i + 0] = 46.0 + rng_unit(&r) * (double)(w - 93);
        out[4 * i + 1] = 46.0 + rng_unit(&r) * (double)(h - 93);
        out[4 * i + 2] = -3.141592653589793 + rng_unit(&r) * 6.283185307179586;
        out[4 * i + 3] = 0.0;
    }
}

/* ------------------------------------------------------------------------
 * Extraction
 * ---------------------------------------------------------------------- */

/* keypoint_in_margin — src/descriptor.cpp:23-27. NaN coordinates fail every
 * comparison and are therefore outside. */
int oracle_in_margin(int w, int h, double x, double y) {
    return x - ORACLE_MARGIN >= 0.0 && y - ORACLE_MARGIN >= 0.0 &&
           x + ORACLE_MARGIN <= (double)(w - 1) && y + ORACLE_MARGIN <= (double)(h - 1);
}

/* sample_bilinear — src/image.cpp:109-126. Returns NaN for an out-of-bounds
 * sample (the reference raises OutOfBounds there). */
static double bilinear(const double* img, int w, int h, double x, double y) {
    if (!(x >= 0.0 && x <= w - 1 && y >= 0.0 && y <= h - 1)) return NAN;
    int x0 = (int)floor(x);
    int y0 = (int)floor(y);
    if (x0 > w - 2) x0 = w - 2;
    if (y0 > h - 2) y0 = h - 2;
    if (x0 < 0) x0 = 0;
    if (y0 < 0) y0 = 0;
    const int x1 = x0 + 1 < w ? x0 + 1 : x0;
    const int y1 = y0 + 1 < h ? y0 + 1 : y0;
    const double fx = x - x0;
    const double fy = y - y0;
    const double top = (1.0 - fx) * img[(size_t)y0 * w + x0] + fx * img[(size_t)y0 * w + x1];
    const double bottom = (1.0 - fx) * img[(size_t)y1 * w + x0] + fx * img[(size_t)y1 * w + x1];
    return (1.0 - fy) * top + fy * bottom;
}

double oracle_sample_bilinear(const double* img, int w, int h, double x, double y) {
    return bilinear(img, w, h, x, y);
}

/* extract_window — src/descriptor.cpp:29-49. kp = {x, y, theta}. Returns 0,
 * or 1 when the keypoint violates the margin (reference: TooCloseToBorder). */
int oracle_extract_window(const double* img, int w, int h, const double* kp, double* win) {
    if (!oracle_in_margin(w, h, kp[0], kp[1])) return 1;
    const double c = cos(kp[2]);
    const double s = sin(kp[2]);
    const double half = (ORACLE_WINDOW - 1) / 2.0;
    for (int v = 0; v < ORACLE_WINDOW; ++v) {
        const double dv = v - half;
        for (int u = 0; u < ORACLE_WINDOW; ++u) {
            const double du = u - half;
            win[(size_t)v * ORACLE_WINDOW + u] =
                bilinear(img, w, h, kp[0] + c * du - s * dv, kp[1] + s * du + c * dv);
        }
    }
    return 0;
}

/* triplet_bit — src/descriptor.cpp:51-77. trip = {ax, ay, bx, by, cx, cy},
 * weights K*K row-major. */
int oracle_triplet_bit(const double* win, const int* trip, int K, const double* weights) {
    const double* anchor = win + (size_t)trip[1] * ORACLE_WINDOW + trip[0];
    const double* comp1 = win + (size_t)trip[3] * ORACLE_WINDOW + trip[2];
    const double* comp2 = win + (size_t)trip[5] * ORACLE_WINDOW + trip[4];
    const double* weight = weights;
    double d1 = 0.0, d2 = 0.0;
    for (int row = 0; row < K; ++row) {
        for (int col = 0; col < K; ++col) {
            const double wgt = weight[col];
            const double a = anchor[col];
            const double e1 = a - comp1[col];
            const double e2 = a - comp2[col];
            d1 += wgt * e1 * e1;
            d2 += wgt * e2 * e2;
        }
        anchor += ORACLE_WINDOW;
        comp1 += ORACLE_WINDOW;
        comp2 += ORACLE_WINDOW;
        weight += K;
    }
    return d1 > d2;
}

/* describe — src/descriptor.cpp:79-88. triplets T*6 ints; out T/8 bytes,
 * bit t -> out[t>>3] |= 1 << (t&7). Returns 1 outside the margin. */
int oracle_describe(const double* img, int w, int h, const double* kp, const int* triplets,
                    int T, int K, const double* weights, uint8_t* out) {
    double* win = (double*)malloc(sizeof(double) * ORACLE_WINDOW * ORACLE_WINDOW);
    if (oracle_extract_window(img, w, h, kp, win)) {
        free(win);
        return 1;
    }
    memset(out, 0, (size_t)T / 8);
    for (int t = 0; t < T; ++t)
        if (oracle_triplet_bit(win, triplets + 6 * (size_t)t, K, weights))
            out[t >> 3] |= (uint8_t)(1u << (t & 7));
    free(win);
    return 0;
}

/* describe_all — src/descriptor.cpp:90-105. kps n x 4 doubles {x,y,theta,score};
 * kept receives the input indices that survive the margin filter (input
 * order), desc kept*T/8 bytes. Returns the kept count. Serial on purpose:
 * bench.py threads it from the outside when it wants all cores. */
size_t oracle_describe_all(const double* img, int w, int h, const double* kps, size_t n,
                           const int* triplets, int T, int K, const double* weights,
                           int64_t* kept, uint8_t* desc) {
    size_t m = 0;
    for (size_t i = 0; i < n; ++i)
        if (oracle_in_margin(w, h, kps[4 * i], kps[4 * i + 1])) kept[m++] = (int64_t)i;
    const size_t bytes = (size_t)T / 8;
    for (size_t slot = 0; slot < m; ++slot)
        oracle_describe(img, w, h, kps + 4 * (size_t)kept[slot], triplets, T, K, weights,
                        desc + slot * bytes);
    return m;
}

/* ------------------------------------------------------------------------
 * Matching
 * ---------------------------------------------------------------------- */

static int popcount64(uint64_t x) {
    x = x - ((x >> 1) & 0x5555555555555555ULL);
    x = (x & 0x3333333333333333ULL) + ((x >> 2) & 0x3333333333333333ULL);
    x = (x + (x >> 4)) & 0x0F0F0F0F0F0F0F0FULL;
    return (int)((x * 0x0101010101010101ULL) >> 56);
}

/* hamming — src/match.cpp:14-31: 64-bit words then a byte tail. Lengths are
 * equal by construction here (the LengthMismatch check lives in the host
 * layers). */
int oracle_hamming(const uint8_t* a, const uint8_t* b, size_t n) {
    const size_t words = n / 8;
    int total = 0;
    for (size_t w = 0; w < words; ++w) {
        uint64_t x, y;
        memcpy(&x, a + w * 8, 8);
        memcpy(&y, b + w * 8, 8);
        total += popcount64(x ^ y);
    }
    for (size_t i = words * 8; i < n; ++i) total += popcount64((uint64_t)(a[i] ^ b[i]));
    return total;
}

/* knn2 — src/match.cpp:33-50. out = {best_index, best_distance,
 * second_distance}; both distances start at the sentinel 8*bytes+1, strict
 * '<' keeps the lowest index on ties. n must be > 0. */
void oracle_knn2(const uint8_t* probe, const uint8_t* gallery, size_t n, int bytes, int* out) {
    const int sentinel = bytes * 8 + 1;
    int best_index = -1, best = sentinel, second = sentinel;
    for (size_t g = 0; g < n; ++g) {
        const int d = oracle_hamming(probe, gallery + g * (size_t)bytes, (size_t)bytes);
        if (d < best) {
            second = best;
            best = d;
            best_index = (int)g;
        } else if (d < second) {
            second = d;
        }
    }
    out[0] = best_index;
    out[1] = best;
    out[2] = second;
}

/* Forward pass of match_brute_force (src/match.cpp:58-60) over probes
 * [begin, end): out + 3*p receives knn2 of probe p. */
void oracle_knn2_range(const uint8_t* probes, size_t begin, size_t end, const uint8_t* gallery,
                       size_t n, int bytes, int* out) {
    for (size_t p = begin; p < end; ++p)
        oracle_knn2(probes + p * (size_t)bytes, gallery, n, bytes, out + 3 * p);
}

/* Filter pass of match_brute_force — src/match.cpp:69-79. forward is Q x 3
 * (from oracle_knn2_range), reverse_best is N ints or NULL when cross_check is
 * off (src/match.cpp:62-67). Writes up to Q rows {probe, gallery, distance,
 * second} in ascending probe order; returns the row count. The ratio test is
 * evaluated in double exactly as the reference does: best < ratio * second. */
size_t oracle_filter_matches(const int* forward, size_t q, int has_ratio, double ratio,
                             int has_max, int max_distance, const int* reverse_best, int* out) {
    size_t m = 0;
    for (size_t p = 0; p < q; ++p) {
        const int best_index = forward[3 * p], best = forward[3 * p + 1],
                  second = forward[3 * p + 2];
        if (has_ratio && !((double)best < ratio * (double)second)) continue;
        if (has_max && best > max_distance) continue;
        if (reverse_best && reverse_best[best_index] != (int)p) continue;
        out[4 * m + 0] = (int)p;
        out[4 * m + 1] = best_index;
        out[4 * m + 2] = best;
        out[4 * m + 3] = second;
        ++m;
    }
    return m;
}

/* match_brute_force — src/match.cpp:52-81, single thread. Returns the match
 * count, or (size_t)-1 for an empty gallery (reference: EmptyGallery, checked
 * before the empty-probes early-out). */
size_t oracle_match(const uint8_t* probes, size_t q, const uint8_t* gallery, size_t n, int bytes,
                    int has_ratio, double ratio, int cross_check, int has_max, int max_distance,
                    int* out) {
    if (n == 0) return (size_t)-1;
    if (q == 0) return 0;
    int* forward = (int*)malloc(sizeof(int) * 3 * q);
    oracle_knn2_range(probes, 0, q, gallery, n, bytes, forward);
    int* reverse_best = NULL;
    if (cross_check) {
        reverse_best = (int*)malloc(sizeof(int) * n);
        for (size_t g = 0; g < n; ++g) {
            int r[3];
            oracle_knn2(gallery + g * (size_t)bytes, probes, q, bytes, r);
            reverse_best[g] = r[0];
        }
    }
    const size_t m = oracle_filter_matches(forward, q, has_ratio, ratio, has_max, max_distance,
                                           reverse_best, out);
    free(forward);
    free(reverse_best);
    return m;
}

/* ------------------------------------------------------------------------
 * Detection (the step before the hot path; "next" row of SURVEY.md §8f)
 * ---------------------------------------------------------------------- */

/* Radius-3 Bresenham circle, clockwise from 12 o'clock — src/detect.cpp:14-16. */
static const int kCircleX[16] = {0, 1, 2, 3, 3, 3, 2, 1, 0, -1, -2, -3, -3, -3, -2, -1};
static const int kCircleY[16] = {-3, -3, -2, -1, 0, 1, 2, 3, 3, 3, 2, 1, 0, -1, -2, -3};

/* evaluate_arc — src/detect.cpp:26-66: segment test at (x, y); score of the maximal
 * contiguous qualifying arc (bright polarity tried first), 0 when it does not fire. */
static double evaluate_arc(const double* img, int w, int x, int y, double threshold) {
    const double center = img[(size_t)y * w + x];
    const double hi = center + threshold;
    const double lo = center - threshold;
    int bright[16], dark[16];
    for (int i = 0; i < 16; ++i) {
        const double v = img[(size_t)(y + kCircleY[i]) * w + (x + kCircleX[i])];
        bright[i] = v > hi;
        dark[i] = v < lo;
    }
    for (int pol = 0; pol < 2; ++pol) {
        const int* mask = pol == 0 ? bright : dark;
        int best_len = 0, best_start = 0, run = 0;
        for (int i = 0; i < 32; ++i) {   /* two laps cover the wraparound */
            if (mask[i % 16]) {
                ++run;
                if (run > best_len) {
                    best_len = run;
                    best_start = i - run + 1;
                }
            } else {
                run = 0;
            }
        }
        if (best_len > 16) best_len = 16;
        if (best_len < 9) continue;
        double score = 0.0;
        for (int i = best_start; i < best_start + best_len; ++i) {
            const int idx = ((i % 16) + 16) % 16;
            score += fabs(img[(size_t)(y + kCircleY[idx]) * w + (x + kCircleX[idx])] - center) - threshold;
        }
        return score;
    }
    return 0.0;
}

/* fast_detect — src/detect.cpp:76-117. out: up to cap rows {x, y, 0, score} in (y, x)
 * order. Returns the number of detections (which may exceed cap), or (size_t)-1 for an
 * image smaller than 7x7 (reference: ImageTooSmall). */
size_t oracle_fast_detect(const double* img, int w, int h, double threshold, int do_nms, double* out,
                          size_t cap) {
    if (w < 7 || h < 7) return (size_t)-1;
    const int x_end = w - 3, y_end = h - 3;
    double* scores = (double*)calloc((size_t)w * h, sizeof(double));
    for (int y = 3; y < y_end; ++y)
        for (int x = 3; x < x_end; ++x) scores[(size_t)y * w + x] = evaluate_arc(img, w, x, y, threshold);
    size_t n = 0;
    for (int y = 3; y < y_end; ++y) {
        for (int x = 3; x < x_end; ++x) {
            const double s = scores[(size_t)y * w + x];
            if (s <= 0.0) continue;
            if (do_nms) {
                int is_max = 1;
                for (int dy = -1; dy <= 1 && is_max; ++dy) {
                    for (int dx = -1; dx <= 1; ++dx) {
                        if (dx == 0 && dy == 0) continue;
                        const int nx = x + dx, ny = y + dy;
                        if (nx < 3 || ny < 3 || nx >= x_end || ny >= y_end) continue;
                        const double ns = scores[(size_t)ny * w + nx];
                        /* ties keep the lexicographically smallest (y, x) */
                        if (ns > s || (ns == s && (ny < y || (ny == y && nx < x)))) {
                            is_max = 0;
                            break;
                        }
                    }
                }
                if (!is_max) continue;
            }
            if (n < cap) {
                out[4 * n + 0] = (double)x;
                out[4 * n + 1] = (double)y;
                out[4 * n + 2] = 0.0;
                out[4 * n + 3] = s;
            }
            ++n;
        }
    }
    free(scores);
    return n;
}

/* orient — src/detect.cpp:119-146 for an integer-centred keypoint (every FAST detection):
 * theta = atan2(m01, m10) over the disc u^2 + v^2 <= radius^2, 0 when both moments vanish.
 * Returns 1 (and leaves theta alone) when the disc leaves the image. */
int oracle_orient(const double* img, int w, int h, double x, double y, int radius, double* theta) {
    if (!(x - radius >= 0.0 && y - radius >= 0.0 && x + radius <= w - 1 && y + radius <= h - 1)) return 1;
    double m10 = 0.0, m01 = 0.0;
    for (int v = -radius; v <= radius; ++v)
        for (int u = -radius; u <= radius; ++u) {
            if (u * u + v * v > radius * radius) continue;
            const double intensity = img[(size_t)((int)y + v) * w + ((int)x + u)];
            m10 += u * intensity;
            m01 += v * intensity;
        }
    *theta = (m10 == 0.0 && m01 == 0.0) ? 0.0 : atan2(m01, m10);
    return 0;
}

/* detect_and_orient — src/detect.cpp:148-157. */
size_t oracle_detect_and_orient(const double* img, int w, int h, double threshold, int do_nms, int radius,
                                double* out, size_t cap) {
    const size_t raw_cap = (size_t)w * h;
    double* raw = (double*)malloc(sizeof(double) * 4 * (raw_cap ? raw_cap : 1));
    const size_t n = oracle_fast_detect(img, w, h, threshold, do_nms, raw, raw_cap);
    if (n == (size_t)-1) {
        free(raw);
        return n;
    }
    size_t m = 0;
    for (size_t i = 0; i < n; ++i) {
        double theta = 0.0;
        if (oracle_orient(img, w, h, raw[4 * i], raw[4 * i + 1], radius, &theta)) continue;
        if (m < cap) {
            out[4 * m + 0] = raw[4 * i];
            out[4 * m + 1] = raw[4 * i + 1];
            out[4 * m + 2] = theta;
            out[4 * m + 3] = raw[4 * i + 3];
        }
        ++m;
    }
    free(raw);
    return m;
}

/* ------------------------------------------------------------------------
 * Trainer scoring (next row): triplet_bits_over — src/pattern.cpp:340-346, the body of
 * select_triplets' parallel_for (:397-400). windows: n upright 64x64 patches
 * (Window64::from_image, src/descriptor.cpp:13-21); candidates: C x 6 ints. out: C rows of
 * `row_bytes` bytes, bit i of row c = triplet_bit(window i, candidate c) stored LSB-first
 * (BitVector, include/latch/pattern.hpp:70-90).
 * ---------------------------------------------------------------------- */
void oracle_triplet_bits(const double* windows, size_t n, const int* candidates, size_t C, int K,
                         const double* weights, uint8_t* out, size_t row_bytes) {
    memset(out, 0, C * row_bytes);
    for (size_t c = 0; c < C; ++c)
        for (size_t i = 0; i < n; ++i)
            if (oracle_triplet_bit(windows + i * 4096, candidates + 6 * c, K, weights))
                out[c * row_bytes + (i >> 3)] |= (uint8_t)(1u << (i & 7));
}
