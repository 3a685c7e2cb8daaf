// Bank-conflict-aware placement of triplets onto lanes for the specialised
// extraction kernel (host side, runs once per clatch_set_pattern).
//
// In the SSD phase lane j of a warp reads window[(y_j + r) * stride + x_j + c] for its
// own triplet's anchor / companion patches with 64-bit shared loads. Such a load is
// served per half-warp (16 lanes x 8 B = 128 B) and is conflict-free iff the 16 lanes
// hit 16 distinct 8-byte bank pairs, i.e. distinct (y_j * stride + x_j) mod 16 — the
// same for every (r, c) step because all lanes advance by the same offset. Measured on
// B200 (profiles/r1a_pipe_peaks.json): 126.8 B/clk/SM when distinct, 42 B/clk/SM for
// random slots. With the triplets in table order the average degree is 3.1
// (profiles/r1a_extract_ncu.json: 65 % of shared wavefronts are conflict replays).
//
// Freedom used here: (1) which triplet sits in which (half-warp, lane) slot — the bit
// index travels with the slot; (2) swapping the two companions of a triplet (the kernel
// then tests d2 > d1 instead of d1 > d2, i.e. the same predicate). A deterministic
// simulated annealing minimises sum over (half-warp, load) of the worst bank-pair
// multiplicity, with the number of colliding lanes as a tie-breaking gradient.
#pragma once

#include <algorithm>
#include <cmath>
#include <cstdint>
#include <utility>
#include <vector>

namespace clatch {

struct SlotEntry {
    uint16_t a, b, c;   // window offsets (y * stride + x) of the loads issued 1st, 2nd, 3rd
    uint16_t bit;       // descriptor bit index; bit 15 set => companions swapped
};

struct SlotPlan {
    std::vector<SlotEntry> slots;   // T entries, slot = thread-visible position
    double avg_degree = 0.0;        // mean worst multiplicity over (half-warp, load)
    double avg_degree_identity = 0.0;
};

namespace detail {

struct GroupHist {
    uint8_t h[3][16];
};

inline int hist_cost(const uint8_t* h) {
    int mx = 0, excess = 0;
    for (int r = 0; r < 16; ++r) {
        mx = std::max<int>(mx, h[r]);
        excess += h[r] > 1 ? h[r] - 1 : 0;
    }
    return 16 * mx + excess;
}

inline int hist_degree(const uint8_t* h) {
    int mx = 0;
    for (int r = 0; r < 16; ++r) mx = std::max<int>(mx, h[r]);
    return mx;
}

} // namespace detail

// triplets: T x {ax, ay, bx, by, cx, cy}. T must be a multiple of 16.
inline SlotPlan plan_slots(const int16_t* triplets, int T, int stride, int iterations = 400000) {
    using namespace detail;
    const int G = T / 16;
    std::vector<uint16_t> off(3 * T);
    for (int t = 0; t < T; ++t)
        for (int k = 0; k < 3; ++k)
            off[3 * t + k] = static_cast<uint16_t>(triplets[6 * t + 2 * k + 1] * stride + triplets[6 * t + 2 * k]);

    std::vector<int> order(T);            // order[slot] = triplet
    std::vector<uint8_t> flip(T, 0);      // per triplet
    for (int t = 0; t < T; ++t) order[t] = t;
    auto res = [&](int t, int k) {        // residue of load k of triplet t under its flip
        const int kk = (k == 0 || !flip[t]) ? k : 3 - k;
        return off[3 * t + kk] & 15;
    };
    std::vector<GroupHist> hist(G);
    auto rebuild = [&](int g) {
        GroupHist gh{};
        for (int l = 0; l < 16; ++l)
            for (int k = 0; k < 3; ++k) ++gh.h[k][res(order[16 * g + l], k)];
        hist[g] = gh;
    };
    auto gcost = [&](int g) { return hist_cost(hist[g].h[0]) + hist_cost(hist[g].h[1]) + hist_cost(hist[g].h[2]); };
    auto degree = [&]() {
        double s = 0;
        for (int g = 0; g < G; ++g)
            for (int k = 0; k < 3; ++k) s += hist_degree(hist[g].h[k]);
        return s / (3.0 * G);
    };
    for (int g = 0; g < G; ++g) rebuild(g);
    SlotPlan plan;
    plan.avg_degree_identity = degree();

    uint64_t rng = 0x9E3779B97F4A7C15ull;   // fixed seed: the plan is a pure function of the pattern
    auto next = [&]() {
        rng ^= rng << 13;
        rng ^= rng >> 7;
        rng ^= rng << 17;
        return rng;
    };
    std::vector<int> cost(G);
    for (int g = 0; g < G; ++g) cost[g] = gcost(g);
    const double t0 = 6.0;
    for (int it = 0; it < iterations && G > 1; ++it) {
        const double temp = t0 * (1.0 - static_cast<double>(it) / iterations) + 0.05;
        const uint64_t r = next();
        const auto accept = [&](int delta) {
            if (delta <= 0) return true;
            const double u = static_cast<double>((next() >> 11) & 0xFFFFF) / 1048576.0;
            return u < std::exp(-delta / temp);
        };
        if ((r & 7) == 0) {                       // flip the companions of one triplet
            const int p = static_cast<int>((r >> 8) % T), g = p / 16, t = order[p];
            const GroupHist saved = hist[g];
            for (int k = 1; k < 3; ++k) --hist[g].h[k][res(t, k)];
            flip[t] ^= 1;
            for (int k = 1; k < 3; ++k) ++hist[g].h[k][res(t, k)];
            const int nc = gcost(g);
            if (accept(nc - cost[g])) cost[g] = nc;
            else { flip[t] ^= 1; hist[g] = saved; }
            continue;
        }
        const int p = static_cast<int>((r >> 8) % T), q = static_cast<int>((r >> 32) % T);
        const int g1 = p / 16, g2 = q / 16;
        if (g1 == g2) continue;
        const GroupHist s1 = hist[g1], s2 = hist[g2];
        const int tp = order[p], tq = order[q];
        for (int k = 0; k < 3; ++k) {
            --hist[g1].h[k][res(tp, k)]; ++hist[g1].h[k][res(tq, k)];
            --hist[g2].h[k][res(tq, k)]; ++hist[g2].h[k][res(tp, k)];
        }
        const int n1 = gcost(g1), n2 = gcost(g2);
        if (accept(n1 + n2 - cost[g1] - cost[g2])) {
            order[p] = tq; order[q] = tp; cost[g1] = n1; cost[g2] = n2;
        } else {
            hist[g1] = s1; hist[g2] = s2;
        }
    }
    plan.avg_degree = degree();
    plan.slots.resize(T);
    for (int s = 0; s < T; ++s) {
        const int t = order[s];
        SlotEntry e;
        e.a = off[3 * t + 0];
        e.b = off[3 * t + (flip[t] ? 2 : 1)];
        e.c = off[3 * t + (flip[t] ? 1 : 2)];
        e.bit = static_cast<uint16_t>(t | (flip[t] ? 0x8000 : 0));
        plan.slots[s] = e;
    }
    return plan;
}

// ---- grouped placement ("quad" and "filtered" kernels) ---------------------------------------
// The multi-window kernels keep FOUR keypoints' windows in shared memory and fill each
// conflict domain with `group` triplets x 4 keypoints, window w displaced by `mod`*w banks:
//   quad kernel      64-bit loads, domain = half-warp = 16 bank pairs: group 4, mod 4
//                    (lane = 4*i + w; window w displaced by 4*w bank pairs)
//   filtered kernel  32-bit loads, domain = warp = 32 banks:           group 8, mod 8
//                    (lane = 4*i + w; window w displaced by 8*w banks)
// The lanes of one triplet then sit on residues x, x+mod, x+2*mod, x+3*mod, so a domain is
// conflict-free as soon as its `group` triplets have distinct residues MOD `mod` in each of
// the three loads — far weaker than distinct residues across the whole domain. What remains
// is the histogram imbalance of the table (a residue class holding more than T/mod anchors
// forces a collision somewhere): degree 1.07 for (4,4), 1.14 for (8,8) on the built-in table.
// Packed 16-bit planes (extract_h16_kernel): a window is stored twice as 16-bit samples, row stride 33 words —
// copy E holds sample (v, u) in halfword 66 v + u, copy O (kH16CopyWords further on) in halfword 66 v + u + 1 — so
// the 7 live pixels of a patch row that starts at ANY column are four aligned 32-bit words of one of the copies.
// A patch anchored at column x, row y is addressed by the word offset of its first pair.
constexpr int kH16RowWords = 33, kH16CopyWords = 64 * kH16RowWords;
inline uint16_t h16_offset(int x, int y) {
    return static_cast<uint16_t>((x & 1) * kH16CopyWords + y * kH16RowWords + ((x + 1) >> 1));
}
// ... and back: word offset -> (column, row) of the patch anchor.
inline void h16_anchor(unsigned off, int& x, int& y) {
    const int odd = off >= static_cast<unsigned>(kH16CopyWords);
    const int r = static_cast<int>(off) - odd * kH16CopyWords;
    y = r / kH16RowWords;
    x = 2 * (r % kH16RowWords) - odd;
}

inline SlotPlan plan_slots_grouped_off(std::vector<uint16_t> off, int T, int group, int mod, int iterations);

inline SlotPlan plan_slots_grouped(const int16_t* triplets, int T, int stride, int group, int mod,
                                   int iterations) {
    std::vector<uint16_t> off(3 * T);
    for (int t = 0; t < T; ++t)
        for (int k = 0; k < 3; ++k)
            off[3 * t + k] = static_cast<uint16_t>(triplets[6 * t + 2 * k + 1] * stride + triplets[6 * t + 2 * k]);
    return plan_slots_grouped_off(std::move(off), T, group, mod, iterations);
}

// The packed-plane layout: 8 triplets x 4 windows per warp, window w displaced by 8 w banks (as the filtered kernel).
inline SlotPlan plan_slots_h16(const int16_t* triplets, int T, int iterations) {
    std::vector<uint16_t> off(3 * T);
    for (int t = 0; t < T; ++t)
        for (int k = 0; k < 3; ++k) off[3 * t + k] = h16_offset(triplets[6 * t + 2 * k], triplets[6 * t + 2 * k + 1]);
    return plan_slots_grouped_off(std::move(off), T, 8, 8, iterations);
}

inline SlotPlan plan_slots_grouped_off(std::vector<uint16_t> off, int T, int group, int mod, int iterations) {
    const int G = T / group;
    std::vector<int> order(T);
    std::vector<uint8_t> flip(T, 0);
    for (int t = 0; t < T; ++t) order[t] = t;
    auto res = [&](int t, int k) {
        const int kk = (k == 0 || !flip[t]) ? k : 3 - k;
        return off[3 * t + kk] % mod;
    };
    // cost of a group: per load, 16 * (worst multiplicity) + colliding lanes
    auto gcost = [&](int g, int* degree_sum) {
        int cost = 0;
        for (int k = 0; k < 3; ++k) {
            int h[16] = {0};
            for (int l = 0; l < group; ++l) ++h[res(order[group * g + l], k)];
            int mx = 0, excess = 0;
            for (int r = 0; r < mod; ++r) {
                mx = std::max(mx, h[r]);
                excess += h[r] > 1 ? h[r] - 1 : 0;
            }
            cost += 16 * mx + excess;
            if (degree_sum) *degree_sum += mx;
        }
        return cost;
    };
    auto degree = [&]() {
        int sum = 0;
        for (int g = 0; g < G; ++g) gcost(g, &sum);
        return sum / (3.0 * G);
    };
    SlotPlan plan;
    plan.avg_degree_identity = degree();
    uint64_t rng = 0x9E3779B97F4A7C15ull;
    auto next = [&]() {
        rng ^= rng << 13;
        rng ^= rng >> 7;
        rng ^= rng << 17;
        return rng;
    };
    std::vector<int> cost(G);
    for (int g = 0; g < G; ++g) cost[g] = gcost(g, nullptr);
    for (int it = 0; it < iterations && G > 1; ++it) {
        const double temp = 4.0 * (1.0 - static_cast<double>(it) / iterations) + 0.05;
        const uint64_t r = next();
        const auto accept = [&](int delta) {
            if (delta <= 0) return true;
            const double u = static_cast<double>((next() >> 11) & 0xFFFFF) / 1048576.0;
            return u < std::exp(-delta / temp);
        };
        if ((r & 7) == 0) {
            const int p = static_cast<int>((r >> 8) % T), g = p / group, t = order[p];
            flip[t] ^= 1;
            const int nc = gcost(g, nullptr);
            if (accept(nc - cost[g])) cost[g] = nc;
            else flip[t] ^= 1;
            continue;
        }
        const int p = static_cast<int>((r >> 8) % T), q = static_cast<int>((r >> 32) % T);
        const int g1 = p / group, g2 = q / group;
        if (g1 == g2) continue;
        std::swap(order[p], order[q]);
        const int n1 = gcost(g1, nullptr), n2 = gcost(g2, nullptr);
        if (accept(n1 + n2 - cost[g1] - cost[g2])) {
            cost[g1] = n1;
            cost[g2] = n2;
        } else {
            std::swap(order[p], order[q]);
        }
    }
    plan.avg_degree = degree();
    plan.slots.resize(T);
    for (int s = 0; s < T; ++s) {
        const int t = order[s];
        SlotEntry e;
        e.a = off[3 * t + 0];
        e.b = off[3 * t + (flip[t] ? 2 : 1)];
        e.c = off[3 * t + (flip[t] ? 1 : 2)];
        e.bit = static_cast<uint16_t>(t | (flip[t] ? 0x8000 : 0));
        plan.slots[s] = e;
    }
    return plan;
}

inline SlotPlan plan_slots_quad(const int16_t* triplets, int T, int stride, int iterations = 300000) {
    return plan_slots_grouped(triplets, T, stride, 4, 4, iterations);
}

// FNV-1a over the triplet table: identifies the built-in pattern, whose (8,8) plan ships
// precomputed (default_plan_f8.inc, made by tools/gen_default_plan.cpp with a long anneal).
inline uint64_t triplet_hash(const int16_t* triplets, int T) {
    uint64_t h = 0xcbf29ce484222325ull;
    for (int i = 0; i < 6 * T; ++i) {
        h = (h ^ static_cast<uint16_t>(triplets[i])) * 0x100000001b3ull;
    }
    return h;
}

} // namespace clatch
