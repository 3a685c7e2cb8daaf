// latch-b200: the reference's `latch detect | describe | match` command line (proj/src/cli.cpp:52-81, 113-199)
// over the B200 library — same sub-commands, options, file formats and exit codes, so a file-based pipeline can
// switch binaries without touching its files:
//   detect    --image in.pgm [--threshold 20] [--no-nms] --out keypoints.tsv
//   describe  --image in.pgm --keypoints kp.tsv [--pattern default|file] --out descriptors.ltch [--workers n]
//   match     --probe a.ltch --gallery b.ltch [--ratio r] [--cross-check] [--max-distance d] --out matches.tsv
// `train` and `eval` are host-side tools outside the hot path: they stay with the reference binary
// and are refused here with a usage error. Exit codes: 0 ok, 1 usage, 2 latch::Error, 3 anything else.
// The option parser is hand-rolled (the reference uses CLI11, which is not vendored): `--name value` and
// `--name=value`, flags without values, `-h/--help`.
#include <cstdio>
#include <iostream>
#include <map>
#include <set>
#include <string>
#include <vector>

#include "latch_b200.hpp"

namespace {

struct Spec {
    std::set<std::string> valued, flags, required;
};

const std::map<std::string, Spec>& specs() {
    static const std::map<std::string, Spec> s = {
        {"detect", {{"--image", "--threshold", "--out"}, {"--no-nms"}, {"--image", "--out"}}},
        {"describe", {{"--image", "--keypoints", "--pattern", "--out", "--workers"}, {}, {"--image", "--keypoints", "--out"}}},
        {"match", {{"--probe", "--gallery", "--ratio", "--max-distance", "--out", "--workers"}, {"--cross-check"},
                   {"--probe", "--gallery", "--out"}}},
    };
    return s;
}

int usage(const std::string& message) {
    std::cerr << "error: " << message << "\n"
              << "usage: latch-b200 detect|describe|match [options]   (see --help)\n";
    return 1;
}

void help() {
    std::cout << "LATCH binary descriptors on B200: detect, describe, match\n"
                 "  detect    --image PGM [--threshold 20] [--no-nms] --out TSV\n"
                 "  describe  --image PGM --keypoints TSV [--pattern default|FILE] --out LTCH [--workers N]\n"
                 "  match     --probe LTCH --gallery LTCH [--ratio R] [--cross-check] [--max-distance D] --out TSV [--workers N]\n"
                 "train / eval: use the reference binary (host-side tools outside the GPU path)\n";
}

bool to_double(const std::string& s, double& v) {
    char* end = nullptr;
    v = std::strtod(s.c_str(), &end);
    return !s.empty() && end && *end == '\0';
}
bool to_int(const std::string& s, int& v) {
    char* end = nullptr;
    const long x = std::strtol(s.c_str(), &end, 10);
    v = static_cast<int>(x);
    return !s.empty() && end && *end == '\0';
}

} // namespace

int main(int argc, char** argv) {
    if (argc < 2) return usage("a sub-command is required");
    const std::string cmd = argv[1];
    if (cmd == "-h" || cmd == "--help") {
        help();
        return 0;
    }
    if (cmd == "train" || cmd == "eval")
        return usage("'" + cmd + "' is a host-side tool outside the GPU path: run it with the reference binary");
    const auto spec = specs().find(cmd);
    if (spec == specs().end()) return usage("unknown sub-command '" + cmd + "'");
    std::map<std::string, std::string> opt;
    for (int i = 2; i < argc; ++i) {
        std::string name = argv[i], value;
        if (name == "-h" || name == "--help") {
            help();
            return 0;
        }
        const std::size_t eq = name.find('=');
        const bool inline_value = eq != std::string::npos;
        if (inline_value) {
            value = name.substr(eq + 1);
            name = name.substr(0, eq);
        }
        if (spec->second.flags.count(name)) {
            if (inline_value) return usage(name + " takes no value");
            opt[name] = "1";
        } else if (spec->second.valued.count(name)) {
            if (!inline_value) {
                if (i + 1 >= argc) return usage(name + " needs a value");
                value = argv[++i];
            }
            opt[name] = value;
        } else {
            return usage("unknown option '" + name + "' for " + cmd);
        }
    }
    for (const std::string& r : spec->second.required)
        if (!opt.count(r)) return usage(r + " is required");

    // range checks, all usage errors (proj/src/cli.cpp:166-177)
    double threshold = latch::kDefaultFastThreshold, ratio = 0.0;
    int workers = 0, max_distance = 0;
    if (opt.count("--threshold") && !to_double(opt["--threshold"], threshold)) return usage("--threshold must be a number");
    if (opt.count("--ratio") && !to_double(opt["--ratio"], ratio)) return usage("--ratio must be a number");
    if (opt.count("--workers") && !to_int(opt["--workers"], workers)) return usage("--workers must be an integer");
    if (opt.count("--max-distance") && !to_int(opt["--max-distance"], max_distance)) return usage("--max-distance must be an integer");
    if (opt.count("--ratio") && !(ratio > 0.0 && ratio <= 1.0)) return usage("--ratio must be in (0, 1]");
    if (opt.count("--max-distance") && max_distance < 0) return usage("--max-distance must be >= 0");
    if (threshold <= 0.0) return usage("--threshold must be > 0");
    if (workers < 0) return usage("--workers must be >= 0");

    try {
        if (cmd == "detect") {
            const latch::Image image = latch::load_pgm_file(opt["--image"]);
            latch::save_keypoints_file(latch::detect_and_orient(image, threshold, !opt.count("--no-nms")), opt["--out"]);
        } else if (cmd == "describe") {
            const latch::Image image = latch::load_pgm_file(opt["--image"]);
            const std::vector<latch::Keypoint> keypoints = latch::load_keypoints_file(opt["--keypoints"]);
            const std::string pat = opt.count("--pattern") ? opt["--pattern"] : "default";
            const latch::TripletPattern pattern = pat == "default" ? latch::default_pattern() : latch::load_pattern_file(pat);
            latch::save_descriptor_file(latch::describe_all(image, keypoints, pattern, workers), opt["--out"]);
        } else {
            std::vector<latch::Descriptor> probes, gallery;
            for (auto& rec : latch::load_descriptor_file(opt["--probe"])) probes.push_back(std::move(rec.second));
            for (auto& rec : latch::load_descriptor_file(opt["--gallery"])) gallery.push_back(std::move(rec.second));
            latch::MatchOptions options;
            if (opt.count("--ratio")) options.ratio = ratio;
            options.cross_check = opt.count("--cross-check") != 0;
            if (opt.count("--max-distance")) options.max_distance = max_distance;
            options.workers = workers;
            latch::save_matches_file(latch::match_brute_force(probes, gallery, options), opt["--out"]);
        }
    } catch (const latch::Error& e) {
        std::cerr << "error: " << e.what() << "\n";
        return 2;
    } catch (const std::exception& e) {
        std::cerr << "internal error: " << e.what() << "\n";
        return 3;
    }
    return 0;
}
