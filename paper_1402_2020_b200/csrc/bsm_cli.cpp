// bsm_cli.cpp -- the command-line tool over the GPU pipeline: the reference
// tool's subcommands, flags, output files and printed lines (tools/bsm.cpp),
// written against the C++ drop-in headers (include/bsm).  Built by the csrc
// Makefile into paper_1402_2020_b200/bsm.
//
//   bsm match LEFT RIGHT OUT [--stages] [--pattern P] [--emit-pattern P]
//   bsm eval RESULT GT [--nonocc M] [--all M] [--disc M] [--threshold T]
//   bsm sweep SCENE... [--n_values 512,1024,...] [--out CSV] [--threshold T]
//   bsm radiometric SET [--out CSV] [--threshold T]
//   bsm bench LEFT RIGHT [--runs K]
// plus --config FILE and the BsmConfig flags on every subcommand (explicit
// flags > config file > defaults).
#include <cstdio>
#include <cstdlib>
#include <filesystem>
#include <functional>
#include <map>
#include <optional>
#include <string>
#include <vector>

#include "bsm/bsm.hpp"

namespace {

struct Usage : std::runtime_error {
    using std::runtime_error::runtime_error;
};

// Minimal subcommand parser: positionals in order, `--name value`,
// `--name=value`, boolean flags.
struct Args {
    std::vector<std::string> pos;
    std::map<std::string, std::string> opt;
    std::map<std::string, bool> flag;
};

Args parse(const std::vector<std::string>& av, const std::vector<std::string>& options,
           const std::vector<std::string>& flags) {
    Args a;
    auto known = [](const std::vector<std::string>& v, const std::string& s) {
        for (const std::string& x : v)
            if (x == s) return true;
        return false;
    };
    for (std::size_t i = 0; i < av.size(); ++i) {
        const std::string& s = av[i];
        if (s.rfind("--", 0) != 0) {
            a.pos.push_back(s);
            continue;
        }
        const std::size_t eq = s.find('=');
        const std::string name = s.substr(0, eq);
        if (known(flags, name) && eq == std::string::npos) {
            a.flag[name] = true;
        } else if (known(options, name)) {
            if (eq != std::string::npos) a.opt[name] = s.substr(eq + 1);
            else if (i + 1 < av.size()) a.opt[name] = av[++i];
            else throw Usage(name + " requires an argument");
        } else {
            throw Usage("The following argument was not expected: " + s);
        }
    }
    return a;
}

const std::vector<std::string> kCfgOpts = {"--config", "--n", "--S", "--spread", "--seed", "--d_max", "--lambda_c",
                                           "--lambda_e", "--lr_tolerance", "--vote_radius", "--gt_scale",
                                           "--threads"};

void apply_flags(const Args& a, bsm::BsmConfig& c) {
    auto get = [&](const char* k) -> const std::string* {
        auto it = a.opt.find(k);
        return it == a.opt.end() ? nullptr : &it->second;
    };
    auto num = [&](const std::string& s, const char* k) {
        char* end = nullptr;
        const double v = std::strtod(s.c_str(), &end);
        if (end == s.c_str() || *end) throw Usage(std::string("invalid value for ") + k + ": " + s);
        return v;
    };
    if (auto s = get("--n")) c.n = int(num(*s, "--n"));
    if (auto s = get("--S")) c.window = int(num(*s, "--S"));
    if (auto s = get("--spread")) c.spread = num(*s, "--spread");
    if (auto s = get("--seed")) c.seed = std::strtoull(s->c_str(), nullptr, 10);
    if (auto s = get("--d_max")) c.d_max = int(num(*s, "--d_max"));
    if (auto s = get("--lambda_c")) c.lambda_c = num(*s, "--lambda_c");
    if (auto s = get("--lambda_e")) c.lambda_e = num(*s, "--lambda_e");
    if (auto s = get("--lr_tolerance")) c.lr_tolerance = num(*s, "--lr_tolerance");
    if (auto s = get("--vote_radius")) c.vote_radius = int(num(*s, "--vote_radius"));
    if (auto s = get("--gt_scale")) c.gt_scale = num(*s, "--gt_scale");
    if (auto s = get("--threads")) c.threads = int(num(*s, "--threads"));
}

std::string stage_path(const std::string& out, const char* stage) {
    std::filesystem::path p(out);
    const std::string ext = p.extension().string();
    p.replace_extension();
    return p.string() + "." + stage + ext;
}

void write_map(const bsm::DisparityMap& m, const std::string& path, double scale) {
    if (std::filesystem::path(path).extension() == ".pfm") bsm::save_disparity_pfm(m, path);
    else bsm::save_disparity(m, path, scale);
}

void report(const char* label, const bsm::ErrorReport& r) {
    std::printf("%-8s %6.2f  (%ld of %ld pixels beyond %.2f)\n", label, r.bad_pixel_rate, r.bad, r.counted,
                r.threshold);
}

double opt_double(const Args& a, const char* k, double def) {
    auto it = a.opt.find(k);
    return it == a.opt.end() ? def : std::strtod(it->second.c_str(), nullptr);
}

std::string opt_string(const Args& a, const char* k, const std::string& def) {
    auto it = a.opt.find(k);
    return it == a.opt.end() ? def : it->second;
}

void need_positionals(const Args& a, std::size_t lo, std::size_t hi, const char* cmd) {
    if (a.pos.size() < lo) throw Usage(std::string(cmd) + ": missing required positional arguments");
    if (a.pos.size() > hi) throw Usage(std::string(cmd) + ": too many positional arguments");
}

int run(int argc, char** argv) {
    std::vector<std::string> av(argv + 1, argv + argc);
    if (av.empty()) throw Usage("A subcommand is required");
    const std::string cmd = av[0];
    av.erase(av.begin());
    bsm::BsmConfig cfg;
    for (std::size_t i = 0; i < av.size(); ++i) {  // the config file loads before flags apply
        if (av[i] == "--config" && i + 1 < av.size()) cfg = bsm::load_config(av[i + 1]);
        else if (av[i].rfind("--config=", 0) == 0) cfg = bsm::load_config(av[i].substr(9));
    }
    auto opts = [](std::vector<std::string> extra) {
        extra.insert(extra.end(), kCfgOpts.begin(), kCfgOpts.end());
        return extra;
    };
    if (cmd == "match") {
        const Args a = parse(av, opts({"--pattern", "--emit-pattern"}), {"--stages"});
        need_positionals(a, 3, 3, "match");
        apply_flags(a, cfg);
        const bsm::RgbImage left = bsm::load_image(a.pos[0]), right = bsm::load_image(a.pos[1]);
        cfg.validate();
        const std::string pin = opt_string(a, "--pattern", "");
        const bsm::SamplingPattern pat = pin.empty() ? bsm::generate_pattern(cfg) : bsm::load_pattern(pin);
        const bool stages = a.flag.count("--stages") > 0;
        const bsm::PipelineResult res = bsm::run_pipeline(left, right, pat, cfg, stages);
        const std::string& out = a.pos[2];
        write_map(res.refined, out, cfg.gt_scale);
        bsm::save_config(cfg, out + ".config.json");
        if (stages) {
            write_map(*res.unmasked, stage_path(out, "unmasked"), cfg.gt_scale);
            write_map(res.left_wta, stage_path(out, "masked"), cfg.gt_scale);
            write_map(res.refined, stage_path(out, "refined"), cfg.gt_scale);
        }
        const std::string pout = opt_string(a, "--emit-pattern", "");
        if (!pout.empty()) bsm::save_pattern(pat, pout);
    } else if (cmd == "eval") {
        const Args a = parse(av, opts({"--nonocc", "--all", "--disc", "--threshold"}), {});
        need_positionals(a, 2, 2, "eval");
        apply_flags(a, cfg);
        const double thr = opt_double(a, "--threshold", 1.0);
        const bsm::DisparityMap result = bsm::load_gt_disparity(a.pos[0], cfg.gt_scale);
        const bsm::DisparityMap gt = bsm::load_gt_disparity(a.pos[1], cfg.gt_scale);
        bool any = false;
        for (const char* r : {"nonocc", "all", "disc"}) {
            const std::string p = opt_string(a, (std::string("--") + r).c_str(), "");
            if (p.empty()) continue;
            any = true;
            const bsm::GrayImage m = bsm::to_gray(bsm::load_image(p));
            report(r, bsm::bad_pixel_rate(result, gt, &m, thr));
        }
        if (!any) report("all", bsm::bad_pixel_rate(result, gt, nullptr, thr));
    } else if (cmd == "sweep") {
        const Args a = parse(av, opts({"--n_values", "--out", "--threshold"}), {});
        need_positionals(a, 1, 1u << 20, "sweep");
        apply_flags(a, cfg);
        std::vector<int> ns;
        const std::string nv = opt_string(a, "--n_values", "512,1024,2048,4096");
        for (std::size_t b = 0; b < nv.size();) {
            const std::size_t e = nv.find(',', b);
            const std::string t = nv.substr(b, e == std::string::npos ? std::string::npos : e - b);
            if (!t.empty()) ns.push_back(std::atoi(t.c_str()));
            if (e == std::string::npos) break;
            b = e + 1;
        }
        std::vector<bsm::StereoDataset> sets;
        for (const std::string& dir : a.pos) {
            const std::string name = std::filesystem::path(dir).filename().string();
            int d = cfg.d_max;
            double scale = cfg.gt_scale;
            for (const bsm::MiddleburyParams& s : bsm::kMiddleburyScenes)
                if (name == s.name) {
                    if (d <= 0) d = s.d_max;
                    scale = s.gt_scale;
                }
            if (d < 1) throw bsm::InvalidArgument("sweep: " + dir + " is not a known scene, pass --d_max");
            sets.push_back(bsm::load_stereo_dataset(dir, name, d, scale));
        }
        std::vector<bsm::SweepScene> scenes;
        for (const bsm::StereoDataset& ds : sets)
            scenes.push_back({&ds.left, &ds.right, &ds.gt, ds.mask_nonocc ? &*ds.mask_nonocc : nullptr, ds.d_max});
        const std::vector<bsm::SweepPoint> pts =
            bsm::length_sweep(scenes, ns, cfg, opt_double(a, "--threshold", 1.0));
        std::printf("%6s  %9s  %12s\n", "n", "avg_error", "wall_seconds");
        std::vector<double> xs, ys;
        for (const bsm::SweepPoint& p : pts) {
            std::printf("%6d  %9.4f  %12.2f\n", p.n, p.avg_error, p.wall_time);
            xs.push_back(double(p.n));
            ys.push_back(p.wall_time);
        }
        if (pts.size() >= 2) std::printf("linear fit of time vs n: R^2 = %.4f\n", bsm::linear_fit_r2(xs, ys));
        const std::string out = opt_string(a, "--out", "sweep.csv");
        bsm::write_sweep_csv(out, pts);
        bsm::save_config(cfg, out + ".config.json");
    } else if (cmd == "radiometric") {
        const Args a = parse(av, opts({"--out", "--threshold"}), {});
        need_positionals(a, 1, 1, "radiometric");
        apply_flags(a, cfg);
        cfg.validate();
        const bsm::RadiometricSet set = bsm::load_radiometric_set(a.pos[0], cfg.d_max, cfg.gt_scale);
        const bsm::SamplingPattern pat = bsm::generate_pattern(cfg);
        const bsm::RadiometricMatrix m =
            bsm::radiometric_protocol(set.lefts, set.rights, set.gt, set.mask_nonocc ? &*set.mask_nonocc : nullptr,
                                      pat, cfg, opt_double(a, "--threshold", 1.0));
        std::printf("%12s %8s %8s %8s\n", "left\\right", "c0", "c1", "c2");
        for (int i = 0; i < 3; ++i)
            std::printf("%12s %8.2f %8.2f %8.2f\n", ("c" + std::to_string(i)).c_str(), m.rate[std::size_t(i)][0],
                        m.rate[std::size_t(i)][1], m.rate[std::size_t(i)][2]);
        std::printf("diagonal mean %.2f, off-diagonal mean %.2f\n", m.diagonal_mean(), m.off_diagonal_mean());
        const std::string out = opt_string(a, "--out", "radiometric.csv");
        bsm::write_radiometric_csv(out, m);
        bsm::save_config(cfg, out + ".config.json");
    } else if (cmd == "bench") {
        const Args a = parse(av, opts({"--runs"}), {});
        need_positionals(a, 2, 2, "bench");
        apply_flags(a, cfg);
        const int runs = int(opt_double(a, "--runs", 3));
        const bsm::RgbImage left = bsm::load_image(a.pos[0]), right = bsm::load_image(a.pos[1]);
        cfg.validate();
        const bsm::SamplingPattern pat = bsm::generate_pattern(cfg);
        const double secs = bsm::time_pipeline(left, right, pat, cfg, runs);
        std::printf("median of %d run%s: %.2f s (%dx%d, d_max=%d, n=%d, threads=%d)\n", runs, runs == 1 ? "" : "s",
                    secs, left.width, left.height, cfg.d_max, cfg.n, cfg.threads);
    } else {
        throw Usage("unknown subcommand '" + cmd + "' (match, eval, sweep, radiometric, bench)");
    }
    return 0;
}

}  // namespace

int main(int argc, char** argv) {
    try {
        return run(argc, argv);
    } catch (const Usage& e) {
        std::fprintf(stderr, "%s\nusage: bsm {match|eval|sweep|radiometric|bench} ... (see --help in DESIGN.md)\n",
                     e.what());
        return 106;
    } catch (const std::exception& e) {
        std::fprintf(stderr, "error: %s\n", e.what());
        return 1;
    }
}
