// `mexp` command line over the B200 drop-in (SURVEY.md section 8(f), ranks 1
// and 4): the reference CLI's subcommands (proj/tools/mexp_cli.cpp:53-163)
// with the same arguments, output format and exit codes. `exp` and `sweep`
// compute on the GPU (include/mexp/expm.hpp, include/mexp/bench.hpp);
// `theta` and `staircase` are table arithmetic.
//
//   mexp exp --in A.txt [--family taylor-new] [--u double|single] [--report]
//   mexp theta [--family taylor] [--u double|single]
//   mexp staircase [--family F] [--u U] [--norm-min X] [--norm-max Y] [--points K] [--out F]
//   mexp sweep [--kinds a,b] [--families f,g] [--n N] [--count C] [--seed S] [--u U]
//              [--norm-min X] [--norm-max Y] [--out F]
#include <cmath>
#include <cstdint>
#include <cstdio>
#include <type_traits>
#include <cstring>
#include <fstream>
#include <iostream>
#include <map>
#include <random>
#include <sstream>
#include <stdexcept>
#include <string>
#include <vector>

#include "mexp/bench.hpp"
#include "mexp/expm.hpp"

namespace {

mexp::Accuracy parse_u(const std::string& s) {
    if (s == "double") return mexp::Accuracy::Double;
    if (s == "single") return mexp::Accuracy::Single;
    throw std::runtime_error("--u must be single or double");
}

mexp::Family parse_family_or_throw(const std::string& s) {
    mexp::Family f;
    if (!mexp::parse_family(s, f)) throw std::runtime_error("unknown family '" + s + "'");
    return f;
}

// --key value / --flag parsing; unknown options are errors
std::map<std::string, std::string> parse_opts(int argc, char** argv, int first,
                                              const std::map<std::string, bool>& spec) {
    std::map<std::string, std::string> out;
    for (int i = first; i < argc; ++i) {
        const std::string k = argv[i];
        const auto it = spec.find(k);
        if (it == spec.end()) throw std::runtime_error("unknown option " + k);
        if (it->second) {
            if (i + 1 >= argc) throw std::runtime_error("missing value for " + k);
            out[k] = argv[++i];
        } else {
            out[k] = "1";
        }
    }
    return out;
}

std::vector<std::string> split_list(const std::string& s) {
    std::vector<std::string> out;
    std::stringstream in(s);
    std::string item;
    while (std::getline(in, item, ','))
        if (!item.empty()) out.push_back(item);
    return out;
}

// stdout, or the --out file
void write_text(const std::string& text, const std::map<std::string, std::string>& o) {
    const auto it = o.find("--out");
    if (it == o.end()) {
        std::cout << text;
        return;
    }
    std::ofstream f(it->second);
    if (!f) throw std::runtime_error("cannot open " + it->second);
    f << text;
}

template <class T>
T num(const std::map<std::string, std::string>& o, const char* key, T dflt) {
    const auto it = o.find(key);
    if (it == o.end()) return dflt;
    std::size_t used = 0;
    T v{};
    if constexpr (std::is_same_v<T, int>) v = std::stoi(it->second, &used);
    else if constexpr (std::is_same_v<T, std::uint64_t>) v = std::stoull(it->second, &used);
    else v = std::stod(it->second, &used);
    if (used != it->second.size()) throw std::runtime_error("bad value for " + std::string(key));
    return v;
}

int usage() {
    std::fprintf(stderr,
                 "usage: mexp exp --in FILE [--family taylor-new] [--u double|single] [--report]\n"
                 "       mexp theta [--family taylor] [--u double|single]\n"
                 "       mexp staircase [--family F] [--u U] [--norm-min X] [--norm-max Y] [--points K] [--out F]\n"
                 "       mexp sweep [--kinds a,b] [--families f,g] [--n N] [--count C] [--seed S] [--u U]\n"
                 "                  [--norm-min X] [--norm-max Y] [--out F]\n");
    return 2;
}

}  // namespace

int main(int argc, char** argv) {
    if (argc < 2) return usage();
    const std::string cmd = argv[1];
    try {
        if (cmd == "exp") {
            auto o = parse_opts(argc, argv, 2,
                                {{"--in", true}, {"--family", true}, {"--u", true}, {"--report", false}});
            if (!o.count("--in")) throw std::runtime_error("--in is required");
            std::ifstream in(o["--in"]);
            if (!in) throw std::runtime_error("cannot open " + o["--in"]);
            const mexp::DenseMatrix a = mexp::parse_matrix(in);
            const auto rep = mexp::expm(a, parse_u(o.count("--u") ? o["--u"] : "double"),
                                        parse_family_or_throw(o.count("--family") ? o["--family"]
                                                                                   : "taylor-new"));
            std::cout << mexp::format_matrix(rep.result);
            if (o.count("--report"))
                std::cerr << mexp::family_name(rep.family) << ' ' << rep.degree << ' ' << rep.s
                          << ' ' << mexp::shortest_double(rep.product_cost()) << ' '
                          << mexp::shortest_double(rep.norm_in) << '\n';
        } else if (cmd == "theta") {
            auto o = parse_opts(argc, argv, 2, {{"--family", true}, {"--u", true}});
            const std::string u = o.count("--u") ? o["--u"] : "double";
            const auto& table = mexp::selection_table(
                parse_family_or_throw(o.count("--family") ? o["--family"] : "taylor"), parse_u(u));
            std::printf("# family %s, u = %s\n# degree  pi  theta\n", mexp::family_name(table.family),
                        u.c_str());
            for (const auto& e : table.entries)
                std::printf("%6d %4d  %.2e\n", e.degree, e.products, e.theta);
        } else if (cmd == "staircase") {
            auto o = parse_opts(argc, argv, 2,
                                {{"--family", true}, {"--u", true}, {"--norm-min", true},
                                 {"--norm-max", true}, {"--points", true}, {"--out", true}});
            const auto rows = mexp::cost_staircase(
                parse_family_or_throw(o.count("--family") ? o["--family"] : "taylor-new"),
                parse_u(o.count("--u") ? o["--u"] : "double"),
                mexp::log_grid(num(o, "--norm-min", 1e-8), num(o, "--norm-max", 64.0),
                               num(o, "--points", 257)));
            write_text(mexp::staircase_csv(rows), o);
        } else if (cmd == "sweep") {
            auto o = parse_opts(argc, argv, 2,
                                {{"--kinds", true}, {"--families", true}, {"--n", true},
                                 {"--count", true}, {"--seed", true}, {"--u", true},
                                 {"--norm-min", true}, {"--norm-max", true}, {"--out", true}});
            std::vector<mexp::GalleryKind> kinds;
            if (!o.count("--kinds") || o["--kinds"].empty()) {
                kinds.assign(mexp::kAllGalleryKinds.begin(), mexp::kAllGalleryKinds.end());
            } else {
                for (const auto& name : split_list(o["--kinds"])) {
                    mexp::GalleryKind k;
                    if (!mexp::parse_gallery_kind(name, k))
                        throw std::runtime_error("unknown gallery kind '" + name + "'");
                    kinds.push_back(k);
                }
            }
            std::vector<mexp::Family> families;
            if (!o.count("--families") || o["--families"].empty())
                families = {mexp::Family::TaylorNew, mexp::Family::TaylorPS, mexp::Family::PadeDiagonal};
            else
                for (const auto& name : split_list(o["--families"]))
                    families.push_back(parse_family_or_throw(name));
            const int n = num(o, "--n", 30), count = num(o, "--count", 200);
            const std::uint64_t seed = num<std::uint64_t>(o, "--seed", 0);
            const double lo = num(o, "--norm-min", 1e-3), hi = num(o, "--norm-max", 1e2);
            if (kinds.empty() || families.empty() || count < 1)
                throw std::runtime_error("sweep needs kinds, families and a count");
            // target norms log-uniform in [norm-min, norm-max] from the base
            // seed, matrix seeds from the base seed and the index
            // (mexp_cli.cpp:146-158)
            std::mt19937_64 rng(seed ^ 0xda3e39cb94b95bdbULL);
            std::vector<mexp::GallerySpec> specs(count);
            const double llo = std::log(lo), lhi = std::log(hi);
            for (int i = 0; i < count; ++i) {
                specs[i].kind = kinds[i % kinds.size()];
                specs[i].n = n;
                specs[i].seed = seed * 1000003ULL + std::uint64_t(i);
                const double f = 0.5 * (mexp::uniform_pm1(rng) + 1.0);
                specs[i].target_norm = std::exp(llo + f * (lhi - llo));
            }
            write_text(mexp::sweep_csv(mexp::error_sweep(specs, families, parse_u(o.count("--u") ? o["--u"] : "double"))), o);
        } else {
            return usage();
        }
    } catch (const std::exception& e) {
        std::cerr << "error: " << e.what() << '\n';
        return 1;
    }
    return 0;
}
