// `mexp` command line over the B200 drop-in:
// the reference CLI's `exp` and `theta` subcommands (proj/tools/mexp_cli.cpp:
// 53-109) with the same arguments, output format and exit codes, computing on
// the GPU through include/mexp/expm.hpp. The reference's `staircase` and
// `sweep` subcommands (paper-figure CSVs over Pade/PS/gallery) are not on the
// B200 path and are rejected.
//
//   mexp exp --in A.txt [--family taylor-new] [--u double|single] [--report]
//   mexp theta [--family taylor] [--u double|single]
#include <cstdio>
#include <cstring>
#include <fstream>
#include <iostream>
#include <map>
#include <stdexcept>
#include <string>

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

int usage() {
    std::fprintf(stderr,
                 "usage: mexp exp --in FILE [--family taylor-new] [--u double|single] [--report]\n"
                 "       mexp theta [--family taylor] [--u double|single]\n");
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
        } else if (cmd == "staircase" || cmd == "sweep") {
            throw std::runtime_error(cmd + " is not on the B200 path (reference-only subcommand)");
        } else {
            return usage();
        }
    } catch (const std::exception& e) {
        std::cerr << "error: " << e.what() << '\n';
        return 1;
    }
    return 0;
}
