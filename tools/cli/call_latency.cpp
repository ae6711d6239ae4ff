// Per-call latency of the C++ drop-in mexp::expm (the reference's own entry
// point, expm.hpp:37) on one host matrix, timed from native code: what a C++
// caller of the reference sees after switching to this library.
//
//   bin/call_latency <matrix.bin: n*n little-endian doubles> <n> [calls]
// prints {"calls": K, "us_per_call": T, "degree": m, "s": s}
#include <chrono>
#include <cstdio>
#include <cstdlib>
#include <vector>

#include "mexp/expm.hpp"

int main(int argc, char** argv) {
    if (argc < 3) {
        std::fprintf(stderr, "usage: %s matrix.bin n [calls]\n", argv[0]);
        return 2;
    }
    const int n = std::atoi(argv[2]);
    const int calls = argc > 3 ? std::atoi(argv[3]) : 1000;
    std::vector<double> data(size_t(n) * n);
    FILE* f = std::fopen(argv[1], "rb");
    if (!f || std::fread(data.data(), sizeof(double), data.size(), f) != data.size()) {
        std::fprintf(stderr, "cannot read %s\n", argv[1]);
        return 2;
    }
    std::fclose(f);
    const mexp::DenseMatrix a(n, data);
    mexp::ExpmReport r{};
    for (int i = 0; i < 20; ++i) r = mexp::expm(a, mexp::Accuracy::Double, mexp::Family::TaylorNew);
    const auto t0 = std::chrono::steady_clock::now();
    for (int i = 0; i < calls; ++i) r = mexp::expm(a, mexp::Accuracy::Double, mexp::Family::TaylorNew);
    const double us =
        std::chrono::duration<double, std::micro>(std::chrono::steady_clock::now() - t0).count() / calls;
    std::printf("{\"calls\": %d, \"us_per_call\": %.3f, \"degree\": %d, \"s\": %d}\n", calls, us, r.degree, r.s);
    return 0;
}
