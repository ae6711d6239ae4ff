// Test helper: prints mexp::gallery(kind, n, seed, target_norm) (the drop-in's
// host gallery) as hex floats, one matrix per line, for the specs given as
// argument quadruples; "error" when the drop-in throws.
#include <cstdio>
#include <cstdlib>
#include <exception>

#include "mexp/gallery.hpp"

int main(int argc, char** argv) {
    for (int a = 1; a + 3 < argc; a += 4) {
        mexp::GallerySpec spec;
        spec.kind = mexp::kAllGalleryKinds[std::atoi(argv[a])];
        spec.n = std::atoi(argv[a + 1]);
        spec.seed = std::strtoull(argv[a + 2], nullptr, 10);
        spec.target_norm = std::strtod(argv[a + 3], nullptr);
        try {
            const auto m = mexp::gallery(spec);
            for (int e = 0; e < spec.n * spec.n; ++e) std::printf(e ? " %a" : "%a", m.data()[e]);
            std::printf("\n");
        } catch (const std::exception&) {
            std::printf("error\n");
        }
    }
    return 0;
}
