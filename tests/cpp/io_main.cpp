// DTEN / TRNG exchange through the C++ facade (host only, no GPU): reads a DTEN and a TRNG written
// by the Python side, writes them back, and reports the errors the readers raise on bad input.
//   io_main <in.dten> <in.trng> <out.dten> <out.trng> <bad-file>...
#include <cstdio>

#include "tenring_b200.hpp"

using namespace tenring::b200;

int main(int argc, char** argv) {
    if (argc < 5) return 2;
    DenseTensor t = read_dten(std::string(argv[1]));
    TRFactors f = read_trng(std::string(argv[2]));
    write_dten(std::string(argv[3]), t);
    write_trng(std::string(argv[4]), f);
    std::printf("dten order %lld size %lld\n", (long long)t.order(), (long long)t.size());
    std::printf("trng cores %lld\n", (long long)f.order());
    for (int i = 5; i < argc; ++i) {
        try {
            (void)read_dten(std::string(argv[i]));
            std::printf("bad %d: accepted\n", i - 5);
        } catch (const format_error& e) {
            std::printf("bad %d: format_error: %s\n", i - 5, e.what());
        }
    }
    return 0;
}
