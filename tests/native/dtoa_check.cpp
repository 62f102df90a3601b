// CPU check of the device JSON number formatter (csrc/json_emit.cuh, compiled
// here as host code) against nlohmann::json's serializer: json(x).dump() for
// random doubles across every binade, integers, halfway/boundary cases.
//   dtoa_check <count> <seed>   -> prints "ok <count>" or the first mismatch
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <random>
#include <string>

#include "json.hpp"
#include "json_emit.cuh"

static bool check(double x, long long& bad) {
    nlohmann::json j = x;
    const std::string ref = j.dump();
    cg::json::Out o{nullptr, 0};
    char buf[64];
    o.buf = buf;
    o.dbl(x);
    const std::string got(buf, (size_t)o.n);
    if (got != ref) {
        if (bad++ < 5) std::printf("mismatch %.17g: got %s ref %s\n", x, got.c_str(), ref.c_str());
        return false;
    }
    return true;
}

int main(int argc, char** argv) {
    const long long count = argc > 1 ? std::atoll(argv[1]) : 1000000;
    std::mt19937_64 g(argc > 2 ? std::strtoull(argv[2], nullptr, 10) : 1);
    long long bad = 0;
    std::uniform_real_distribution<double> U(0, 1);
    for (long long i = 0; i < count; ++i) {
        double x;
        switch (i % 6) {
            case 0: {  // random bit patterns (all binades, subnormals, NaN/inf -> null)
                uint64_t b = g();
                std::memcpy(&x, &b, 8);
                break;
            }
            case 1: x = U(g) * 100.0; break;                       // scores, thresholds
            case 2: x = (double)(g() % 100000); break;              // integral tokens
            case 3: x = std::ldexp(U(g) + 0.5, (int)(g() % 200) - 100); break;
            case 4: x = std::nextafter(std::pow(10.0, (int)(g() % 40) - 20), (g() & 1) ? 0.0 : 1e300); break;
            default: x = U(g) * std::pow(10.0, (int)(g() % 30) - 15); break;
        }
        check(x, bad);
        check(-x, bad);
    }
    const double special[] = {0.0, -0.0, 1e15, 1e16, 123456789012345.0, 1234567890123456.0, 0.0001, 0.00001,
                              5e-324, 2.2250738585072014e-308, 1.7976931348623157e308, 0.1, 0.2, 0.3, 1.0 / 3};
    for (double x : special) check(x, bad);
    if (bad) {
        std::printf("FAIL %lld\n", bad);
        return 1;
    }
    std::printf("ok %lld\n", count);
    return 0;
}
