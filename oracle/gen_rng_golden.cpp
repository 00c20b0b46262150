// Emits golden vectors from the C++ standard library the reference uses for its
// generators (problems.cpp:65-96: std::mt19937_64 + hand-rolled Box-Muller;
// tests/oracles.hpp:39-46: std::uniform_real_distribution(-1,1)). Used to pin the
// oracle's C restatement of both. Built and run by tests/golden/make_golden.py.
#include <cmath>
#include <cstdio>
#include <random>

static double uniform_open_closed(std::mt19937_64& gen) {
    return (static_cast<double>(gen() >> 11) + 1.0) * 0x1.0p-53;
}

int main() {
    std::printf("{\n");
    {   // raw engine output
        std::mt19937_64 g(1234);
        std::printf("\"mt64_1234\": [");
        for (int i = 0; i < 8; ++i) std::printf("%s\"%llu\"", i ? ", " : "", (unsigned long long)g());
        std::printf("],\n");
    }
    {   // random_rhs(rows=7, s=1, seed=1234) Box-Muller with spare
        std::mt19937_64 gen(1234);
        double spare = 0.0;
        bool have = false;
        std::printf("\"random_rhs_7_1234\": [");
        for (int i = 0; i < 7; ++i) {
            double v;
            if (have) { v = spare; have = false; }
            else {
                const double u1 = uniform_open_closed(gen), u2 = uniform_open_closed(gen);
                const double radius = std::sqrt(-2.0 * std::log(u1));
                const double angle = 2.0 * M_PI * u2;
                v = radius * std::cos(angle);
                spare = radius * std::sin(angle);
                have = true;
            }
            std::printf("%s%.17g", i ? ", " : "", v);
        }
        std::printf("],\n");
    }
    {   // oracles::random_dense(rows=5, cols=2, seed=7)
        std::mt19937_64 gen(7);
        std::uniform_real_distribution<double> dist(-1.0, 1.0);
        std::printf("\"random_dense_5x2_7\": [");
        for (int i = 0; i < 10; ++i) std::printf("%s%.17g", i ? ", " : "", dist(gen));
        std::printf("]\n");
    }
    std::printf("}\n");
    return 0;
}
