// Per-signal latency of the drop-in C++ path (include/dctplus_b200/dctplus.hpp):
// DctPlusPlan::forward(s, ws) on one host std::vector per call — what a caller
// of the reference's per-signal loop (bench.hpp:139-169) gets by switching
// headers.  Prints one JSON line per case: median / p10 / p90 microseconds.
#include <algorithm>
#include <chrono>
#include <cstdio>
#include <random>
#include <vector>

#include "dctplus_b200/dctplus.hpp"

using namespace dctplus_b200;

static void run(const char* name, std::size_t n, const RankOneUpdate& u) {
    const DctPlusPlan plan(n, u, 1e-12);
    DctPlusWorkspace ws = plan.make_workspace();
    std::mt19937_64 g(7);
    std::normal_distribution<double> nd;
    std::vector<double> s(n);
    for (auto& v : s) v = nd(g);
    for (int i = 0; i < 200; ++i) plan.forward(s, ws);
    std::vector<double> us;
    for (int i = 0; i < 3000; ++i) {
        const auto t0 = std::chrono::steady_clock::now();
        plan.forward(s, ws);
        const auto t1 = std::chrono::steady_clock::now();
        us.push_back(std::chrono::duration<double, std::micro>(t1 - t0).count());
    }
    std::sort(us.begin(), us.end());
    std::printf("{\"case\": \"%s\", \"n\": %zu, \"median_us\": %.2f, \"p10_us\": %.2f, \"p90_us\": %.2f}\n", name, n,
                us[us.size() / 2], us[us.size() / 10], us[us.size() * 9 / 10]);
    std::fflush(stdout);
}

int main() {
    run("C1 n=64 self_loop(1,0.5)", 64, RankOneUpdate::self_loop(1, 0.5));
    run("C2 n=256 edge_delta(128,129,-0.7)", 256, RankOneUpdate::edge_delta(128, 129, -0.7));
    run("C3 n=1024 edge_delta(1,1024,1.0)", 1024, RankOneUpdate::edge_delta(1, 1024, 1.0));
    return 0;
}
