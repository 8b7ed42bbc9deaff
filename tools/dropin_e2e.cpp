// tools/dropin_e2e.cpp -- the drop-in's end-to-end time with the reference's
// return type (bench.py `e2e_dropin`).
//
// Mirrors the Algorithm-2 per-orbit loop (pipeline.hpp:58-72): for one n,
// every characteristic map of idcm_orbits(n, 4) -> enumerate_wpm with the
// UBT cap -> std::vector<PureComplex> per map, through the C++ drop-in
// plseeds_b200::enumerate_orbits (include/plseeds_b200.hpp: one device
// launch for all maps, then the PureComplex vectors built on the host).
// Timed on the host around the call, after one warm-up; prints one JSON line.
//   usage: dropin_e2e N DEVICE REPS
#include <algorithm>
#include <chrono>
#include <cstdio>
#include <cstdlib>
#include <vector>

#include "plseeds_b200.hpp"

int main(int argc, char** argv) {
    const int n = argc > 1 ? std::atoi(argv[1]) : 5;
    const int dev = argc > 2 ? std::atoi(argv[2]) : 0;
    const int reps = argc > 3 ? std::max(1, std::atoi(argv[3])) : 7;
    try {
        long long wpms = 0, facets = 0;
        std::vector<double> ms;
        for (int r = 0; r <= reps; ++r) {
            const auto t0 = std::chrono::steady_clock::now();
            const auto lists = plseeds_b200::enumerate_orbits(n, 4, dev);
            const double dt = std::chrono::duration<double, std::milli>(std::chrono::steady_clock::now() - t0).count();
            if (r == 0) continue;  // warm-up: module load, pools
            ms.push_back(dt);
            wpms = facets = 0;
            for (const auto& l : lists) {
                wpms += (long long)l.size();
                for (const auto& K : l) facets += (long long)K.facets.size();
            }
        }
        std::vector<double> s = ms;
        std::sort(s.begin(), s.end());
        std::printf("{\"call\": \"plseeds_b200::enumerate_orbits (C++ drop-in, std::vector<PureComplex> per map)\", "
                    "\"n\": %d, \"wpms\": %lld, \"facets\": %lld, \"wall_ms\": %.4f, \"min_ms\": %.4f, \"reps\": %d}\n",
                    n, wpms, facets, s[s.size() / 2], s[0], reps);
        return 0;
    } catch (const std::exception& e) {
        std::fprintf(stderr, "dropin_e2e: %s\n", e.what());
        return 1;
    }
}
