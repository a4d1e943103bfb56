// End-to-end timing of the C++ drop-in (liblamfast.so) exactly as a user of
// the reference API calls it: lamfast::assembleFast(setup) returning a
// StiffnessMatrix of std::vectors (pageable host memory).  Builds BASELINE
// C4 (or C2 / C3) through the reference's own types, times `reps` calls and
// prints one JSON line; bench.py reports it as e2e_dropin.
//   build/dropin_e2e [C4|C3|C2] [reps]
#include <algorithm>
#include <chrono>
#include <cmath>
#include <cstdio>
#include <cstring>
#include <memory>
#include <string>
#include <vector>

#include "lamfast/assembly.hpp"
#include "lamfast/fast.hpp"
#include "lamfast/geometry.hpp"
#include "lamfast/materials.hpp"
#include "lamfast/sparse.hpp"
#include "lamfast/splines.hpp"

using namespace lamfast;

static OrthotropicConstants orthotropic() { // BASELINE.json constants
    OrthotropicConstants c;
    c.E1 = 25.0;
    c.E2 = c.E3 = 1.0;
    c.G12 = c.G13 = 0.5;
    c.G23 = 0.2;
    c.nu12 = c.nu13 = c.nu23 = 0.25;
    return c;
}

static KnotVector c0Knots(int p, int m) { // every interior knot k/m repeated p times (C0)
    std::vector<double> k(static_cast<std::size_t>(p) + 1, 0.0);
    for (int i = 1; i < m; ++i)
        for (int r = 0; r < p; ++r)
            k.push_back(static_cast<double>(i) / m);
    k.insert(k.end(), static_cast<std::size_t>(p) + 1, 1.0);
    return KnotVector(p, k);
}

int main(int argc, char** argv) {
    const std::string cfg = argc > 1 ? argv[1] : "C4";
    const int reps = argc > 2 ? std::atoi(argv[2]) : 3;
    const double pi = 3.14159265358979323846;
    int p = 2, ex = 128, ey = 64, m = 128;
    double lx = 2.0, ly = 1.0, h = 0.2;
    std::vector<LayerSpec> layers;
    if (cfg == "C4") {
        const OrthotropicConstants soft = OrthotropicConstants::isotropic(0.5, 0.3);
        for (int k = 0; k < m; ++k)
            layers.push_back(k % 2 ? LayerSpec{soft, 0.0} : LayerSpec{orthotropic(), k % 4 == 0 ? 0.0 : 0.5 * pi});
    } else if (cfg == "C3") {
        p = 3, ex = ey = 64, m = 64, lx = ly = 1.0;
        const double cyc[4] = {0.0, 0.25 * pi, -0.25 * pi, 0.5 * pi};
        for (int k = 0; k < m; ++k)
            layers.push_back({orthotropic(), cyc[k % 4]});
    } else { // C2
        p = 2, ex = ey = 32, m = 16, lx = ly = 1.0, h = 0.1;
        for (int k = 0; k < m; ++k) {
            const int j = k < 8 ? k : 15 - k;
            layers.push_back({orthotropic(), j % 2 ? 0.5 * pi : 0.0});
        }
    }
    ProblemSetup setup{TensorProductSpace(KnotVector::uniform(p, ex), KnotVector::uniform(p, ey), c0Knots(2, m)),
                       ExtrudedGeometry(std::make_shared<PlanarRectangle>(lx, ly), Eigen::Vector3d(0, 0, h)),
                       Layup::equalLayers(layers)};
    std::vector<double> ms;
    long long nnz = 0;
    for (int r = 0; r < reps + 1; ++r) { // first call: warm-up
        const auto t0 = std::chrono::steady_clock::now();
        StiffnessMatrix K = assembleFast(setup);
        const auto t1 = std::chrono::steady_clock::now();
        if (r > 0)
            ms.push_back(std::chrono::duration<double, std::milli>(t1 - t0).count());
        nnz = static_cast<long long>(K.values().size());
    }
    // what the std::vector result costs by itself: allocating and
    // value-initialising arrays of the same sizes (single thread, as the
    // vectors' constructors do)
    const auto a0 = std::chrono::steady_clock::now();
    {
        std::vector<double> v(static_cast<std::size_t>(nnz));
        std::vector<int> c(static_cast<std::size_t>(nnz));
        std::vector<long long> rp(static_cast<std::size_t>(3LL * setup.space.numFunctions() + 1));
        if (v[nnz / 2] != 0.0 || c[nnz / 3] != 0 || rp[0] != 0)
            std::printf("?\n");
    }
    const auto a1 = std::chrono::steady_clock::now();
    double mean = 0.0;
    for (double x : ms)
        mean += x;
    mean /= static_cast<double>(ms.size());
    std::printf("{\"config\": \"%s\", \"nnz\": %lld, \"reps\": %d, \"ms_mean\": %.3f, \"ms_min\": %.3f, "
                "\"value\": %.6e, \"ms_vector_init\": %.3f}\n",
                cfg.c_str(), nnz, reps, mean, *std::min_element(ms.begin(), ms.end()),
                static_cast<double>(nnz) / (mean / 1e3),
                std::chrono::duration<double, std::milli>(a1 - a0).count());
    return 0;
}
