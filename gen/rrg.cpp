// rrg.cpp -- deterministic synthetic random-geometric-graph (RRG) generator.
//
// Input generator shared by the oracle side and the CUDA side (through
// Python); it holds NONE of the method's arithmetic (no g, no policy, no
// promising test).  It plays the role of PI-RRT#'s exploration phase
// ("random sampling and extension"), which is out of the
// hot path: it emits points, edge costs (Euclidean, cached once per edge as in
// PAPER.md:310-314) and the heuristic h (Euclidean distance to x_goal,
// admissible).
//
// Recipe:
//   * vertex 0 = x_init = (0.1,...,0.1), vertex 1 = x_goal = (0.9,...,0.9)
//     (PAPER.md:198);
//   * n_boxes axis-aligned boxes with per-axis side U[side_lo, side_hi] and
//     lower corner U[0, 1-side]; a box containing x_init or x_goal is redrawn;
//   * vertices i >= 2 uniform in [0,1]^d, redrawn while inside a box;
//   * vertex i >= 2 connects to every earlier j < i with |x_i - x_j| <=
//     r(i+1), r(m) = gamma (ln m / m)^(1/d), when the segment misses every
//     box (exact slab test).  Edge cost = |x_i - x_j| in fp64.
//   * RNG: SplitMix64 stream; output independent of the thread count.
#include <algorithm>
#include <cmath>
#include <cstdint>
#include <cstring>
#include <vector>
#include <atomic>
#include <thread>

namespace {

struct SplitMix64 {
    uint64_t s;
    explicit SplitMix64(uint64_t seed) : s(seed) {}
    uint64_t next() {
        uint64_t z = (s += 0x9E3779B97F4A7C15ull);
        z = (z ^ (z >> 30)) * 0xBF58476D1CE4E5B9ull;
        z = (z ^ (z >> 27)) * 0x94D049BB133111EBull;
        return z ^ (z >> 31);
    }
    double uniform() { return (double)(next() >> 11) * (1.0 / 9007199254740992.0); }
};

struct Gen {
    int d = 2;
    int64_t n = 0;
    double gamma = 1.0;
    int n_boxes = 0;
    std::vector<double> pts;    // n * d
    std::vector<double> boxes;  // n_boxes * 2d: lo[d], hi[d]
    std::vector<double> h;      // n
    std::vector<int64_t> off;   // n + 1
    std::vector<int32_t> idx;   // earlier neighbour j of vertex i
    std::vector<double> cost;   // |x_i - x_j|
    int64_t n_isolated = 0;
    int64_t n_candidates = 0;
};

double dist(const double* a, const double* b, int d) {
    double s = 0.0;
    for (int k = 0; k < d; ++k) {
        double t = a[k] - b[k];
        s += t * t;
    }
    return std::sqrt(s);
}

bool in_box(const double* p, const double* box, int d) {
    for (int k = 0; k < d; ++k)
        if (p[k] < box[k] || p[k] > box[d + k]) return false;
    return true;
}

// segment p->q intersects closed box (slab test)
bool seg_hits_box(const double* p, const double* q, const double* box, int d) {
    double t0 = 0.0, t1 = 1.0;
    for (int k = 0; k < d; ++k) {
        double lo = box[k], hi = box[d + k];
        double dk = q[k] - p[k];
        if (dk == 0.0) {
            if (p[k] < lo || p[k] > hi) return false;
            continue;
        }
        double ta = (lo - p[k]) / dk, tb = (hi - p[k]) / dk;
        if (ta > tb) std::swap(ta, tb);
        if (ta > t0) t0 = ta;
        if (tb < t1) t1 = tb;
        if (t0 > t1) return false;
    }
    return true;
}

// dynamic-chunk parallel for over [lo, hi) with std::thread (results are
// written per index, so the output does not depend on the thread count)
template <class F>
void parallel_for(int64_t lo, int64_t hi, int threads, F&& f) {
    if (threads <= 0) threads = (int)std::thread::hardware_concurrency();
    if (threads < 1) threads = 1;
    std::atomic<int64_t> next(lo);
    const int64_t chunk = 256;
    auto worker = [&]() {
        for (;;) {
            int64_t a = next.fetch_add(chunk);
            if (a >= hi) break;
            int64_t b = std::min(hi, a + chunk);
            for (int64_t i = a; i < b; ++i) f(i);
        }
    };
    std::vector<std::thread> pool;
    for (int t = 1; t < threads; ++t) pool.emplace_back(worker);
    worker();
    for (auto& t : pool) t.join();
}

double radius(double gamma, int64_t m, int d) {
    if (m < 2) return 1e300;
    double lm = std::log((double)m);
    return gamma * std::pow(lm / (double)m, 1.0 / d);
}

}  // namespace

extern "C" {

void* gen_rrg(int d, int64_t n, double gamma, int n_boxes, double side_lo,
              double side_hi, uint64_t seed, int threads) {
    if (d < 1 || d > 16 || n < 2) return nullptr;
    Gen* G = new Gen();
    G->d = d; G->n = n; G->gamma = gamma; G->n_boxes = n_boxes;
    SplitMix64 rng(seed);
    std::vector<double> xi(d, 0.1), xg(d, 0.9);
    // boxes
    G->boxes.resize((size_t)n_boxes * 2 * d);
    for (int bI = 0; bI < n_boxes; ++bI) {
        double* box = &G->boxes[(size_t)bI * 2 * d];
        for (int tries = 0; tries < 100000; ++tries) {
            for (int k = 0; k < d; ++k) {
                double side = side_lo + (side_hi - side_lo) * rng.uniform();
                double lo = (1.0 - side) * rng.uniform();
                box[k] = lo; box[d + k] = lo + side;
            }
            if (!in_box(xi.data(), box, d) && !in_box(xg.data(), box, d)) break;
        }
    }
    // points
    G->pts.resize((size_t)n * d);
    for (int k = 0; k < d; ++k) { G->pts[k] = xi[k]; G->pts[d + k] = xg[k]; }
    for (int64_t i = 2; i < n; ++i) {
        double* p = &G->pts[(size_t)i * d];
        for (int tries = 0; ; ++tries) {
            for (int k = 0; k < d; ++k) p[k] = rng.uniform();
            bool inside = false;
            for (int bI = 0; bI < n_boxes && !inside; ++bI)
                inside = in_box(p, &G->boxes[(size_t)bI * 2 * d], d);
            if (!inside || tries > 1000000) break;
        }
    }
    G->h.resize(n);
    for (int64_t i = 0; i < n; ++i) G->h[i] = dist(&G->pts[(size_t)i * d], xg.data(), d);
    G->h[1] = 0.0;

    // uniform grid with cell side >= r(n) (the smallest radius used)
    double rmin = radius(gamma, n, d);
    int m = (int)std::floor(1.0 / rmin);
    if (m < 1) m = 1;
    // keep the cell count bounded
    while (m > 1 && std::pow((double)m, d) > 4.0 * (double)n) --m;
    int64_t ncell = 1;
    for (int k = 0; k < d; ++k) ncell *= m;
    const double side = 1.0 / m;
    auto cell_coord = [&](double x) {
        int c = (int)std::floor(x * m);
        return c < 0 ? 0 : (c >= m ? m - 1 : c);
    };
    std::vector<int64_t> cell_of(n);
    for (int64_t i = 0; i < n; ++i) {
        int64_t c = 0;
        for (int k = 0; k < d; ++k) c = c * m + cell_coord(G->pts[(size_t)i * d + k]);
        cell_of[i] = c;
    }
    std::vector<int64_t> cstart(ncell + 1, 0);
    for (int64_t i = 0; i < n; ++i) cstart[cell_of[i] + 1]++;
    for (int64_t c = 0; c < ncell; ++c) cstart[c + 1] += cstart[c];
    std::vector<int32_t> cpts(n);
    {
        std::vector<int64_t> cur(cstart.begin(), cstart.end() - 1);
        for (int64_t i = 0; i < n; ++i) cpts[cur[cell_of[i]]++] = (int32_t)i;  // ascending id per cell
    }
    // coordinates in cell order, so that scanning a cell reads contiguous memory
    std::vector<double> cpos((size_t)n * d);
    for (int64_t t = 0; t < n; ++t)
        std::memcpy(&cpos[(size_t)t * d], &G->pts[(size_t)cpts[t] * d], sizeof(double) * d);

    std::vector<std::vector<std::pair<int32_t, double>>> nb(n);
    std::vector<int64_t> cand_count(n, 0);
    parallel_for(2, n, threads, [&](int64_t i) {
        const double* p = &G->pts[(size_t)i * d];
        const double R = radius(gamma, i + 1, d);
        auto& out = nb[i];
        int64_t cand = 0;
        const double R2 = R * R;
        auto consider_at = [&](int32_t j, const double* q) {
            ++cand;
            // squared distance with early exit; same summation order as dist()
            double s2 = 0.0;
            for (int k = 0; k < d; ++k) {
                double t = p[k] - q[k];
                s2 += t * t;
                if (s2 > R2 * (1.0 + 1e-12)) return;
            }
            double dd = std::sqrt(s2);
            if (dd > R) return;
            for (int bI = 0; bI < n_boxes; ++bI)
                if (seg_hits_box(q, p, &G->boxes[(size_t)bI * 2 * d], d)) return;
            out.push_back({j, dd});
        };
        auto consider = [&](int32_t j) { consider_at(j, &G->pts[(size_t)j * d]); };
        int kr = (int)std::ceil(R / side);
        double cells_scanned = std::pow(2.0 * kr + 1.0, d);
        if (kr >= m || cells_scanned * (1.0 + (double)n / ncell) > (double)i) {
            for (int32_t j = 0; j < i; ++j) consider(j);
        } else {
            int lo[16], hi[16], cc[16];
            for (int k = 0; k < d; ++k) {
                int c = cell_coord(p[k]);
                lo[k] = std::max(0, c - kr);
                hi[k] = std::min(m - 1, c + kr);
                cc[k] = lo[k];
            }
            for (;;) {
                int64_t c = 0;
                for (int k = 0; k < d; ++k) c = c * m + cc[k];
                for (int64_t t = cstart[c]; t < cstart[c + 1]; ++t) {
                    int32_t j = cpts[t];
                    if (j >= i) break;  // ascending ids in a cell
                    consider_at(j, &cpos[(size_t)t * d]);
                }
                int k = d - 1;
                while (k >= 0 && cc[k] == hi[k]) { cc[k] = lo[k]; --k; }
                if (k < 0) break;
                ++cc[k];
            }
            std::sort(out.begin(), out.end(),
                      [](const std::pair<int32_t, double>& a, const std::pair<int32_t, double>& b) {
                          return a.first < b.first;
                      });
        }
        cand_count[i] = cand;
    });
    G->off.assign(n + 1, 0);
    for (int64_t i = 0; i < n; ++i) {
        G->off[i + 1] = G->off[i] + (int64_t)nb[i].size();
        if (i >= 2 && nb[i].empty()) G->n_isolated++;
        G->n_candidates += cand_count[i];
    }
    G->idx.resize(G->off[n]);
    G->cost.resize(G->off[n]);
    parallel_for(0, n, threads, [&](int64_t i) {
        int64_t o = G->off[i];
        for (auto& jc : nb[i]) { G->idx[o] = jc.first; G->cost[o] = jc.second; ++o; }
        std::vector<std::pair<int32_t, double>>().swap(nb[i]);
    });
    return G;
}

// Only the sampling half of gen_rrg (same RNG stream: the same boxes and
// points), for a planner that builds its edges on the device
// (pirrt_extend_batch).  boxes [n_boxes][2][d], pts [n][d].
int gen_points(int d, int64_t n, int n_boxes, double side_lo, double side_hi, uint64_t seed,
               double* boxes, double* pts) {
    if (d < 1 || d > 16 || n < 2) return -1;
    SplitMix64 rng(seed);
    std::vector<double> xi(d, 0.1), xg(d, 0.9);
    for (int bI = 0; bI < n_boxes; ++bI) {
        double* box = &boxes[(size_t)bI * 2 * d];
        for (int tries = 0; tries < 100000; ++tries) {
            for (int k = 0; k < d; ++k) {
                double side = side_lo + (side_hi - side_lo) * rng.uniform();
                double lo = (1.0 - side) * rng.uniform();
                box[k] = lo; box[d + k] = lo + side;
            }
            if (!in_box(xi.data(), box, d) && !in_box(xg.data(), box, d)) break;
        }
    }
    for (int k = 0; k < d; ++k) { pts[k] = xi[k]; pts[d + k] = xg[k]; }
    for (int64_t i = 2; i < n; ++i) {
        double* p = &pts[(size_t)i * d];
        for (int tries = 0; ; ++tries) {
            for (int k = 0; k < d; ++k) p[k] = rng.uniform();
            bool inside = false;
            for (int bI = 0; bI < n_boxes && !inside; ++bI) inside = in_box(p, &boxes[(size_t)bI * 2 * d], d);
            if (!inside || tries > 1000000) break;
        }
    }
    return 0;
}

void gen_sizes(void* h, int64_t* n, int64_t* n_pairs, int64_t* n_isolated,
               int64_t* n_candidates) {
    Gen* G = (Gen*)h;
    *n = G->n;
    *n_pairs = G->off[G->n];
    *n_isolated = G->n_isolated;
    *n_candidates = G->n_candidates;
}

void gen_copy(void* h, double* pts, double* boxes, double* hv, int64_t* off,
              int32_t* idx, double* cost) {
    Gen* G = (Gen*)h;
    if (pts) std::memcpy(pts, G->pts.data(), G->pts.size() * sizeof(double));
    if (boxes) std::memcpy(boxes, G->boxes.data(), G->boxes.size() * sizeof(double));
    if (hv) std::memcpy(hv, G->h.data(), G->h.size() * sizeof(double));
    if (off) std::memcpy(off, G->off.data(), G->off.size() * sizeof(int64_t));
    if (idx) std::memcpy(idx, G->idx.data(), G->idx.size() * sizeof(int32_t));
    if (cost) std::memcpy(cost, G->cost.data(), G->cost.size() * sizeof(double));
}

void gen_free(void* h) { delete (Gen*)h; }

}  // extern "C"
