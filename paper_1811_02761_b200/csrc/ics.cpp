// Initial conditions: bit-identical, multithreaded restatement of gravitree's
// samplers (models.cpp, rng.hpp) so benchmark inputs equal the reference's
// sample_model(name, n, seed) bit for bit (SURVEY §8d synthetic inputs).
//
// The reference draws from one counter-based stream per component
// (rng.hpp:11-64).  For the Jeans spheres (NFW, Hernquist; models.cpp:
// 207-240) and the exponential disk (models.cpp:307-369) every particle
// consumes a fixed pattern of counters: radius/phi/z uniforms (3) plus three
// Box-Muller normals whose spare carries across particles, i.e. 12 counters
// per PAIR of particles.  Particle 2p therefore starts at counter 12p and the
// stream can be evaluated in parallel.  Plummer velocities are rejection
// sampled (variable consumption) and stay sequential.  Compiled with
// -ffp-contract=off and no -march, like the reference, so libm calls and
// arithmetic round identically.
#include <algorithm>
#include <cmath>
#include <cstdint>
#include <cstring>
#include <functional>
#include <stdexcept>
#include <string>
#include <thread>
#include <vector>

namespace {

constexpr double kPi = 3.14159265358979323846;
constexpr double kTwoPi = 2.0 * kPi;

inline uint64_t mix(uint64_t seed, uint64_t stream, uint64_t counter) {  // rng.hpp:38-52
    uint64_t z = seed + 0x9e3779b97f4a7c15ULL * (stream + 1);
    z ^= z >> 30;
    z *= 0xbf58476d1ce4e5b9ULL;
    z += counter * 0x9e3779b97f4a7c15ULL;
    z ^= z >> 27;
    z *= 0x94d049bb133111ebULL;
    z ^= z >> 31;
    z *= 0xd6e8feb86659fd93ULL;
    z ^= z >> 32;
    return z;
}

// Stream positioned at an arbitrary counter.
struct Stream {
    uint64_t seed, stream, ctr;
    double unit() { return static_cast<double>(mix(seed, stream, ctr++) >> 11) * 0x1.0p-53; }
    double pos() { return 1.0 - unit(); }
    double range(double lo, double hi) { return lo + (hi - lo) * unit(); }
    // one Box-Muller pair (rng.hpp:26-37): first = r cos a, second (spare) = r sin a
    void pair(double& c, double& s) {
        const double u1 = pos();
        const double u2 = unit();
        const double r = std::sqrt(-2.0 * std::log(u1));
        const double a = 6.283185307179586476925286766559 * u2;
        s = r * std::sin(a);
        c = r * std::cos(a);
    }
};

struct V3 {
    double x, y, z;
};

inline V3 direction(Stream& s) {  // models.cpp:18-23
    const double ct = s.range(-1.0, 1.0);
    const double st = std::sqrt(std::max(0.0, 1.0 - ct * ct));
    const double ph = s.range(0.0, kTwoPi);
    return {st * std::cos(ph), st * std::sin(ph), ct};
}

double bisect(const std::function<double(double)>& fn, double target, double lo, double hi) {  // models.cpp:68-78
    for (int it = 0; it < 80; ++it) {
        const double mid = 0.5 * (lo + hi);
        if (fn(mid) < target)
            lo = mid;
        else
            hi = mid;
    }
    return 0.5 * (lo + hi);
}

double nfw_mu(double x) { return std::log1p(x) - x / (1.0 + x); }
double hern_frac(double r, double a) {
    const double q = r / (r + a);
    return q * q;
}
double plum_frac(double r, double a) {
    const double r2 = r * r;
    return r2 * r / std::pow(r2 + a * a, 1.5);
}

enum Kind { kPlummer, kHernquist, kNfw, kDisk };
struct Comp {
    Kind kind;
    double mass, scale, height, q_floor;
    double cutoff() const { return 20.0 * scale; }
};

double comp_enclosed(const Comp& c, double r) {  // models.cpp:174-195
    const double rc = c.cutoff();
    const double rr = std::min(r, rc);
    switch (c.kind) {
        case kPlummer: return c.mass * plum_frac(rr, c.scale) / plum_frac(rc, c.scale);
        case kHernquist: return c.mass * hern_frac(rr, c.scale) / hern_frac(rc, c.scale);
        case kNfw: return c.mass * nfw_mu(rr / c.scale) / nfw_mu(rc / c.scale);
        case kDisk: {
            const double x = rr / c.scale, xc = rc / c.scale;
            const double f = 1.0 - (1.0 + x) * std::exp(-x);
            const double fc = 1.0 - (1.0 + xc) * std::exp(-xc);
            return c.mass * f / fc;
        }
    }
    return 0.0;
}

struct Catalog {
    std::vector<Comp> comps;
    double enclosed(double r) const {
        double m = 0.0;
        for (const Comp& c : comps) m += comp_enclosed(c, r);
        return m;
    }
    double vcirc(double R) const { return R <= 0.0 ? 0.0 : std::sqrt(1.0 * enclosed(R) / R); }
};

struct Jeans {  // models.cpp:27-66
    double ln_min, ln_max, inv_step;
    std::vector<double> s2;
    Jeans(const std::function<double(double)>& rho, const std::function<double(double)>& mtot, double r_min,
          double r_cut, int grid = 1024)
        : ln_min(std::log(r_min)), ln_max(std::log(r_cut)), inv_step(0.0), s2(grid, 0.0) {
        std::vector<double> r(grid), f(grid);
        const double step = (ln_max - ln_min) / (grid - 1);
        inv_step = 1.0 / step;
        for (int i = 0; i < grid; ++i) {
            r[i] = std::exp(ln_min + step * i);
            f[i] = rho(r[i]) * 1.0 * mtot(r[i]) / (r[i] * r[i]);
        }
        double tail = 0.0;
        for (int i = grid - 2; i >= 0; --i) {
            tail += 0.5 * (f[i] * r[i] + f[i + 1] * r[i + 1]) * step;
            const double rh = rho(r[i]);
            s2[i] = rh > 0.0 ? tail / rh : 0.0;
        }
    }
    double sigma(double radius) const {
        const double lr = std::log(std::max(radius, 1e-300));
        if (lr <= ln_min) return std::sqrt(s2.front());
        if (lr >= ln_max) return 0.0;
        const double t = (lr - ln_min) * inv_step;
        const auto i = static_cast<size_t>(t);
        const double w = t - static_cast<double>(i);
        return std::sqrt(std::max(0.0, s2[i] * (1.0 - w) + s2[i + 1] * w));
    }
};

template <typename F>
void parallel_pairs(size_t n, unsigned threads, F&& fn) {
    const size_t pairs = (n + 1) / 2;
    if (threads <= 1 || pairs < 4096) {
        fn(size_t(0), pairs);
        return;
    }
    std::vector<std::thread> pool;
    for (unsigned t = 0; t < threads; ++t)
        pool.emplace_back([&, t] { fn(pairs * t / threads, pairs * (t + 1) / threads); });
    for (auto& th : pool) th.join();
}

// fixed-pattern particle: 3 uniforms for geometry, then 3 normals (12 counters per pair)
struct Draw {
    double u[3];
    double nrm[3];
};
inline void draw_pair(Stream& s, Draw& a, Draw& b) {
    double A0, A1, B0, B1, C0, C1;
    a.u[0] = s.unit(), a.u[1] = s.unit(), a.u[2] = s.unit();
    s.pair(A0, A1);
    s.pair(B0, B1);
    a.nrm[0] = A0, a.nrm[1] = A1, a.nrm[2] = B0;
    b.u[0] = s.unit(), b.u[1] = s.unit(), b.u[2] = s.unit();
    s.pair(C0, C1);
    b.nrm[0] = B1, b.nrm[1] = C0, b.nrm[2] = C1;
}

void recentre(size_t n, double* vel) {  // models.cpp:205-212
    double vx = 0.0, vy = 0.0, vz = 0.0;
    for (size_t i = 0; i < n; ++i) vx += vel[3 * i], vy += vel[3 * i + 1], vz += vel[3 * i + 2];
    const double inv = 1.0 / static_cast<double>(n);
    vx *= inv, vy *= inv, vz *= inv;
    for (size_t i = 0; i < n; ++i) vel[3 * i] -= vx, vel[3 * i + 1] -= vy, vel[3 * i + 2] -= vz;
}

// Jeans sphere (models.cpp:218-240): positions by inverse CDF, isotropic Gaussian velocities
void jeans_sphere(size_t n, double mass, double scale, double r_cut, uint64_t seed, uint64_t stream,
                  const std::function<double(double)>& rho, const std::function<double(double)>& frac,
                  const std::function<double(double)>& mtot_in, const std::function<double(double)>& inverse_frac,
                  unsigned threads, double* m, double* pos, double* vel) {
    const double pm = mass / static_cast<double>(n);
    for (size_t i = 0; i < n; ++i) m[i] = pm;
    const double f_cut = frac(r_cut);
    std::function<double(double)> mtot = mtot_in;
    if (!mtot) mtot = [&](double r) { return mass * frac(std::min(r, r_cut)) / f_cut; };
    const Jeans jeans(rho, mtot, scale * 1e-4, r_cut);
    auto inverse = [&](double u) {
        const double target = u * f_cut;
        if (inverse_frac) return inverse_frac(target);
        return bisect(frac, target, 0.0, r_cut);
    };
    parallel_pairs(n, threads, [&](size_t p0, size_t p1) {
        Stream s{seed, stream, 12 * p0};
        for (size_t p = p0; p < p1; ++p) {
            Draw d[2];
            draw_pair(s, d[0], d[1]);
            for (int k = 0; k < 2; ++k) {
                const size_t i = 2 * p + k;
                if (i >= n) break;
                const double r = inverse(d[k].u[0]);
                const double ct = -1.0 + (1.0 - -1.0) * d[k].u[1];
                const double st = std::sqrt(std::max(0.0, 1.0 - ct * ct));
                const double ph = 0.0 + (kTwoPi - 0.0) * d[k].u[2];
                pos[3 * i] = st * std::cos(ph) * r;
                pos[3 * i + 1] = st * std::sin(ph) * r;
                pos[3 * i + 2] = ct * r;
                const double sg = jeans.sigma(r);
                vel[3 * i] = sg * d[k].nrm[0], vel[3 * i + 1] = sg * d[k].nrm[1], vel[3 * i + 2] = sg * d[k].nrm[2];
            }
        }
    });
    recentre(n, vel);
}

void hernquist(size_t n, double mass, double a, uint64_t seed, uint64_t stream, double r_cut,
               const std::function<double(double)>& mtot, unsigned threads, double* m, double* pos, double* vel) {
    auto rho = [a](double r) {
        const double x = std::max(r, 1e-12 * a) / a;
        return 1.0 / (x * std::pow(1.0 + x, 3.0));
    };
    auto frac = [a](double r) { return hern_frac(r, a); };
    auto inv = [a](double target) {
        const double q = std::sqrt(target);
        return a * q / (1.0 - q);
    };
    jeans_sphere(n, mass, a, r_cut, seed, stream, rho, frac, mtot, inv, threads, m, pos, vel);
}

void nfw(size_t n, double mass, double rs, double r_cut, uint64_t seed, uint64_t stream,
         const std::function<double(double)>& mtot, unsigned threads, double* m, double* pos, double* vel) {
    auto rho = [rs](double r) {
        const double x = std::max(r, 1e-12 * rs) / rs;
        return 1.0 / (x * (1.0 + x) * (1.0 + x));
    };
    auto frac = [rs](double r) { return nfw_mu(r / rs); };
    jeans_sphere(n, mass, rs, r_cut, seed, stream, rho, frac, mtot, nullptr, threads, m, pos, vel);
}

void plummer(size_t n, double mass, double a, uint64_t seed, uint64_t stream, double r_cut, double* m, double* pos,
             double* vel) {  // models.cpp:242-267, sequential (rejection sampling)
    const double pm = mass / static_cast<double>(n);
    for (size_t i = 0; i < n; ++i) m[i] = pm;
    Stream s{seed, stream, 0};
    const double f_cut = plum_frac(r_cut, a);
    for (size_t i = 0; i < n; ++i) {
        const double u = s.unit() * f_cut;
        const double u23 = std::cbrt(u) * std::cbrt(u);
        const double r = a * std::sqrt(u23 / (1.0 - u23));
        const V3 d = direction(s);
        pos[3 * i] = d.x * r, pos[3 * i + 1] = d.y * r, pos[3 * i + 2] = d.z * r;
        double q = 0.0;
        for (;;) {
            const double qt = s.unit();
            const double y = s.range(0.0, 0.1);
            const double o = 1.0 - qt * qt;
            if (y < qt * qt * o * o * o * std::sqrt(o)) {
                q = qt;
                break;
            }
        }
        const double v_esc = std::sqrt(2.0 * mass) / std::pow(r * r + a * a, 0.25);
        const V3 e = direction(s);
        const double sc = q * v_esc;
        vel[3 * i] = e.x * sc, vel[3 * i + 1] = e.y * sc, vel[3 * i + 2] = e.z * sc;
    }
    recentre(n, vel);
}

void disk(size_t n, double mass, double r_d, double z_d, uint64_t seed, const Catalog& prov, double q_floor,
          double r_cut, double z_cut, unsigned threads, double* m, double* pos, double* vel) {  // models.cpp:307-369
    if (r_cut <= 0.0) r_cut = 20.0 * r_d;
    if (z_cut <= 0.0) z_cut = 10.0 * z_d;
    if (!(q_floor > 0.0)) q_floor = 1.0;
    const double pm = mass / static_cast<double>(n);
    for (size_t i = 0; i < n; ++i) m[i] = pm;
    const double xc = r_cut / r_d;
    const double f_cut = 1.0 - (1.0 + xc) * std::exp(-xc);
    auto radial = [](double x) { return 1.0 - (1.0 + x) * std::exp(-x); };
    const int grid = 512;
    const double ln_min = std::log(r_d * 1e-3), ln_max = std::log(r_cut);
    const double step = (ln_max - ln_min) / (grid - 1);
    std::vector<double> rad(grid), om2(grid), sr(grid), sp(grid), sz(grid);
    const double sigma0 = mass / (kTwoPi * r_d * r_d * f_cut);
    for (int i = 0; i < grid; ++i) {
        rad[i] = std::exp(ln_min + step * i);
        const double vc = prov.vcirc(rad[i]);
        om2[i] = vc * vc / (rad[i] * rad[i]);
    }
    for (int i = 0; i < grid; ++i) {
        const int lo = std::max(0, i - 1), hi = std::min(grid - 1, i + 1);
        const double dln = step * (hi - lo);
        const double dw2 = (om2[hi] - om2[lo]) / dln;
        const double kappa = std::sqrt(std::max(om2[i], 4.0 * om2[i] + dw2));
        const double surface = sigma0 * std::exp(-rad[i] / r_d);
        sr[i] = 3.36 * surface * q_floor / kappa;
        sp[i] = sr[i] * kappa / (2.0 * std::sqrt(om2[i]));
        sz[i] = std::sqrt(kPi * surface * z_d);
    }
    auto lookup = [&](const std::vector<double>& tab, double R) {
        const double lr = std::log(std::max(R, rad.front()));
        if (lr >= ln_max) return tab.back();
        const double t = (lr - ln_min) / step;
        const auto i = static_cast<size_t>(t);
        const double w = t - static_cast<double>(i);
        return tab[i] * (1.0 - w) + tab[i + 1] * w;
    };
    const double z_range = std::tanh(z_cut / z_d);
    parallel_pairs(n, threads, [&](size_t p0, size_t p1) {
        Stream s{seed, 0, 12 * p0};
        for (size_t p = p0; p < p1; ++p) {
            Draw d[2];
            draw_pair(s, d[0], d[1]);
            for (int k = 0; k < 2; ++k) {
                const size_t i = 2 * p + k;
                if (i >= n) break;
                const double x = bisect(radial, d[k].u[0] * f_cut, 0.0, xc);
                const double R = x * r_d;
                const double ph = 0.0 + (kTwoPi - 0.0) * d[k].u[1];
                const double z = z_d * std::atanh(z_range * (-1.0 + (1.0 - -1.0) * d[k].u[2]));
                pos[3 * i] = R * std::cos(ph), pos[3 * i + 1] = R * std::sin(ph), pos[3 * i + 2] = z;
                const double v_r = lookup(sr, R) * d[k].nrm[0];
                const double v_phi = prov.vcirc(R) + lookup(sp, R) * d[k].nrm[1];
                const double v_z = lookup(sz, R) * d[k].nrm[2];
                vel[3 * i] = v_r * std::cos(ph) - v_phi * std::sin(ph);
                vel[3 * i + 1] = v_r * std::sin(ph) + v_phi * std::cos(ph);
                vel[3 * i + 2] = v_z;
            }
        }
    });
    recentre(n, vel);
}

Catalog m31() {  // models.cpp:107-136
    return Catalog{{{kNfw, 81.1, 7.63, 0.0, 0.0},
                    {kHernquist, 0.8, 9.0, 0.0, 0.0},
                    {kHernquist, 3.24, 0.61, 0.0, 0.0},
                    {kDisk, 3.66, 5.4, 0.6, 1.8}}};
}

std::vector<size_t> apportion(const Catalog& cat, size_t n_total) {  // models.cpp:371-389
    const size_t k = cat.comps.size();
    double total = 0.0;
    for (const Comp& c : cat.comps) total += c.mass;
    std::vector<size_t> counts(k);
    std::vector<std::pair<double, size_t>> rem(k);
    size_t assigned = 0;
    for (size_t c = 0; c < k; ++c) {
        const double share = static_cast<double>(n_total) * cat.comps[c].mass / total;
        counts[c] = static_cast<size_t>(share);
        rem[c] = {share - static_cast<double>(counts[c]), c};
        assigned += counts[c];
    }
    std::sort(rem.begin(), rem.end(), [](const auto& a, const auto& b) {
        if (a.first != b.first) return a.first > b.first;
        return a.second < b.second;
    });
    for (size_t i = 0; assigned < n_total; ++i, ++assigned) ++counts[rem[i % k].second];
    return counts;
}

void build_m31(size_t n_total, uint64_t seed, unsigned threads, double* m, double* pos, double* vel) {
    const Catalog cat = m31();
    if (n_total < cat.comps.size()) throw std::runtime_error("build_m31: not enough particles for every component");
    double total = 0.0;
    for (const Comp& c : cat.comps) total += c.mass;
    const std::vector<size_t> counts = apportion(cat, n_total);
    for (size_t c : counts)
        if (c == 0) throw std::runtime_error("build_m31: n_total too small to populate every component");
    const double pmass = total / static_cast<double>(n_total);
    std::function<double(double)> mtot = [&cat](double r) { return cat.enclosed(r); };
    size_t off = 0;
    for (size_t c = 0; c < cat.comps.size(); ++c) {
        const Comp& sp = cat.comps[c];
        const double cm = pmass * static_cast<double>(counts[c]);
        const uint64_t stream = 100 + c;
        double *mm = m + off, *pp = pos + 3 * off, *vv = vel + 3 * off;
        switch (sp.kind) {
            case kNfw: nfw(counts[c], cm, sp.scale, sp.cutoff(), seed, stream, mtot, threads, mm, pp, vv); break;
            case kHernquist:
                hernquist(counts[c], cm, sp.scale, seed, stream, sp.cutoff(), mtot, threads, mm, pp, vv);
                break;
            case kPlummer: plummer(counts[c], cm, sp.scale, seed, stream, sp.cutoff(), mm, pp, vv); break;
            case kDisk:
                disk(counts[c], cm, sp.scale, sp.height, mix(seed, stream, 0), cat, sp.q_floor, sp.cutoff(),
                     10.0 * sp.height, threads, mm, pp, vv);
                break;
        }
        off += counts[c];
    }
}

thread_local std::string g_ic_err;

}  // namespace

extern "C" {

const char* g2_ics_last_error(void) { return g_ic_err.c_str(); }

// sample_model (models.cpp:442-460): "plummer", "hernquist", "nfw", "disk", "m31".
// Returns 0, or 3 (data error) with g2_ics_last_error().
int g2_sample_model(const char* name, size_t n, uint64_t seed, unsigned threads, double* mass, double* pos,
                    double* vel) {
    try {
        if (n < 1) throw std::runtime_error("sampler: need at least one particle");
        if (threads == 0) threads = std::max(1u, std::thread::hardware_concurrency());
        const std::string nm(name);
        if (nm == "plummer") {
            plummer(n, 1.0, 1.0, seed, 0, 20.0, mass, pos, vel);
        } else if (nm == "hernquist") {
            hernquist(n, 1.0, 1.0, seed, 0, 20.0, nullptr, threads, mass, pos, vel);
        } else if (nm == "nfw") {
            nfw(n, 1.0, 1.0, 20.0, seed, 0, nullptr, threads, mass, pos, vel);
        } else if (nm == "disk") {
            const Catalog cat{{{kDisk, 1.0, 1.0, 0.1, 1.5}}};
            disk(n, 1.0, 1.0, 0.1, seed, cat, 1.5, 0.0, 0.0, threads, mass, pos, vel);
        } else if (nm == "m31") {
            build_m31(n, seed, threads, mass, pos, vel);
        } else {
            throw std::runtime_error("unknown model: " + nm);
        }
        return 0;
    } catch (const std::exception& e) {
        g_ic_err = e.what();
        return 3;
    }
}

}  // extern "C"
