// D3Q19 lattice constants and the canonical per-site arithmetic, shared by
// the host (setup, known-answer helpers) and the sm_100a kernels.
//
// Parity contract: the reference compiles with -ffp-contract=off
// (proj/CMakeLists.txt:15) and funnels all physics through
// lattice.hpp:99-149.  We build host code with -ffp-contract=off and device
// code with --fmad=false, and restate the same expression trees below.  The
// only rewrites are the exact ones: multiplications by +-1.0 become the
// operand or its negation, and "+ f*0.0" terms are dropped (exact up to the
// sign of an exactly-zero sum, which compares equal under the reference's
// `==`).  Inverse directions share the quadratic term,
// which is exact because (-a)*(-a) == a*a in IEEE arithmetic.
#pragma once

#include <cstdint>

#if defined(__CUDACC__)
#define SPLB_HD __host__ __device__ __forceinline__
#else
#define SPLB_HD inline
#endif

namespace splbcu {

constexpr int kQ = 19;

// lattice.hpp:23-43: rest; +x -x +y -y +z -z; xy(++,--,+-,-+), xz(...), yz(...)
// Packed as (c+1) in 2 bits per direction so host and device code share one
// definition without a __constant__ table.
namespace detail {
constexpr uint64_t pack19(const int (&c)[19]) {
    uint64_t r = 0;
    for (int i = 0; i < 19; ++i) r |= uint64_t(c[i] + 1) << (2 * i);
    return r;
}
constexpr int kCxTab[19] = {0, 1, -1, 0, 0, 0, 0, 1, -1, 1, -1, 1, -1, 1, -1, 0, 0, 0, 0};
constexpr int kCyTab[19] = {0, 0, 0, 1, -1, 0, 0, 1, -1, -1, 1, 0, 0, 0, 0, 1, -1, 1, -1};
constexpr int kCzTab[19] = {0, 0, 0, 0, 0, 1, -1, 0, 0, 0, 0, 1, -1, -1, 1, 1, -1, -1, 1};
constexpr uint64_t kCxPack = pack19(kCxTab);
constexpr uint64_t kCyPack = pack19(kCyTab);
constexpr uint64_t kCzPack = pack19(kCzTab);
}  // namespace detail
SPLB_HD constexpr int cx(int i) { return int((detail::kCxPack >> (2 * i)) & 3u) - 1; }
SPLB_HD constexpr int cy(int i) { return int((detail::kCyPack >> (2 * i)) & 3u) - 1; }
SPLB_HD constexpr int cz(int i) { return int((detail::kCzPack >> (2 * i)) & 3u) - 1; }
// lattice.hpp:45-46: inverse(i) = i+1 for odd i, i-1 for even i >= 2
SPLB_HD constexpr int inv(int i) { return i == 0 ? 0 : ((i & 1) ? i + 1 : i - 1); }
// lattice.hpp:48-52 (same constant expressions, so the same doubles)
constexpr double kW0 = 1.0 / 3.0;
constexpr double kW1 = 1.0 / 18.0;
constexpr double kW2 = 1.0 / 36.0;
constexpr double kCs2 = 1.0 / 3.0;  // lattice.hpp:54

SPLB_HD double weight(int i) { return i == 0 ? kW0 : (i <= 6 ? kW1 : kW2); }

struct Macro {
    double rho, ux, uy, uz;
};

// kernel::macro_of (lattice.hpp:106-119).  Each accumulator runs over the
// directions in ascending order; zero-coefficient terms are dropped and
// +-1 coefficients folded (exact, see header).
SPLB_HD Macro macro_of(const double* f) {
    double rho = f[0];
#pragma unroll
    for (int i = 1; i < kQ; ++i) rho = rho + f[i];
    double mx = f[1];
    mx = mx - f[2];
    mx = mx + f[7];
    mx = mx - f[8];
    mx = mx + f[9];
    mx = mx - f[10];
    mx = mx + f[11];
    mx = mx - f[12];
    mx = mx + f[13];
    mx = mx - f[14];
    double my = f[3];
    my = my - f[4];
    my = my + f[7];
    my = my - f[8];
    my = my - f[9];
    my = my + f[10];
    my = my + f[15];
    my = my - f[16];
    my = my + f[17];
    my = my - f[18];
    double mz = f[5];
    mz = mz - f[6];
    mz = mz + f[11];
    mz = mz - f[12];
    mz = mz - f[13];
    mz = mz + f[14];
    mz = mz + f[15];
    mz = mz - f[16];
    mz = mz - f[17];
    mz = mz + f[18];
    return {rho, mx / rho, my / rho, mz / rho};
}

// kernel::usq_term (lattice.hpp:122-124): 1.5*((ux*ux + uy*uy) + uz*uz)
SPLB_HD double usq_term(double ux, double uy, double uz) {
    return 1.5 * ((ux * ux + uy * uy) + uz * uz);
}

// c_i . u for the even-indexed member of each inverse pair (i = 1,3,5,...),
// i.e. (cx*ux + cy*uy) + cz*uz with the exact folds; the odd partner is its
// negation.  Index p = 0..8 selects directions 1,3,5,7,9,11,13,15,17.
SPLB_HD void cdot_pairs(double ux, double uy, double uz, double c[9]) {
    c[0] = ux;       // dir 1  (+1, 0, 0)
    c[1] = uy;       // dir 3  ( 0,+1, 0)
    c[2] = uz;       // dir 5  ( 0, 0,+1)
    c[3] = ux + uy;  // dir 7  (+1,+1, 0)
    c[4] = ux - uy;  // dir 9  (+1,-1, 0)
    c[5] = ux + uz;  // dir 11 (+1, 0,+1)
    c[6] = ux - uz;  // dir 13 (+1, 0,-1)
    c[7] = uy + uz;  // dir 15 ( 0,+1,+1)
    c[8] = uy - uz;  // dir 17 ( 0,+1,-1)
}

// Full equilibrium set (lattice.hpp:128-133 applied to i = 0..18):
// feq_i = (w_i*rho) * (((1 + cu3) + ((0.5*cu3)*cu3)) - usq15),
// cu3 = 3*(c_i.u).  For the inverse partner cu3 -> -cu3 exactly.
SPLB_HD void feq_all(double rho, double ux, double uy, double uz, double feq[kQ]) {
    const double usq15 = usq_term(ux, uy, uz);
    const double wr0 = kW0 * rho, wr1 = kW1 * rho, wr2 = kW2 * rho;
    // i = 0: cu3 = 3*(+-0) so (1 + cu3) + (0.5*cu3)*cu3 == 1 exactly.
    feq[0] = wr0 * (1.0 - usq15);
    double c[9];
    cdot_pairs(ux, uy, uz, c);
#pragma unroll
    for (int p = 0; p < 9; ++p) {
        const double cu3 = 3.0 * c[p];
        const double q = (0.5 * cu3) * cu3;
        const double wr = p < 3 ? wr1 : wr2;
        feq[2 * p + 1] = wr * (((1.0 + cu3) + q) - usq15);
        feq[2 * p + 2] = wr * (((1.0 - cu3) + q) - usq15);
    }
}

// Single-direction equilibrium (for the Nash pressure iolet, boundary.hpp:129-132).
SPLB_HD double feq_one(int i, double rho, double ux, double uy, double uz) {
    const double usq15 = usq_term(ux, uy, uz);
    if (i == 0) return (kW0 * rho) * (1.0 - usq15);
    double c[9];
    cdot_pairs(ux, uy, uz, c);
    const int p = (i - 1) >> 1;
    const double cu3 = (i & 1) ? 3.0 * c[p] : -(3.0 * c[p]);
    const double wr = (i <= 6 ? kW1 : kW2) * rho;
    return wr * (((1.0 + cu3) + ((0.5 * cu3) * cu3)) - usq15);
}

// kernel::relax (lattice.hpp:136-138)
SPLB_HD double relax(double f, double feq, double omega) { return f - omega * (f - feq); }

// kernel::ladd_term (lattice.hpp:142-147): (((2*w_i)*rho)*cu)*3 with
// cu = (cx*ub0 + cy*ub1) + cz*ub2 folded.
SPLB_HD double ladd_term(int i, double rho, double ub0, double ub1, double ub2) {
    double c[9];
    cdot_pairs(ub0, ub1, ub2, c);
    const int p = (i - 1) >> 1;
    const double cu = (i & 1) ? c[p] : -c[p];
    return (((2.0 * weight(i)) * rho) * cu) * 3.0;
}

// iolet_weight (boundary.hpp:107-113)
SPLB_HD double iolet_weight(const double center[3], const double normal[3],
                            double radius, int x, int y, int z) {
    const double d0 = double(x) - center[0];
    const double d1 = double(y) - center[1];
    const double d2 = double(z) - center[2];
    const double axial = (d0 * normal[0] + d1 * normal[1]) + d2 * normal[2];
    const double r0 = d0 - normal[0] * axial;
    const double r1 = d1 - normal[1] * axial;
    const double r2 = d2 - normal[2] * axial;
    const double w = 1.0 - ((r0 * r0 + r1 * r1) + r2 * r2) / (radius * radius);
    return w < 0.0 ? 0.0 : (w > 1.0 ? 1.0 : w);
}

}  // namespace splbcu
