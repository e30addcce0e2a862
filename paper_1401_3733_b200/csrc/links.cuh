// Gauge-link storage formats and the link x half-spinor multiply (sm_100a).
//
// The reference stores every represented link as a dense dr x dr complex (or
// real, adjoint) matrix (proj/include/latbench/fields.hpp:37-57). Links are
// 67-86 % of the Dslash's compulsory HBM traffic, so the device keeps them in
// the most compact exact form the group structure allows and rebuilds the
// represented matrix in registers (fp64 FMAs are nearly free in this
// HBM-bound kernel):
//
//   GF_FULL : dense dr x dr (any representation), antiperiodic sign baked in
//   GF_SU2  : SU(2) element U = [[al, be], [-conj(be), conj(al)]], 2 complex:
//             fundamental (dr = 2) directly; adjoint (dr = 3, real) through
//             R_ab = 1/2 tr(s_a U s_b U^dag) = (a0^2 - |a|^2) d_ab + 2 a_a a_b
//             - 2 a0 eps_abc a_c with al = a0 + i a3, be = a2 + i a1
//             (group.cpp:126-143 convention, checked in tests/test_host.py)
//   GF_R12  : SU(3) rows 0 and 1 (6 complex); row 2 = conj(row0 x row1)
//   GF_R10  : SU(3) row 0 and U_11, U_12 (5 complex, 80 B): U_10 from the
//             orthogonality of rows 0 and 1,
//             U_10 = -(conj(U_01) U_11 + conj(U_02) U_12) / conj(U_00),
//             then row 2 as R12. Trig-free; the division by U_00 is well
//             conditioned for near-unit links (|U_00| ~ 1) and loses at most
//             eps / |U_00| for Haar links; the upload check (1e-12) falls
//             back to R12 for any field where it would not be exact
//   GF_AS4  : two-index antisymmetric rep of SU(4) (dr = 6) stored as the
//             fundamental 4 x 4 element (16 complex instead of 36); entries
//             R_(ij),(kl) = u_ik u_jl - u_il u_jk (group.cpp:146-158) are
//             formed in registers. Uploaded through lbcu_gauge_upload_fundamental.
//   GF_AS4R : the same representation as a REAL SO(6) matrix. The 6 of SU(4)
//             is a real representation: in the basis B whose columns are
//             s(e_a + g e_b), i s(e_a - g e_b) for the complementary index
//             pairs (01|23, g=+1), (02|13, g=-1), (03|12, g=+1), s = 1/sqrt2,
//             R' = B^dag R B is real orthogonal (36 doubles = 288 B, stored as
//             18 double2). Kernels carry colour vectors in Wt = sqrt2 B^dag:
//             Wt (R h) = R' (Wt h), so h is rotated per hop (12 adds), the
//             multiply is real x complex (a quarter of the FP64 work of the
//             AS4 minors), and the accumulator is rotated back once per site,
//             acc = 1/2 Wt^dag acc'.
//
// Compact formats are chosen at upload only when every link reconstructs to
// within 1e-12 of the uploaded matrix (gauge.cu), so arbitrary user links
// (non-unitary, tampered) stay exact in GF_FULL. In compact formats the
// antiperiodic time sign is applied in the kernel instead of being baked in
// (a baked -U would break det U = 1 for SU(3)).
#pragma once

#include <type_traits>

#include "device.cuh"

namespace lbcu {

// Link loads: the read-only path. (L1::no_allocate hints, to leave L1 to the
// neighbour spinors, measured 0-8 % slower: the full Dphi's two parities
// share links through L1.)
// SM = true: the entry sits in a shared-memory tile staged by a bulk async
// copy (dslash.cu, link staging), read with a plain load.
template <bool SM = false, class T>
__device__ __forceinline__ T ldlink(const T* p) {
  if constexpr (SM) return *p;
  else return __ldg(p);
}

enum GaugeFmt { GF_FULL = 0, GF_SU2 = 1, GF_R12 = 2, GF_AS4 = 3, GF_AS4R = 4, GF_R10 = 5 };

template <bool REAL>
using LinkT = std::conditional_t<REAL, double, double2>;

template <int D, bool REAL, int FMT>
struct LinkFmt {
  static constexpr bool valid = FMT == GF_FULL || (FMT == GF_SU2 && ((D == 2 && !REAL) || (D == 3 && REAL))) ||
                                ((FMT == GF_R12 || FMT == GF_R10) && D == 3 && !REAL) ||
                                ((FMT == GF_AS4 || FMT == GF_AS4R) && D == 6 && !REAL);
  static constexpr int entries =
      FMT == GF_FULL ? D * D
                     : (FMT == GF_SU2 ? 2 : (FMT == GF_R12 ? 6 : (FMT == GF_R10 ? 5 : (FMT == GF_AS4 ? 16 : 18))));
  using Elem = std::conditional_t<FMT == GF_FULL, LinkT<REAL>, double2>;
};

// lexicographic pairs i < j of SU(4) indices (group.cpp:119-124)
__host__ __device__ constexpr int as4_i(int p) { return p < 3 ? 0 : (p < 5 ? 1 : 2); }
__host__ __device__ constexpr int as4_j(int p) { return p < 3 ? p + 1 : (p < 5 ? p - 1 : 3); }

__device__ __forceinline__ double2 cconj(double2 a) { return make_double2(a.x, -a.y); }
__device__ __forceinline__ double2 cmul(double2 a, double2 b) {
  return make_double2(fma(a.x, b.x, -a.y * b.y), fma(a.x, b.y, a.y * b.x));
}
__device__ __forceinline__ double2 csub(double2 a, double2 b) { return make_double2(a.x - b.x, a.y - b.y); }

// ---- GF_AS4R basis (see header) --------------------------------------------
// pair k = 0, 1, 2 couples colour indices a = k and b = 5 - k with sign g
__host__ __device__ constexpr double as4r_sign(int k) { return k == 1 ? -1.0 : 1.0; }

// B[i][x] (unitary, columns = real basis vectors)
__device__ __forceinline__ double2 as4r_B(int i, int x) {
  constexpr double s = 0.70710678118654752440;
  const int k = x >> 1, a = k, b = 5 - k;
  const double g = as4r_sign(k);
  if (i != a && i != b) return make_double2(0.0, 0.0);
  if (x & 1) return i == a ? make_double2(0.0, s) : make_double2(0.0, -g * s);
  return make_double2(i == a ? s : g * s, 0.0);
}

// R' = B^dag R B from a dense AS link; returns max |Im R'| (0 for SU(4))
__device__ __forceinline__ double as4r_from_dense(const double2 (&u)[36], double2 (&st)[18]) {
  double worst = 0.0;
#pragma unroll
  for (int x = 0; x < 6; ++x) {
    double row[6];
#pragma unroll
    for (int y = 0; y < 6; ++y) {
      double2 acc = make_double2(0.0, 0.0);
#pragma unroll
      for (int i = 0; i < 6; ++i) {
        const double2 bi = as4r_B(i, x);
        if (bi.x == 0.0 && bi.y == 0.0) continue;
#pragma unroll
        for (int j = 0; j < 6; ++j) {
          const double2 bj = as4r_B(j, y);
          if (bj.x == 0.0 && bj.y == 0.0) continue;
          const double2 t = cmul(cmul(cconj(bi), u[i * 6 + j]), bj);
          acc.x += t.x;
          acc.y += t.y;
        }
      }
      row[y] = acc.x;
      worst = fmax(worst, fabs(acc.y));
    }
#pragma unroll
    for (int q = 0; q < 3; ++q) st[3 * x + q] = make_double2(row[2 * q], row[2 * q + 1]);
  }
  return worst;
}

// o = Wt h = sqrt2 B^dag h
__device__ __forceinline__ void as4r_in(double2 (&o)[6], const double2 (&h)[6]) {
#pragma unroll
  for (int k = 0; k < 3; ++k) {
    const double g = as4r_sign(k);
    const double2 ha = h[k], hb = h[5 - k];
    o[2 * k] = make_double2(fma(g, hb.x, ha.x), fma(g, hb.y, ha.y));
    const double2 d = make_double2(fma(-g, hb.x, ha.x), fma(-g, hb.y, ha.y));
    o[2 * k + 1] = make_double2(d.y, -d.x);  // -i d
  }
}

// v <- scale * Wt^dag v, Wt^dag = sqrt2 B
__device__ __forceinline__ void as4r_out(double2 (&v)[6], double scale) {
  double2 w[6];
#pragma unroll
  for (int k = 0; k < 3; ++k) {
    const double g = as4r_sign(k);
    const double2 p = v[2 * k], q = v[2 * k + 1];
    w[k] = make_double2(scale * (p.x - q.y), scale * (p.y + q.x));          // p + i q
    w[5 - k] = make_double2(g * scale * (p.x + q.y), g * scale * (p.y - q.x));  // g (p - i q)
  }
#pragma unroll
  for (int c = 0; c < 6; ++c) v[c] = w[c];
}

// Rebuild the represented link (row-major D x D) from compact entries.
template <int D, bool REAL, int FMT>
__device__ __forceinline__ void build_link(LinkT<REAL> (&u)[D * D],
                                           const double2 (&s)[LinkFmt<D, REAL, FMT>::entries]) {
  static_assert(FMT != GF_FULL, "dense links need no rebuild");
  if constexpr (FMT == GF_SU2 && !REAL) {
    const double2 al = s[0], be = s[1];
    u[0] = al;
    u[1] = be;
    u[2] = make_double2(-be.x, be.y);
    u[3] = cconj(al);
  } else if constexpr (FMT == GF_SU2 && REAL) {
    const double2 al = s[0], be = s[1];
    const double a0 = al.x, a3 = al.y, a2 = be.x, a1 = be.y;
    const double d = a0 * a0 - (a1 * a1 + a2 * a2 + a3 * a3);
    const double t1 = 2.0 * a1, t2 = 2.0 * a2, t3 = 2.0 * a3, w = 2.0 * a0;
    u[0] = fma(t1, a1, d);
    u[1] = fma(t1, a2, w * a3);
    u[2] = fma(t1, a3, -w * a2);
    u[3] = fma(t2, a1, -w * a3);
    u[4] = fma(t2, a2, d);
    u[5] = fma(t2, a3, w * a1);
    u[6] = fma(t3, a1, w * a2);
    u[7] = fma(t3, a2, -w * a1);
    u[8] = fma(t3, a3, d);
  } else if constexpr (FMT == GF_R12 || FMT == GF_R10) {
    if constexpr (FMT == GF_R12) {
#pragma unroll
      for (int e = 0; e < 6; ++e) u[e] = s[e];
    } else {
      u[0] = s[0];
      u[1] = s[1];
      u[2] = s[2];
      u[4] = s[3];
      u[5] = s[4];
      // rows 0 and 1 orthogonal: conj(u0) u3 + conj(u1) u4 + conj(u2) u5 = 0
      const double2 t = make_double2(fma(u[1].x, u[4].x, fma(u[1].y, u[4].y, fma(u[2].x, u[5].x, u[2].y * u[5].y))),
                                     fma(u[1].x, u[4].y, fma(-u[1].y, u[4].x, fma(u[2].x, u[5].y, -u[2].y * u[5].x))));
      const double inv = -1.0 / fma(u[0].x, u[0].x, u[0].y * u[0].y);  // u3 = -t / conj(u0) = -t u0 / |u0|^2
      u[3] = make_double2(inv * fma(t.x, u[0].x, -t.y * u[0].y), inv * fma(t.x, u[0].y, t.y * u[0].x));
    }
    u[6] = cconj(csub(cmul(u[1], u[5]), cmul(u[2], u[4])));
    u[7] = cconj(csub(cmul(u[2], u[3]), cmul(u[0], u[5])));
    u[8] = cconj(csub(cmul(u[0], u[4]), cmul(u[1], u[3])));
  } else if constexpr (FMT == GF_AS4R) {  // R = B R' B^dag
    double m[36];
#pragma unroll
    for (int e = 0; e < 18; ++e) {
      m[2 * e] = s[e].x;
      m[2 * e + 1] = s[e].y;
    }
#pragma unroll
    for (int i = 0; i < 6; ++i)
#pragma unroll
      for (int j = 0; j < 6; ++j) {
        double2 acc = make_double2(0.0, 0.0);
#pragma unroll
        for (int x = 0; x < 6; ++x)
#pragma unroll
          for (int y = 0; y < 6; ++y) {
            const double2 bx = as4r_B(i, x), by = cconj(as4r_B(j, y));
            const double2 t = cmul(bx, by);
            acc.x = fma(m[x * 6 + y], t.x, acc.x);
            acc.y = fma(m[x * 6 + y], t.y, acc.y);
          }
        u[i * 6 + j] = acc;
      }
  } else {  // GF_AS4: all 36 minors of the fundamental element
#pragma unroll
    for (int p = 0; p < 6; ++p)
#pragma unroll
      for (int q = 0; q < 6; ++q) {
        const int i = as4_i(p), j = as4_j(p), k = as4_i(q), l = as4_j(q);
        u[p * 6 + q] = csub(cmul(s[i * 4 + k], s[j * 4 + l]), cmul(s[i * 4 + l], s[j * 4 + k]));
      }
  }
}

// Load a link from its storage (read-only path) and rebuild it.
template <int D, bool REAL, int FMT, bool SM = false>
__device__ __forceinline__ void load_link(LinkT<REAL> (&u)[D * D],
                                          const typename LinkFmt<D, REAL, FMT>::Elem* __restrict__ p,
                                          long long st) {
  if constexpr (FMT == GF_FULL) {
#pragma unroll
    for (int e = 0; e < D * D; ++e) u[e] = ldlink<SM>(p + (long long)e * st);
  } else {
    double2 s[LinkFmt<D, REAL, FMT>::entries];
#pragma unroll
    for (int e = 0; e < LinkFmt<D, REAL, FMT>::entries; ++e) s[e] = ldlink<SM>(p + (long long)e * st);
    build_link<D, REAL, FMT>(u, s);
  }
}

// GF_AS4R: g' = M hp with M = R' (or R'^T for the dagger), all in the Wt
// basis; the link is streamed one stored row (3 double2) at a time.
template <bool DAG, bool SM = false>
__device__ __forceinline__ void as4r_mul(double2 (&g)[2][6], const double2* __restrict__ p, long long st,
                                         const double2 (&hp)[2][6]) {
#pragma unroll
  for (int r = 0; r < 6; ++r) g[0][r] = g[1][r] = make_double2(0.0, 0.0);
#pragma unroll
  for (int r = 0; r < 6; ++r) {
    double m[6];
#pragma unroll
    for (int q = 0; q < 3; ++q) {
      const double2 v = ldlink<SM>(p + (long long)(3 * r + q) * st);
      m[2 * q] = v.x;
      m[2 * q + 1] = v.y;
    }
#pragma unroll
    for (int c = 0; c < 6; ++c) {
      if constexpr (DAG) {  // g[c] += R'_rc hp[r]
        rmac(g[0][c], m[c], hp[0][r]);
        rmac(g[1][c], m[c], hp[1][r]);
      } else {  // g[r] += R'_rc hp[c]
        rmac(g[0][r], m[c], hp[0][c]);
        rmac(g[1][r], m[c], hp[1][c]);
      }
    }
  }
}

// g[a][r] = sum_c M_rc h[a][c] with M = U (DAG = false) or U^dag (DAG = true)
template <int D, bool REAL, int FMT, bool DAG, bool SM = false>
__device__ __forceinline__ void link_mul(double2 (&g)[2][D],
                                         const typename LinkFmt<D, REAL, FMT>::Elem* __restrict__ p,
                                         long long st, const double2 (&h)[2][D]) {
  if constexpr (FMT == GF_AS4R) {  // result in the standard basis
    double2 hp[2][6];
    as4r_in(hp[0], h[0]);
    as4r_in(hp[1], h[1]);
    as4r_mul<DAG, SM>(g, p, st, hp);
    as4r_out(g[0], 0.5);
    as4r_out(g[1], 0.5);
    return;
  }
#pragma unroll
  for (int r = 0; r < D; ++r) g[0][r] = g[1][r] = make_double2(0.0, 0.0);
  if constexpr (FMT == GF_FULL) {
    // stream the entries: no need to hold the whole matrix in registers
#pragma unroll
    for (int r = 0; r < D; ++r)
#pragma unroll
      for (int c = 0; c < D; ++c) {
        const auto u = ldlink<SM>(p + (long long)(DAG ? c * D + r : r * D + c) * st);
        if constexpr (REAL) {
          rmac(g[0][r], u, h[0][c]);
          rmac(g[1][r], u, h[1][c]);
        } else if constexpr (DAG) {
          cmac_conj(g[0][r], u, h[0][c]);
          cmac_conj(g[1][r], u, h[1][c]);
        } else {
          cmac(g[0][r], u, h[0][c]);
          cmac(g[1][r], u, h[1][c]);
        }
      }
  } else {
    LinkT<REAL> u[D * D];
    load_link<D, REAL, FMT, SM>(u, p, st);
#pragma unroll
    for (int r = 0; r < D; ++r)
#pragma unroll
      for (int c = 0; c < D; ++c) {
        const auto e = u[DAG ? c * D + r : r * D + c];
        if constexpr (REAL) {
          rmac(g[0][r], e, h[0][c]);
          rmac(g[1][r], e, h[1][c]);
        } else if constexpr (DAG) {
          cmac_conj(g[0][r], e, h[0][c]);
          cmac_conj(g[1][r], e, h[1][c]);
        } else {
          cmac(g[0][r], e, h[0][c]);
          cmac(g[1][r], e, h[1][c]);
        }
      }
  }
}

// Row-fused multiply + spin reconstruction: for each colour row r,
//   g_a = sum_c M_rc h[a][c]  (a = 0, 1), then
//   acc[0][r] += g_0; acc[1][r] += g_1; acc[2][r] += Q0 g_R0; acc[3][r] += Q1 g_R1
// so the 2 x D intermediate g never has to be held in registers.
template <int D, bool REAL, int FMT, bool DAG, int R0, int R1, int Q0, int Q1, bool SM = false>
__device__ __forceinline__ void link_mul_acc(double2 (&acc)[4][D],
                                             const typename LinkFmt<D, REAL, FMT>::Elem* __restrict__ p,
                                             long long st, const double2 (&h)[2][D]) {
  if constexpr (FMT == GF_AS4R) {  // acc in the Wt basis (site_body rotates back)
    double2 hp[2][6], g[2][6];
    as4r_in(hp[0], h[0]);
    as4r_in(hp[1], h[1]);
    as4r_mul<DAG, SM>(g, p, st, hp);
#pragma unroll
    for (int r = 0; r < 6; ++r) {
      acc[0][r] = cadd(acc[0][r], g[0][r]);
      acc[1][r] = cadd(acc[1][r], g[1][r]);
      acc[2][r] = cadd(acc[2][r], phm<Q0>(g[R0][r]));
      acc[3][r] = cadd(acc[3][r], phm<Q1>(g[R1][r]));
    }
    return;
  }
  if constexpr (FMT == GF_AS4) {
    // keep only the fundamental element in registers; form each minor when used
    double2 s[16];
#pragma unroll
    for (int e = 0; e < 16; ++e) s[e] = ldlink<SM>(p + (long long)e * st);
#pragma unroll
    for (int r = 0; r < 6; ++r) {
      double2 g0 = make_double2(0.0, 0.0), g1 = make_double2(0.0, 0.0);
#pragma unroll
      for (int c = 0; c < 6; ++c) {
        // M_rc = R_rc, or conj(R_cr) for the dagger
        const int pr = DAG ? c : r, pc = DAG ? r : c;
        const int i = as4_i(pr), j = as4_j(pr), k = as4_i(pc), l = as4_j(pc);
        const double2 e = csub(cmul(s[i * 4 + k], s[j * 4 + l]), cmul(s[i * 4 + l], s[j * 4 + k]));
        if constexpr (DAG) {
          cmac_conj(g0, e, h[0][c]);
          cmac_conj(g1, e, h[1][c]);
        } else {
          cmac(g0, e, h[0][c]);
          cmac(g1, e, h[1][c]);
        }
      }
      acc[0][r] = cadd(acc[0][r], g0);
      acc[1][r] = cadd(acc[1][r], g1);
      acc[2][r] = cadd(acc[2][r], phm<Q0>(R0 == 0 ? g0 : g1));
      acc[3][r] = cadd(acc[3][r], phm<Q1>(R1 == 0 ? g0 : g1));
    }
    return;
  }
  [[maybe_unused]] LinkT<REAL> u[FMT == GF_FULL ? 1 : D * D];
  if constexpr (FMT != GF_FULL) load_link<D, REAL, FMT, SM>(u, p, st);
#pragma unroll
  for (int r = 0; r < D; ++r) {
    double2 g0 = make_double2(0.0, 0.0), g1 = make_double2(0.0, 0.0);
#pragma unroll
    for (int c = 0; c < D; ++c) {
      const int idx = DAG ? c * D + r : r * D + c;
      LinkT<REAL> e;
      if constexpr (FMT == GF_FULL) e = ldlink<SM>(p + (long long)idx * st);
      else e = u[idx];
      if constexpr (REAL) {
        rmac(g0, e, h[0][c]);
        rmac(g1, e, h[1][c]);
      } else if constexpr (DAG) {
        cmac_conj(g0, e, h[0][c]);
        cmac_conj(g1, e, h[1][c]);
      } else {
        cmac(g0, e, h[0][c]);
        cmac(g1, e, h[1][c]);
      }
    }
    acc[0][r] = cadd(acc[0][r], g0);
    acc[1][r] = cadd(acc[1][r], g1);
    acc[2][r] = cadd(acc[2][r], phm<Q0>(R0 == 0 ? g0 : g1));
    acc[3][r] = cadd(acc[3][r], phm<Q1>(R1 == 0 ? g0 : g1));
  }
}

}  // namespace lbcu
