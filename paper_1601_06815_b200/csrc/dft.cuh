// dft.cuh -- register-resident small DFT codelets for the OaA block transforms.
//
// PAPER.md:27 (§2): "Each convolution in OaA can be efficiently computed in the
// frequency domain, where the bottleneck is the complexity of each 2-D fast Fourier
// transform O(n² log n)".  The block transforms here are P = 2n−1 points per axis
// ("2n−1 in OaAconv"), i.e. P ∈ {1,3,5,7,9,11,13,15} for n ≤ 8.  All
// twiddles are compile-time constants (folded into FFMA immediates); inputs that are
// known to be zero (the n of P points that a zero-padded n×n block leaves non-zero)
// are pruned at compile time through the MASK template parameter (bit j set = input j
// may be non-zero).
//
// Codelets (SIGN = −1 forward, +1 inverse, unnormalised):
//   * dft_pair   : any odd P, pairing x_j with x_{P−j} (cos/sin split); 36 flops at P=5.
//   * dft15_pfa  : P = 15 by Good–Thomas 3×5 prime-factor mapping, no twiddles.
//   * dft9_ct    : P = 9 by Cooley–Tukey 3×3 with 4 twiddles.
//   * c2r_half   : Hermitian half-spectrum Z[0..H) → real y[0..P) (pairs p, P−p);
//                  P = 15 by a Hermitian-pruned PFA 3×5 (c2r15_pfa).
#pragma once
#include <cstdint>

#ifndef OAA_HD
#define OAA_HD __host__ __device__ __forceinline__
#endif

namespace oaa {

constexpr double kTwoPi = 6.283185307179586476925286766559;

constexpr double cx_sin_r(double x) {
  double x2 = x * x, t = x, s = x;
  for (int i = 1; i < 16; ++i) {
    t *= -x2 / ((2.0 * i) * (2.0 * i + 1.0));
    s += t;
  }
  return s;
}
constexpr double cx_cos_r(double x) {
  double x2 = x * x, t = 1.0, s = 1.0;
  for (int i = 1; i < 16; ++i) {
    t *= -x2 / ((2.0 * i - 1.0) * (2.0 * i));
    s += t;
  }
  return s;
}
// cos / sin of 2π·m/P with m reduced into (−P/2, P/2] before the series.
constexpr double cx_cos2pi(int m, int P) {
  m %= P;
  if (m < 0) m += P;
  if (2 * m > P) m -= P;
  return cx_cos_r(kTwoPi * m / P);
}
constexpr double cx_sin2pi(int m, int P) {
  m %= P;
  if (m < 0) m += P;
  if (2 * m > P) m -= P;
  return cx_sin_r(kTwoPi * m / P);
}

template <int P>
struct Tw {
  float c[P], s[P];
  constexpr Tw() : c(), s() {
    for (int m = 0; m < P; ++m) {
      c[m] = (float)cx_cos2pi(m, P);
      s[m] = (float)cx_sin2pi(m, P);
    }
  }
};

constexpr bool bit(unsigned mask, int j) { return (mask >> j) & 1u; }
constexpr unsigned full_mask(int P) { return (P >= 32) ? 0xffffffffu : ((1u << P) - 1u); }
constexpr unsigned lead_mask(int nz) { return (nz >= 32) ? 0xffffffffu : ((1u << nz) - 1u); }

// ---------------------------------------------------------------- generic odd P
// y[k] = Σ_j x[j]·exp(SIGN·2πi·jk/P).  In/out arrays may alias only if identical.
template <int P, int SIGN, unsigned MASK>
OAA_HD void dft_pair(const float* xr, const float* xi, float* yr, float* yi) {
  static_assert(P % 2 == 1, "odd P only");
  constexpr Tw<P> tw{};
  constexpr int h = (P - 1) / 2;
  if constexpr (P == 1) {
    yr[0] = bit(MASK, 0) ? xr[0] : 0.f;
    yi[0] = bit(MASK, 0) ? xi[0] : 0.f;
  } else {
    float sr[h + 1], si[h + 1], dr[h + 1], di[h + 1];
#pragma unroll
    for (int j = 1; j <= h; ++j) {
      const bool a = bit(MASK, j), b = bit(MASK, P - j);
      if (a && b) {
        sr[j] = xr[j] + xr[P - j];
        si[j] = xi[j] + xi[P - j];
        dr[j] = xr[j] - xr[P - j];
        di[j] = xi[j] - xi[P - j];
      } else if (a) {
        sr[j] = xr[j]; si[j] = xi[j]; dr[j] = xr[j]; di[j] = xi[j];
      } else if (b) {
        sr[j] = xr[P - j]; si[j] = xi[P - j]; dr[j] = -xr[P - j]; di[j] = -xi[P - j];
      } else {
        sr[j] = si[j] = dr[j] = di[j] = 0.f;
      }
    }
    const bool z0 = bit(MASK, 0);
    const float x0r = z0 ? xr[0] : 0.f, x0i = z0 ? xi[0] : 0.f;
    float out_r[P], out_i[P];
    {
      float ar = x0r, ai = x0i;
#pragma unroll
      for (int j = 1; j <= h; ++j)
        if (bit(MASK, j) || bit(MASK, P - j)) { ar += sr[j]; ai += si[j]; }
      out_r[0] = ar;
      out_i[0] = ai;
    }
#pragma unroll
    for (int k = 1; k <= h; ++k) {
      float ar = x0r, ai = x0i, br = 0.f, bi = 0.f;
      bool bfirst = true;
#pragma unroll
      for (int j = 1; j <= h; ++j) {
        if (!(bit(MASK, j) || bit(MASK, P - j))) continue;
        const float c = tw.c[(j * k) % P], s = tw.s[(j * k) % P];
        ar = fmaf(c, sr[j], ar);
        ai = fmaf(c, si[j], ai);
        if (bfirst) { br = s * dr[j]; bi = s * di[j]; bfirst = false; }
        else { br = fmaf(s, dr[j], br); bi = fmaf(s, di[j], bi); }
      }
      // X[k] = A + SIGN·i·B ; X[P−k] = A − SIGN·i·B
      out_r[k] = ar - SIGN * bi;
      out_i[k] = ai + SIGN * br;
      out_r[P - k] = ar + SIGN * bi;
      out_i[P - k] = ai - SIGN * br;
    }
#pragma unroll
    for (int k = 0; k < P; ++k) { yr[k] = out_r[k]; yi[k] = out_i[k]; }
  }
}

// ---------------------------------------------------------- P = 15, PFA 3 × 5
// n = (5·n1 + 3·n2) mod 15, k = (10·k1 + 6·k2) mod 15  ⇒  W15^{nk} = W3^{n1k1}·W5^{n2k2}.
constexpr unsigned pfa15_in_mask5(unsigned mask, int n1) {
  unsigned m = 0;
  for (int n2 = 0; n2 < 5; ++n2)
    if (bit(mask, (5 * n1 + 3 * n2) % 15)) m |= 1u << n2;
  return m;
}
constexpr unsigned pfa15_mask3(unsigned mask) {
  unsigned m = 0;
  for (int n1 = 0; n1 < 3; ++n1)
    if (pfa15_in_mask5(mask, n1)) m |= 1u << n1;
  return m;
}
template <int SIGN, unsigned MASK>
OAA_HD void dft15_pfa(const float* xr, const float* xi, float* yr, float* yi) {
  float ar[3][5], ai[3][5];
#pragma unroll
  for (int n1 = 0; n1 < 3; ++n1) {
    float tr[5], ti[5];
#pragma unroll
    for (int n2 = 0; n2 < 5; ++n2) {
      const int idx = (5 * n1 + 3 * n2) % 15;
      tr[n2] = xr[idx];
      ti[n2] = xi[idx];
    }
    // masks must be compile-time: dispatch on n1 explicitly
    if (n1 == 0) dft_pair<5, SIGN, pfa15_in_mask5(MASK, 0)>(tr, ti, ar[0], ai[0]);
    if (n1 == 1) dft_pair<5, SIGN, pfa15_in_mask5(MASK, 1)>(tr, ti, ar[1], ai[1]);
    if (n1 == 2) dft_pair<5, SIGN, pfa15_in_mask5(MASK, 2)>(tr, ti, ar[2], ai[2]);
  }
#pragma unroll
  for (int k2 = 0; k2 < 5; ++k2) {
    float tr[3] = {ar[0][k2], ar[1][k2], ar[2][k2]};
    float ti[3] = {ai[0][k2], ai[1][k2], ai[2][k2]};
    float orr[3], oi[3];
    dft_pair<3, SIGN, pfa15_mask3(MASK)>(tr, ti, orr, oi);
#pragma unroll
    for (int k1 = 0; k1 < 3; ++k1) {
      const int k = (10 * k1 + 6 * k2) % 15;
      yr[k] = orr[k1];
      yi[k] = oi[k1];
    }
  }
}

// ----------------------------------------------------------- P = 9, CT 3 × 3
// n = 3·n1 + n2, k = k1 + 3·k2:  X[k] = Σ_{n2} W9^{n2 k1} [Σ_{n1} x[3n1+n2] W3^{n1 k1}] W3^{n2 k2}
constexpr unsigned ct9_in_mask3(unsigned mask, int n2) {
  unsigned m = 0;
  for (int n1 = 0; n1 < 3; ++n1)
    if (bit(mask, 3 * n1 + n2)) m |= 1u << n1;
  return m;
}
template <int SIGN, unsigned MASK>
OAA_HD void dft9_ct(const float* xr, const float* xi, float* yr, float* yi) {
  constexpr Tw<9> tw{};
  float br[3][3], bi[3][3];  // [n2][k1]
#pragma unroll
  for (int n2 = 0; n2 < 3; ++n2) {
    float tr[3], ti[3];
#pragma unroll
    for (int n1 = 0; n1 < 3; ++n1) { tr[n1] = xr[3 * n1 + n2]; ti[n1] = xi[3 * n1 + n2]; }
    if (n2 == 0) dft_pair<3, SIGN, ct9_in_mask3(MASK, 0)>(tr, ti, br[0], bi[0]);
    if (n2 == 1) dft_pair<3, SIGN, ct9_in_mask3(MASK, 1)>(tr, ti, br[1], bi[1]);
    if (n2 == 2) dft_pair<3, SIGN, ct9_in_mask3(MASK, 2)>(tr, ti, br[2], bi[2]);
  }
  // twiddles W9^{SIGN·n2·k1}
#pragma unroll
  for (int n2 = 1; n2 < 3; ++n2) {
#pragma unroll
    for (int k1 = 1; k1 < 3; ++k1) {
      const float c = tw.c[(n2 * k1) % 9], s = SIGN * tw.s[(n2 * k1) % 9];
      const float r = br[n2][k1], i = bi[n2][k1];
      br[n2][k1] = fmaf(r, c, -i * s);
      bi[n2][k1] = fmaf(r, s, i * c);
    }
  }
  constexpr unsigned m2 = (ct9_in_mask3(MASK, 0) ? 1u : 0u) | (ct9_in_mask3(MASK, 1) ? 2u : 0u) |
                          (ct9_in_mask3(MASK, 2) ? 4u : 0u);
#pragma unroll
  for (int k1 = 0; k1 < 3; ++k1) {
    float tr[3] = {br[0][k1], br[1][k1], br[2][k1]};
    float ti[3] = {bi[0][k1], bi[1][k1], bi[2][k1]};
    float orr[3], oi[3];
    dft_pair<3, SIGN, m2>(tr, ti, orr, oi);
#pragma unroll
    for (int k2 = 0; k2 < 3; ++k2) { yr[k1 + 3 * k2] = orr[k2]; yi[k1 + 3 * k2] = oi[k2]; }
  }
}

// -------------------------------------------------------------- dispatcher
template <int P, int SIGN, unsigned MASK = full_mask(P)>
OAA_HD void dft(const float* xr, const float* xi, float* yr, float* yi) {
  if constexpr (P == 15) dft15_pfa<SIGN, MASK>(xr, xi, yr, yi);
  else if constexpr (P == 9) dft9_ct<SIGN, MASK>(xr, xi, yr, yi);
  else dft_pair<P, SIGN, MASK>(xr, xi, yr, yi);
}

// ------------------------------------------------- Hermitian half → real (inverse)
// y[p] = Z0r + Σ_{f=1}^{H−1} 2·Re(Z[f]·exp(+2πi·f·p/P)),  H = (P+1)/2 (odd P).
// P = 15 Hermitian → real by the 3 × 5 prime-factor map of dft15_pfa with the roles of
// the index maps swapped (input k = 5k1 + 3k2, output n = 10n1 + 6n2, both mod 15):
//   A[n1][k2] = Σ_k1 Z[5k1 + 3k2]·W3^{n1 k1}      (Hermitian in k2: only k2 = 0, 1, 2;
//                                                  column k2 = 0 is real)
//   y[10n1 + 6n2] = Σ_k2 A[n1][k2]·W5^{n2 k2}     (three real-output 5-point c2r)
// Z[k] for k ≥ 8 is conj(Z[15 − k]).  ~74 flops instead of ~120 for the direct form.
template <int P>
OAA_HD void c2r_half(const float* zr, const float* zi, float* y);

OAA_HD void c2r15_pfa(const float* zr, const float* zi, float* y) {
  constexpr float r3 = 1.7320508075688772f;
  // k2 = 0: (Z0, Z5, conj Z5) → real
  const float t0 = zr[0] - zr[5];
  float a0[3] = {fmaf(2.f, zr[5], zr[0]), fmaf(-r3, zi[5], t0), fmaf(r3, zi[5], t0)};
  // k2 = 1: (Z3, conj Z7, conj Z2);  k2 = 2: (Z6, conj Z4, Z1)
  float xr1[3] = {zr[3], zr[7], zr[2]}, xi1[3] = {zi[3], -zi[7], -zi[2]};
  float xr2[3] = {zr[6], zr[4], zr[1]}, xi2[3] = {zi[6], -zi[4], zi[1]};
  float a1r[3], a1i[3], a2r[3], a2i[3];
  dft_pair<3, +1, 7u>(xr1, xi1, a1r, a1i);
  dft_pair<3, +1, 7u>(xr2, xi2, a2r, a2i);
#pragma unroll
  for (int n1 = 0; n1 < 3; ++n1) {
    const float cr[3] = {a0[n1], a1r[n1], a2r[n1]};
    const float ci[3] = {0.f, a1i[n1], a2i[n1]};
    float o[5];
    c2r_half<5>(cr, ci, o);
#pragma unroll
    for (int n2 = 0; n2 < 5; ++n2) y[(10 * n1 + 6 * n2) % 15] = o[n2];
  }
}

template <int P>
OAA_HD void c2r_half(const float* zr, const float* zi, float* y) {
  constexpr Tw<P> tw{};
  constexpr int H = (P + 1) / 2;
  if constexpr (P == 15) {
    c2r15_pfa(zr, zi, y);
  } else if constexpr (P == 1) {
    y[0] = zr[0];
  } else {
    float s = 0.f;
#pragma unroll
    for (int f = 1; f < H; ++f) s += zr[f];
    y[0] = fmaf(2.f, s, zr[0]);
#pragma unroll
    for (int p = 1; p < H; ++p) {
      float a = zr[0], b = 0.f;
#pragma unroll
      for (int f = 1; f < H; ++f) {
        const float c2 = 2.f * tw.c[(f * p) % P], s2 = 2.f * tw.s[(f * p) % P];
        a = fmaf(c2, zr[f], a);
        b = (f == 1) ? s2 * zi[f] : fmaf(s2, zi[f], b);
      }
      y[p] = a - b;
      y[P - p] = a + b;
    }
  }
}

}  // namespace oaa
