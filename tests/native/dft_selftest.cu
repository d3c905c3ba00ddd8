// Host build of the product's DFT codelets (paper_1601_06815_b200/csrc/dft.cuh) so the
// CPU test suite can compare them with numpy's FFT (a library routine) without a GPU.
#include <cstring>
#include "../../paper_1601_06815_b200/csrc/dft.cuh"

template <int P>
static int run(int sign, int nz, const float* xr, const float* xi, float* yr, float* yi) {
  float a[P], b[P], c[P], d[P];
  for (int i = 0; i < P; ++i) { a[i] = xr[i]; b[i] = xi[i]; }
  const int n = (P + 1) / 2;
  if (sign < 0 && nz == n) oaa::dft<P, -1, oaa::lead_mask((P + 1) / 2)>(a, b, c, d);
  else if (sign < 0) oaa::dft<P, -1>(a, b, c, d);
  else oaa::dft<P, +1>(a, b, c, d);
  for (int i = 0; i < P; ++i) { yr[i] = c[i]; yi[i] = d[i]; }
  return 0;
}

template <int P>
static void c2r(const float* zr, const float* zi, float* y) {
  float a[(P + 1) / 2], b[(P + 1) / 2], o[P];
  for (int i = 0; i < (P + 1) / 2; ++i) { a[i] = zr[i]; b[i] = zi[i]; }
  oaa::c2r_half<P>(a, b, o);
  for (int i = 0; i < P; ++i) y[i] = o[i];
}

extern "C" int dft_selftest(int P, int sign, int nz, const float* xr, const float* xi, float* yr,
                            float* yi) {
  switch (P) {
    case 1: return run<1>(sign, nz, xr, xi, yr, yi);
    case 3: return run<3>(sign, nz, xr, xi, yr, yi);
    case 5: return run<5>(sign, nz, xr, xi, yr, yi);
    case 7: return run<7>(sign, nz, xr, xi, yr, yi);
    case 9: return run<9>(sign, nz, xr, xi, yr, yi);
    case 11: return run<11>(sign, nz, xr, xi, yr, yi);
    case 13: return run<13>(sign, nz, xr, xi, yr, yi);
    case 15: return run<15>(sign, nz, xr, xi, yr, yi);
  }
  return -1;
}

extern "C" int c2r_selftest(int P, const float* zr, const float* zi, float* y) {
  switch (P) {
    case 1: c2r<1>(zr, zi, y); return 0;
    case 3: c2r<3>(zr, zi, y); return 0;
    case 5: c2r<5>(zr, zi, y); return 0;
    case 7: c2r<7>(zr, zi, y); return 0;
    case 9: c2r<9>(zr, zi, y); return 0;
    case 11: c2r<11>(zr, zi, y); return 0;
    case 13: c2r<13>(zr, zi, y); return 0;
    case 15: c2r<15>(zr, zi, y); return 0;
  }
  return -1;
}
