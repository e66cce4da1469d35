// Index maps of the three implicit-GEMM forms (FPROP / DGRAD / WGRAD) over the
// NHWC label-batched maps described in common.cuh.  Shared by the SIMT engine
// (gemm_simt.cu) and the tcgen05 engine (gemm_tc.cu): both ask the same
// questions ("which global address holds A[m][k]?") and differ only in how the
// tile is staged and multiplied.
//
// Reference semantics: conv fwd = im2col + W*col (network.cpp:63-102); conv
// backward = W^T*go + col2im scatter, gw += go*col^T (network.cpp:104-144);
// ConvTranspose2d is the adjoint pair; dense = the k=1 special
// case (network.cpp:28-45).  Here the scatter (col2im) is replaced by the
// phase-decomposed gather, so every output element is written exactly once by
// one GEMM row and no float atomics are needed.
#pragma once

#include "common.cuh"

namespace pg {

// Per-(label, phase) problem view, built once per CTA.
struct GemmView {
  int M, N, K;
  // DGRAD phase data
  int ry, rx, y0, x0, ny, nx, ntx;
  const float* A;  // label-offset base of the A source tensor
  const float* Bw; // label-offset base of the B source (weight or big map)
  float* C;        // label-offset output
  const float* bias;
};

PG_DEV int ceil_div_dev(int a, int b) { return (a + b - 1) / b; }

// Number of phases for a GEMM launch (DGRAD decomposes the big map by stride).
__host__ __device__ inline int gemm_phases(const GemmArgs& a) { return a.kind == GEMM_DGRAD ? a.g.s * a.g.s : 1; }

PG_DEV GemmView make_view(const GemmArgs& a, int label, int phase) {
  const ConvGeo& g = a.g;
  GemmView v;
  v.ry = v.rx = v.y0 = v.x0 = v.ny = v.nx = v.ntx = 0;
  v.C = a.out + (long long)label * a.out_ls;
  v.bias = a.bias ? a.bias + (long long)label * a.bias_ls : nullptr;
  if (a.kind == GEMM_FPROP) {
    v.M = g.B * g.SH * g.SW;
    v.N = g.CS;
    v.K = g.k * g.k * g.CG;
    v.A = a.big + (long long)label * a.big_ls;
    v.Bw = a.w + (long long)label * a.w_ls;
  } else if (a.kind == GEMM_DGRAD) {
    v.ry = phase / g.s;
    v.rx = phase % g.s;
    v.y0 = phase_origin(v.ry, g.s, g.p);
    v.x0 = phase_origin(v.rx, g.s, g.p);
    v.ny = v.y0 < g.GH ? ceil_div_dev(g.GH - v.y0, g.s) : 0;
    v.nx = v.x0 < g.GW ? ceil_div_dev(g.GW - v.x0, g.s) : 0;
    int nty = v.ry < g.k ? ceil_div_dev(g.k - v.ry, g.s) : 0;
    v.ntx = v.rx < g.k ? ceil_div_dev(g.k - v.rx, g.s) : 0;
    v.M = g.B * v.ny * v.nx;
    v.N = g.CG;
    v.K = nty * v.ntx * g.CS;
    v.A = a.small + (long long)label * a.small_ls;
    v.Bw = a.w + (long long)label * a.w_ls;
  } else {  // WGRAD
    v.M = g.CS;
    v.N = g.k * g.k * g.CG;
    v.K = g.B * g.SH * g.SW;
    v.A = a.small + (long long)label * a.small_ls;
    v.Bw = a.big + (long long)label * a.big_ls;
  }
  return v;
}

// ---- FPROP ----------------------------------------------------------------
// A[m][kk]: m = (b, i, j) small pixel, kk = (tap, cg); K-major (cg contiguous).
PG_DEV const float* fprop_a_ptr(const ConvGeo& g, const GemmView& v, int m, int kk) {
  int cg = kk % g.CG, tap = kk / g.CG;
  int ki = tap / g.k, kj = tap % g.k;
  int j = m % g.SW, t = m / g.SW;
  int i = t % g.SH, b = t / g.SH;
  int y = i * g.s - g.p + ki, x = j * g.s - g.p + kj;
  if (y < 0 || y >= g.GH || x < 0 || x >= g.GW) return nullptr;
  return v.A + (((long long)b * g.GH + y) * g.GW + x) * g.CG + cg;
}
// B[n][kk] = W[cs=n][tap][cg]; K-major, contiguous over the whole K.
PG_DEV const float* fprop_b_ptr(const ConvGeo&, const GemmView& v, int n, int kk) {
  return v.Bw + (long long)n * v.K + kk;
}
PG_DEV float* fprop_c_ptr(const ConvGeo& g, const GemmView& v, int m, int n) {
  return v.C + (long long)m * g.CS + n;
}

// ---- DGRAD (one phase) ------------------------------------------------------
// A[m][kk]: m = (b, yi, xi) big pixel of the phase; kk = (tap of phase, cs).
PG_DEV const float* dgrad_a_ptr(const ConvGeo& g, const GemmView& v, int m, int kk) {
  int cs = kk % g.CS, t = kk / g.CS;
  int ty = t / v.ntx, tx = t % v.ntx;
  int ki = v.ry + ty * g.s, kj = v.rx + tx * g.s;
  int xi = m % v.nx, r = m / v.nx;
  int yi = r % v.ny, b = r / v.ny;
  int y = v.y0 + yi * g.s, x = v.x0 + xi * g.s;
  int i = (y + g.p - ki) / g.s, j = (x + g.p - kj) / g.s;
  if (i < 0 || i >= g.SH || j < 0 || j >= g.SW) return nullptr;
  return v.A + (((long long)b * g.SH + i) * g.SW + j) * g.CS + cs;
}
// B[n = cg][kk = (tap, cs)] = W[cs][ki][kj][cg]; MN-major (cg contiguous).
PG_DEV const float* dgrad_b_ptr(const ConvGeo& g, const GemmView& v, int n, int kk) {
  int cs = kk % g.CS, t = kk / g.CS;
  int ty = t / v.ntx, tx = t % v.ntx;
  int ki = v.ry + ty * g.s, kj = v.rx + tx * g.s;
  return v.Bw + (((long long)cs * g.k + ki) * g.k + kj) * g.CG + n;
}
PG_DEV float* dgrad_c_ptr(const ConvGeo& g, const GemmView& v, int m, int n) {
  int xi = m % v.nx, r = m / v.nx;
  int yi = r % v.ny, b = r / v.ny;
  int y = v.y0 + yi * g.s, x = v.x0 + xi * g.s;
  return v.C + (((long long)b * g.GH + y) * g.GW + x) * g.CG + n;
}

// ---- WGRAD ------------------------------------------------------------------
// A[m = cs][kk = spix] = smallg[spix][cs]; MN-major.
PG_DEV const float* wgrad_a_ptr(const ConvGeo& g, const GemmView& v, int m, int kk) {
  return v.A + (long long)kk * g.CS + m;
}
// B[n = (tap, cg)][kk = spix] = big[gather(spix, tap)][cg]; MN-major.
PG_DEV const float* wgrad_b_ptr(const ConvGeo& g, const GemmView& v, int n, int kk) {
  int cg = n % g.CG, tap = n / g.CG;
  int ki = tap / g.k, kj = tap % g.k;
  int j = kk % g.SW, t = kk / g.SW;
  int i = t % g.SH, b = t / g.SH;
  int y = i * g.s - g.p + ki, x = j * g.s - g.p + kj;
  if (y < 0 || y >= g.GH || x < 0 || x >= g.GW) return nullptr;
  return v.Bw + (((long long)b * g.GH + y) * g.GW + x) * g.CG + cg;
}
PG_DEV float* wgrad_c_ptr(const ConvGeo&, const GemmView& v, int m, int n) { return v.C + (long long)m * v.N + n; }

}  // namespace pg
