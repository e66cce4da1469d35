// HBM-bound kernels of the training step, all batched over the L labels of a
// GPU: per-channel reductions (BatchNorm statistics and backward sums, bias
// gradients), BatchNorm apply with the fused activation, the fused
// activation/BatchNorm backward, the GAN losses, Adam, and data movement.
// Reductions are deterministic: fixed row chunks, fixed in-block order and a
// fixed-order second pass over the chunk partials (no float atomics).
#include "kernels.hpp"

#include <algorithm>
#include <cmath>

namespace pg {

namespace {

constexpr int RED_NT = 256;

// rows per reduction chunk: 512, halved (down to 32) until every label has
// ~10 blocks, so the small deep-layer maps (a few hundred rows per label)
// are not latency bound on a handful of blocks.  A pure function of the map:
// the reduce kernel and every reader of its partials agree on it.
__host__ __device__ inline int red_rows(const ChannelMap& cm) {
  const int c4n = cm.Cp / 4, gpb = c4n < RED_NT ? c4n : RED_NT, ny = (c4n + gpb - 1) / gpb;
  // per-label criterion only (never the label count), so a label's sums round
  // identically however the labels are grouped (test_grouping_invariance);
  // < 10 blocks per label reproduces the old whole-grid rule at L = 125
  int rows = 512;
  while (rows > 32 && ny * ((cm.R + rows - 1) / rows) < 10) rows >>= 1;
  return rows;
}

PG_DEV float4 f4(float v) { return make_float4(v, v, v, v); }
PG_DEV float4 add4(float4 a, float4 b) { return make_float4(a.x + b.x, a.y + b.y, a.z + b.z, a.w + b.w); }
PG_DEV float4 ld4(const float* p) { return __ldg(reinterpret_cast<const float4*>(p)); }

// BN output before the activation, a = gamma * istd: ONE rounding point shared
// by bn_apply and the backward kernels that recompute the activation output
// from the pre-BN map (bit-identical to the y bn_apply wrote)
PG_DEV float bn_pre(float a, float x, float m, float b) { return __fmaf_rn(a, x - m, b); }
// the activation backward of a BN block can be taken from (x, BN coefficients)
// instead of a stored y when the derivative depends on y only through its sign
__host__ __device__ inline bool sign_act(int act) { return act == ACT_RELU || act == ACT_LRELU; }

// Per-channel sums over the rows of [L][R][Cp] maps.  Block = (label, chunk of
// red_rows(cm) rows, up to 256 float4 channel groups): a thread owns 4 channels
// (float4 loads along the row) and a row lane; the row lanes are combined in
// shared memory in a fixed order, and the chunk partials by the finalize
// kernels in chunk order (deterministic, no atomics).  Mode and activation are
// template parameters (straight-line loop bodies: the loads of several rows
// are issued together).  REC (RED_BN_BWD, ReLU / LeakyReLU): the activation
// output is recomputed from x and the BN coefficients (bn_pre) instead of read.
template <int MODE, int ACT, bool REC>
__global__ void __launch_bounds__(RED_NT) channel_reduce_kernel(ChannelMap cm, const float* __restrict__ x,
                                                                const float* __restrict__ gy,
                                                                const float* __restrict__ y,
                                                                const float* __restrict__ mean, float slope,
                                                                float* __restrict__ partial, float* __restrict__ g_out,
                                                                BnCoef bc) {
  const int l = blockIdx.z, chunk = blockIdx.x, nchunk = gridDim.x;
  const int c4n = cm.Cp / 4;
  const int gpb = c4n < RED_NT ? c4n : RED_NT;  // channel groups per block
  const int lanes = RED_NT / gpb;
  const int t = threadIdx.x, gi = t % gpb, lr = t / gpb;
  const int g = blockIdx.y * gpb + gi;
  float4 s0 = f4(0.f), s1 = f4(0.f), s2 = f4(0.f);
  if (g < c4n && lr < lanes) {
    const float4 mu = (MODE == RED_SQDEV || MODE == RED_BN_BWD) ? ld4(mean + (long long)l * cm.Cp + 4 * g) : f4(0.f);
    float ra[4] = {0.f, 0.f, 0.f, 0.f}, rm[4] = {0.f, 0.f, 0.f, 0.f}, rb[4] = {0.f, 0.f, 0.f, 0.f};
    if (REC) {
#pragma unroll
      for (int u = 0; u < 4; ++u) {
        const int c = 4 * g + u;
        const long long mc = (long long)l * cm.Cp + c;
        if (c < cm.C) {  // as bn_apply holds them (zero on padding channels)
          ra[u] = bc.gb[(long long)l * bc.gb_ls + c] * bc.istd[mc];
          rm[u] = mean[mc];
          rb[u] = bc.gb[(long long)l * bc.gb_ls + cm.C + c];
        }
      }
    }
    const long long base = (long long)l * cm.ls + 4 * g;
    const int rows = red_rows(cm);
    const int r_end = min(cm.R, (chunk + 1) * rows);
#pragma unroll 4
    for (int r = chunk * rows + lr; r < r_end; r += lanes) {
      const long long o = base + (long long)r * cm.Cp;
      if (MODE == RED_SUM) {
        s0 = add4(s0, ld4(x + o));
      } else if (MODE == RED_SQDEV) {
        const float4 v = ld4(x + o);
        const float dx = v.x - mu.x, dy = v.y - mu.y, dz = v.z - mu.z, dw = v.w - mu.w;
        s0 = add4(s0, make_float4(dx * dx, dy * dy, dz * dz, dw * dw));
      } else {
        const float4 g4 = ld4(gy + o);
        const float4 v = MODE == RED_BN_BWD ? ld4(x + o) : f4(0.f);
        float4 y4;
        if (REC)
          y4 = make_float4(act_fwd(ACT, bn_pre(ra[0], v.x, rm[0], rb[0]), slope),
                           act_fwd(ACT, bn_pre(ra[1], v.y, rm[1], rb[1]), slope),
                           act_fwd(ACT, bn_pre(ra[2], v.z, rm[2], rb[2]), slope),
                           act_fwd(ACT, bn_pre(ra[3], v.w, rm[3], rb[3]), slope));
        else
          y4 = ACT == ACT_NONE ? f4(0.f) : ld4(y + o);
        const float4 g1 = make_float4(act_bwd(ACT, g4.x, y4.x, slope), act_bwd(ACT, g4.y, y4.y, slope),
                                      act_bwd(ACT, g4.z, y4.z, slope), act_bwd(ACT, g4.w, y4.w, slope));
        s0 = add4(s0, g1);
        if (MODE == RED_ACT_G && g_out) *reinterpret_cast<float4*>(g_out + o) = g1;  // the activation backward itself
        if (MODE == RED_BN_BWD) {
          const float4 d = make_float4(v.x - mu.x, v.y - mu.y, v.z - mu.z, v.w - mu.w);
          s1 = add4(s1, make_float4(g1.x * d.x, g1.y * d.y, g1.z * d.z, g1.w * d.w));
          s2 = add4(s2, d);
        }
      }
    }
  }
  __shared__ float4 sm[3][RED_NT];
  sm[0][t] = s0;
  sm[1][t] = s1;
  sm[2][t] = s2;
  __syncthreads();
  if (lr != 0 || g >= c4n) return;
  const int nk = MODE == RED_BN_BWD ? 3 : 1;
  for (int k = 0; k < 3; ++k) {
    float4 acc = f4(0.f);
    if (k < nk)
      for (int i = 0; i < lanes; ++i) acc = add4(acc, sm[k][i * gpb + gi]);
    *reinterpret_cast<float4*>(partial + (((long long)l * nchunk + chunk) * 3 + k) * cm.Cp + 4 * g) = acc;
  }
}

PG_DEV float sum_partials(const ChannelMap& cm, const float* partial, int l, int k, int c) {
  const int nchunk = cm.nslot > 0 ? cm.nslot : (cm.R + red_rows(cm) - 1) / red_rows(cm);
  const int pk = cm.nslot > 0 ? 4 : 3;
  // sixteen loads in flight, added in chunk order (the sum is bit-identical to
  // the plain loop; the plain loop waited one load latency per chunk)
  const float* p = partial + ((long long)l * nchunk * pk + k) * cm.Cp + c;
  const long long step = (long long)pk * cm.Cp;
  float t = 0.f;
  int ch = 0;
  for (; ch + 16 <= nchunk; ch += 16) {
    float v[16];
#pragma unroll
    for (int u = 0; u < 16; ++u) v[u] = __ldg(p + (ch + u) * step);
#pragma unroll
    for (int u = 0; u < 16; ++u) t += v[u];
  }
  for (; ch < nchunk; ++ch) t += __ldg(p + ch * step);
  return t;
}

// The three sums k = 0, 1, 2 of sum_partials at once: 24 loads in flight
// instead of 8, each sum added in chunk order (bit-identical to three calls)
PG_DEV void sum_partials3(const ChannelMap& cm, const float* partial, int l, int c, float& t0, float& t1,
                          float& t2) {
  const int nchunk = cm.nslot > 0 ? cm.nslot : (cm.R + red_rows(cm) - 1) / red_rows(cm);
  const int pk = cm.nslot > 0 ? 4 : 3;
  const float* p = partial + (long long)l * nchunk * pk * cm.Cp + c;
  const long long step = (long long)pk * cm.Cp;
  t0 = t1 = t2 = 0.f;
  int ch = 0;
  for (; ch + 8 <= nchunk; ch += 8) {
    float v0[8], v1[8], v2[8];
#pragma unroll
    for (int u = 0; u < 8; ++u) {
      const float* q = p + (ch + u) * step;
      v0[u] = __ldg(q);
      v1[u] = __ldg(q + cm.Cp);
      v2[u] = __ldg(q + 2 * cm.Cp);
    }
#pragma unroll
    for (int u = 0; u < 8; ++u) {
      t0 += v0[u];
      t1 += v1[u];
      t2 += v2[u];
    }
  }
  for (; ch < nchunk; ++ch) {
    const float* q = p + ch * step;
    t0 += __ldg(q);
    t1 += __ldg(q + cm.Cp);
    t2 += __ldg(q + 2 * cm.Cp);
  }
}

// Per-slot {shift, sum d, sum d^2, n} (d = z - shift) -> mean and biased
// variance over all rows (network.cpp:171-184), running stats as
// bn_finalize_var.  The slots are re-expressed against one per-channel
// reference K (the first entry's shift, a value of the channel itself) and
// summed in f64: with d' = shift - K,  S1 += sum_d + n d',  S2 += sum_d2 +
// 2 d' sum_d + n d'^2  -- additions only (the per-slot Chan merge spent most of
// the kernel in f64 divisions).  Block = 32 channels x nl lanes: lane j sums
// the (slot, pack column) entries j, j + nl, ... in order, then a fixed
// pairwise tree adds the lanes (deterministic, independent of timing).
struct Sums {
  double n, s1, s2;
};
constexpr int FIN_MAX_LANES = 32;
template <int NP>  // npack when 1 or 4 (shift / mask instead of an integer division per entry), 0: runtime
__global__ void __launch_bounds__(32 * FIN_MAX_LANES) bn_stats_finalize_kernel(ChannelMap cm, const float* stat,
                                                                              float* mean, float* istd, float* running,
                                                                              long long run_ls, float eps, float mom,
                                                                              int update) {
  const int l = blockIdx.y, c = blockIdx.x * 32 + threadIdx.x, j = threadIdx.y, nl = blockDim.y;
  __shared__ Sums sm[FIN_MAX_LANES][32];
  Sums a{0.0, 0.0, 0.0};
  const int W = cm.Cp * cm.npack;  // statistic row width
  const float* base = stat + (long long)l * cm.nslot * 4 * W + (c < cm.Cp ? c : 0);
  const double K = base[3 * W] > 0.f ? (double)base[0] : 0.0;
  if (c < cm.Cp) {
    const int items = cm.nslot * cm.npack;
    for (int k0 = j; k0 < items; k0 += 4 * nl) {
      float e0[4], e1[4], e2[4], e3[4];
#pragma unroll
      for (int u = 0; u < 4; ++u) {  // four entries in flight before any is added
        const int k = k0 + u * nl;
        e0[u] = e1[u] = e2[u] = e3[u] = 0.f;
        if (k < items) {
          const int np = NP ? NP : cm.npack;
          const float* e = base + (long long)(k / np) * 4 * W + (k % np) * cm.Cp;
          e0[u] = e[0];
          e1[u] = e[W];
          e2[u] = e[2 * W];
          e3[u] = e[3 * W];
        }
      }
#pragma unroll
      for (int u = 0; u < 4; ++u) {
        const double nb = e3[u];
        if (nb <= 0.0) continue;
        const double d = (double)e0[u] - K, s1 = e1[u];
        a.n += nb;
        a.s1 += s1 + nb * d;
        a.s2 += (double)e2[u] + 2.0 * d * s1 + nb * d * d;
      }
    }
  }
  sm[j][threadIdx.x] = a;
  for (int h = nl / 2; h > 0; h >>= 1) {
    __syncthreads();
    if (j < h) {
      const Sums b = sm[j + h][threadIdx.x];
      a.n += b.n;
      a.s1 += b.s1;
      a.s2 += b.s2;
      sm[j][threadIdx.x] = a;
    }
  }
  if (j != 0 || c >= cm.Cp) return;
  const int i = l * cm.Cp + c;
  const double mu = a.n > 0.0 ? K + a.s1 / a.n : 0.0;
  const double var = a.n > 0.0 ? fmax(a.s2 - a.s1 * (a.s1 / a.n), 0.0) / a.n : 0.0;
  mean[i] = (float)mu;
  istd[i] = 1.f / sqrtf((float)var + eps);
  if (update && c < cm.C) {
    float* rm = running + (long long)l * run_ls;
    float* rv = rm + cm.C;
    const float m = (float)cm.R;
    const float unbias = m > 1.f ? m / (m - 1.f) : 1.f;
    rm[c] = (1.f - mom) * rm[c] + mom * (float)mu;
    rv[c] = (1.f - mom) * rv[c] + mom * (float)var * unbias;
  }
}

// [L][nslot][4][Cp] slot sums -> [L][1][4][Cp] (entries 0..2), fixed order
__global__ void slot_sum_kernel(ChannelMap cm, const float* stat, float* out) {
  const int l = blockIdx.y, c = blockIdx.x * 32 + threadIdx.x, j = threadIdx.y;
  __shared__ float sm[3][8][33];
  float t[3] = {0.f, 0.f, 0.f};
  const int W = cm.Cp * cm.npack;
  if (c < cm.Cp)
    for (int s = j; s < cm.nslot; s += 8)
      for (int q = 0; q < cm.npack; ++q) {
        const float* e = stat + ((long long)l * cm.nslot + s) * 4 * W + q * cm.Cp + c;
        t[0] += e[0];
        t[1] += e[W];
        t[2] += e[2 * W];
      }
  for (int k = 0; k < 3; ++k) sm[k][j][threadIdx.x] = t[k];
  __syncthreads();
  if (j < 3 && c < cm.Cp) {
    float r = 0.f;
    for (int k = 0; k < 8; ++k) r += sm[j][k][threadIdx.x];
    out[((long long)l * 4 + j) * cm.Cp + c] = r;
  }
}

__global__ void bn_finalize_mean_kernel(ChannelMap cm, const float* partial, float* mean) {
  int i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= cm.L * cm.Cp) return;
  int l = i / cm.Cp, c = i % cm.Cp;
  mean[i] = sum_partials(cm, partial, l, 0, c) / (float)cm.R;
}

__global__ void bn_finalize_var_kernel(ChannelMap cm, const float* partial, const float* mean, float* istd,
                                       float* running, long long run_ls, float eps, float mom, int update) {
  int i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= cm.L * cm.Cp) return;
  int l = i / cm.Cp, c = i % cm.Cp;
  const float m = (float)cm.R;
  float var = sum_partials(cm, partial, l, 0, c) / m;
  istd[i] = 1.f / sqrtf(var + eps);
  if (update && c < cm.C) {
    // running buffers: [mean[C]][var[C]] per label (reference buffer layout)
    float* rm = running + (long long)l * run_ls;
    float* rv = rm + cm.C;
    float unbias = m > 1.f ? m / (m - 1.f) : 1.f;
    rm[c] = (1.f - mom) * rm[c] + mom * mean[i];
    rv[c] = (1.f - mom) * rv[c] + mom * var * unbias;
  }
}

__global__ void bn_eval_stats_kernel(ChannelMap cm, const float* running, long long run_ls, float eps, float* mean,
                                     float* istd) {
  int i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= cm.L * cm.Cp) return;
  int l = i / cm.Cp, c = i % cm.Cp;
  if (c < cm.C) {
    const float* rm = running + (long long)l * run_ls;
    mean[i] = rm[c];
    istd[i] = 1.f / sqrtf(rm[cm.C + c] + eps);
  } else {
    mean[i] = 0.f;
    istd[i] = 0.f;
  }
}

// float4 over [L][R][Cp] (Cp % 4 == 0).  When the grid stride is a multiple of
// the row width (the usual case: Cp / 4 divides 256), each thread keeps one
// channel group for all its elements and holds its coefficients in registers.
template <int ACT>
__global__ void __launch_bounds__(256) bn_apply_kernel(ChannelMap cm, const float* __restrict__ x,
                                                       const float* __restrict__ mean, const float* __restrict__ istd,
                                                       const float* __restrict__ gb, long long gb_ls, int act,
                                                       float slope, float* __restrict__ y) {
  const int c4n = cm.Cp / 4;
  const long long per = (long long)cm.R * c4n;
  const int l = blockIdx.y;
  const float* gamma = gb + (long long)l * gb_ls;
  const float* beta = gamma + cm.C;
  const long long stride = (long long)gridDim.x * blockDim.x;
  const long long q0 = blockIdx.x * (long long)blockDim.x + threadIdx.x;
  if (stride % c4n == 0) {
    const int c0 = (int)(q0 % c4n) * 4;
    float a[4], m[4], bb[4];
#pragma unroll
    for (int u = 0; u < 4; ++u) {
      const int c = c0 + u;
      const long long mc = (long long)l * cm.Cp + c;
      const bool ok = c < cm.C;
      a[u] = ok ? gamma[c] * istd[mc] : 0.f;
      m[u] = ok ? mean[mc] : 0.f;
      bb[u] = ok ? beta[c] : 0.f;
    }
    const float* xl = x + (long long)l * cm.ls;
    float* yl = y + (long long)l * cm.ls;
    auto apply = [&](float4 v) {
      const float r[4] = {v.x, v.y, v.z, v.w};
      float o4[4];
#pragma unroll
      for (int u = 0; u < 4; ++u)
        o4[u] = c0 + u < cm.C ? act_fwd(ACT, bn_pre(a[u], r[u], m[u], bb[u]), slope) : 0.f;
      return make_float4(o4[0], o4[1], o4[2], o4[3]);
    };
    long long q = q0;
    // four independent float4 loads in flight per thread
    for (; q + 3 * stride < per; q += 4 * stride) {
      float4 v[4];
#pragma unroll
      for (int k = 0; k < 4; ++k) v[k] = ld4(xl + (q + k * stride) * 4);
#pragma unroll
      for (int k = 0; k < 4; ++k) *reinterpret_cast<float4*>(yl + (q + k * stride) * 4) = apply(v[k]);
    }
    for (; q < per; q += stride) *reinterpret_cast<float4*>(yl + q * 4) = apply(ld4(xl + q * 4));
    return;
  }
  for (long long q = q0; q < per; q += stride) {
    const long long o = (long long)l * cm.ls + q * 4;
    const int c0 = (int)((q * 4) % cm.Cp);
    float4 v = *reinterpret_cast<const float4*>(x + o);
    float r[4] = {v.x, v.y, v.z, v.w};
#pragma unroll
    for (int u = 0; u < 4; ++u) {
      int c = c0 + u;
      if (c < cm.C) {
        long long mc = (long long)l * cm.Cp + c;
        r[u] = act_fwd(ACT, bn_pre(gamma[c] * istd[mc], r[u], mean[mc], beta[c]), slope);
      } else {
        r[u] = 0.f;
      }
    }
    *reinterpret_cast<float4*>(y + o) = make_float4(r[0], r[1], r[2], r[3]);
  }
}

// coef[l][c][3] = {gamma*istd, 2*dvar/m, dmean/m}
__global__ void bn_bwd_finalize_kernel(ChannelMap cm, const float* partial, const float* istd, const float* gb,
                                       long long gb_ls, float* dgb, long long dgb_ls, float* dbias, long long dbias_ls,
                                       int accumulate, int train, float* coef) {
  int i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= cm.L * cm.Cp) return;
  int l = i / cm.Cp, c = i % cm.Cp;
  float* cf = coef + (long long)i * 3;
  if (c >= cm.C) {
    cf[0] = cf[1] = cf[2] = 0.f;
    return;
  }
  const float m = (float)cm.R;
  float S1, S2, S3;
  sum_partials3(cm, partial, l, c, S1, S2, S3);
  const float is = istd[i];
  const float gamma = gb[(long long)l * gb_ls + c];
  float dg = S2 * is, db = S1;
  float a = gamma * is, dvar = 0.f, dmean = 0.f;
  if (train) {
    dvar = gamma * S2 * (-0.5f) * is * is * is;
    dmean = -gamma * S1 * is + dvar * (-2.f / m) * S3;
  }
  cf[0] = a;
  cf[1] = 2.f * dvar / m;
  cf[2] = dmean / m;
  if (dgb) {
    float* dgp = dgb + (long long)l * dgb_ls;
    if (accumulate) {
      dgp[c] += dg;
      dgp[cm.C + c] += db;
    } else {
      dgp[c] = dg;
      dgp[cm.C + c] = db;
    }
  }
  if (dbias) {
    // sum over rows of gz, in closed form from the channel sums
    float sgz = a * S1 + cf[1] * S3 + dmean;
    float* d = dbias + (long long)l * dbias_ls + c;
    *d = accumulate ? *d + sgz : sgz;
  }
}

// Per-channel coefficients of one float4 channel group for bn_bwd_apply.
struct BwdCoef4 {
  float cf0[4], cf1[4], cf2[4], m[4], ra[4], rm[4], rb[4];
};
PG_DEV void load_bwd_coef(BwdCoef4& k, const ChannelMap& cm, int l, int c0, const float* mean, const float* coef,
                          const BnCoef& bc, bool rec) {
#pragma unroll
  for (int u = 0; u < 4; ++u) {
    const int c = c0 + u;
    const long long mc = (long long)l * cm.Cp + c;
    k.cf0[u] = coef[mc * 3];
    k.cf1[u] = coef[mc * 3 + 1];
    k.cf2[u] = coef[mc * 3 + 2];
    k.m[u] = mean[mc];
    const bool ok = rec && c < cm.C;
    // as bn_apply holds them (a = gamma istd, zero coefficients on padding channels)
    k.ra[u] = ok ? bc.gb[(long long)l * bc.gb_ls + c] * bc.istd[mc] : 0.f;
    k.rm[u] = ok ? k.m[u] : 0.f;
    k.rb[u] = ok ? bc.gb[(long long)l * bc.gb_ls + cm.C + c] : 0.f;
  }
}
PG_DEV float4 bwd_apply4(const BwdCoef4& k, int act, float slope, bool rec, float4 g4, float4 y4, float4 x4) {
  const float g[4] = {g4.x, g4.y, g4.z, g4.w}, xx[4] = {x4.x, x4.y, x4.z, x4.w};
  float yy[4] = {y4.x, y4.y, y4.z, y4.w}, r[4];
#pragma unroll
  for (int u = 0; u < 4; ++u) {
    if (rec) yy[u] = act_fwd(act, bn_pre(k.ra[u], xx[u], k.rm[u], k.rb[u]), slope);
    const float g1 = act_bwd(act, g[u], yy[u], slope);
    r[u] = g1 * k.cf0[u] + k.cf1[u] * (xx[u] - k.m[u]) + k.cf2[u];
  }
  return make_float4(r[0], r[1], r[2], r[3]);
}

// gz = act_bwd(gy, y) gamma istd + 2 dvar (x - mean) / m + dmean / m.  With
// bc.istd (ReLU / LeakyReLU) y is recomputed from x instead of read.  When the
// grid stride is a multiple of the row width each thread keeps one channel
// group and its coefficients in registers, four float4 loads of each map in flight.
__global__ void __launch_bounds__(256) bn_bwd_apply_kernel(ChannelMap cm, const float* __restrict__ gy,
                                                           const float* __restrict__ y, const float* __restrict__ x,
                                                           const float* __restrict__ mean,
                                                           const float* __restrict__ coef, int act, float slope,
                                                           float* __restrict__ gz, BnCoef bc) {
  const int c4n = cm.Cp / 4;
  const long long per = (long long)cm.R * c4n;
  const int l = blockIdx.y;
  const bool rec = bc.istd != nullptr && sign_act(act);
  const bool ld_y = act != ACT_NONE && !rec;
  const long long stride = (long long)gridDim.x * blockDim.x;
  const long long q0 = blockIdx.x * (long long)blockDim.x + threadIdx.x;
  const float* gl = gy + (long long)l * cm.ls;
  const float* yl = y + (long long)l * cm.ls;
  const float* xl = x + (long long)l * cm.ls;
  float* ol = gz + (long long)l * cm.ls;
  const float4 z4 = make_float4(0.f, 0.f, 0.f, 0.f);
  BwdCoef4 k;
  if (stride % c4n == 0) {
    load_bwd_coef(k, cm, l, (int)(q0 % c4n) * 4, mean, coef, bc, rec);
    long long q = q0;
    for (; q + 3 * stride < per; q += 4 * stride) {
      float4 g4[4], y4[4], x4[4];
#pragma unroll
      for (int j = 0; j < 4; ++j) {
        const long long o = (q + j * stride) * 4;
        g4[j] = ld4(gl + o);
        x4[j] = ld4(xl + o);
        y4[j] = ld_y ? ld4(yl + o) : z4;
      }
#pragma unroll
      for (int j = 0; j < 4; ++j)
        *reinterpret_cast<float4*>(ol + (q + j * stride) * 4) = bwd_apply4(k, act, slope, rec, g4[j], y4[j], x4[j]);
    }
    for (; q < per; q += stride) {
      const long long o = q * 4;
      *reinterpret_cast<float4*>(ol + o) =
          bwd_apply4(k, act, slope, rec, ld4(gl + o), ld_y ? ld4(yl + o) : z4, ld4(xl + o));
    }
    return;
  }
  for (long long q = q0; q < per; q += stride) {
    const long long o = q * 4;
    load_bwd_coef(k, cm, l, (int)(q % c4n) * 4, mean, coef, bc, rec);
    *reinterpret_cast<float4*>(ol + o) =
        bwd_apply4(k, act, slope, rec, ld4(gl + o), ld_y ? ld4(yl + o) : z4, ld4(xl + o));
  }
}

template <int ACT>
__global__ void __launch_bounds__(256) act_bwd_kernel(ChannelMap cm, const float* __restrict__ gy,
                                                      const float* __restrict__ y, float slope, float* g) {
  const long long per = (long long)cm.R * cm.Cp / 4;
  const int l = blockIdx.y;
  const float* gl = gy + (long long)l * cm.ls;
  const float* yl = y + (long long)l * cm.ls;
  float* ol = g + (long long)l * cm.ls;
  const long long stride = (long long)gridDim.x * blockDim.x;
  auto bwd = [&](float4 g4, float4 y4) {
    return make_float4(act_bwd(ACT, g4.x, y4.x, slope), act_bwd(ACT, g4.y, y4.y, slope),
                       act_bwd(ACT, g4.z, y4.z, slope), act_bwd(ACT, g4.w, y4.w, slope));
  };
  long long q = blockIdx.x * (long long)blockDim.x + threadIdx.x;
  for (; q + 3 * stride < per; q += 4 * stride) {  // four float4 of each map in flight
    float4 g4[4], y4[4];
#pragma unroll
    for (int j = 0; j < 4; ++j) {
      g4[j] = *reinterpret_cast<const float4*>(gl + (q + j * stride) * 4);
      y4[j] = *reinterpret_cast<const float4*>(yl + (q + j * stride) * 4);
    }
#pragma unroll
    for (int j = 0; j < 4; ++j) *reinterpret_cast<float4*>(ol + (q + j * stride) * 4) = bwd(g4[j], y4[j]);
  }
  for (; q < per; q += stride)
    *reinterpret_cast<float4*>(ol + q * 4) =
        bwd(*reinterpret_cast<const float4*>(gl + q * 4), *reinterpret_cast<const float4*>(yl + q * 4));
}

__global__ void bias_finalize_kernel(ChannelMap cm, const float* partial, float* dbias, long long dbias_ls,
                                     int accumulate) {
  int i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= cm.L * cm.C) return;
  int l = i / cm.C, c = i % cm.C;
  float s = sum_partials(cm, partial, l, 0, c);
  float* d = dbias + (long long)l * dbias_ls + c;
  *d = accumulate ? *d + s : s;
}

// ---- losses: one block per label, fixed-order tree in double ----
__device__ double block_sum(double v, double* sm) {
  const int t = threadIdx.x;
  sm[t] = v;
  __syncthreads();
  for (int w = blockDim.x / 2; w > 0; w >>= 1) {
    if (t < w) sm[t] += sm[t + w];
    __syncthreads();
  }
  double r = sm[0];
  __syncthreads();
  return r;
}

PG_DEV double clampd(double p, double c) { return fmin(fmax(p, c), 1.0 - c); }
PG_DEV bool inside(double p, double c) { return p > c && p < 1.0 - c; }

__global__ void loss_d_kernel(int B, const float* pr, const float* pf, int ps, double clamp, float* gr, float* gf,
                              double* rep) {
  extern __shared__ double sm[];
  const int l = blockIdx.x, i = threadIdx.x;
  double lr = 0, lf = 0, mr = 0, mf = 0;
  if (i < B) {
    long long o = ((long long)l * B + i) * ps;
    double a = pr[o], b = pf[o];
    lr = log(clampd(a, clamp));
    lf = log(1.0 - clampd(b, clamp));
    mr = a;
    mf = b;
    gr[o] = inside(a, clamp) ? (float)(-0.5 / ((double)B * a)) : 0.f;
    gf[o] = inside(b, clamp) ? (float)(0.5 / ((double)B * (1.0 - b))) : 0.f;
    for (int c = 1; c < ps; ++c) gr[o + c] = gf[o + c] = 0.f;
  }
  double slr = block_sum(lr, sm), slf = block_sum(lf, sm), smr = block_sum(mr, sm), smf = block_sum(mf, sm);
  if (i == 0) {
    rep[l * 4 + 0] = -0.5 * slr / B - 0.5 * slf / B;
    rep[l * 4 + 2] = smr / B;
    rep[l * 4 + 3] = smf / B;
  }
}

__global__ void loss_g_kernel(int B, const float* pf, int ps, double clamp, float* g, double* rep) {
  extern __shared__ double sm[];
  const int l = blockIdx.x, i = threadIdx.x;
  double lg = 0;
  if (i < B) {
    long long o = ((long long)l * B + i) * ps;
    double b = pf[o];
    lg = log(clampd(b, clamp));
    g[o] = inside(b, clamp) ? (float)(-0.5 / ((double)B * b)) : 0.f;
    for (int c = 1; c < ps; ++c) g[o + c] = 0.f;
  }
  double s = block_sum(lg, sm);
  if (i == 0) rep[l * 4 + 1] = 0.5 * s / B;
}

// ---- Adam ----
__global__ void nonfinite_kernel(long long P, const float* __restrict__ g, int* flags) {
  const int l = blockIdx.y;
  const float* gl = g + (long long)l * P;
  bool bad = false;
  for (long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x; i < P / 4; i += (long long)gridDim.x * blockDim.x) {
    float4 v = reinterpret_cast<const float4*>(gl)[i];
    bad |= !isfinite(v.x) || !isfinite(v.y) || !isfinite(v.z) || !isfinite(v.w);
  }
  if (__any_sync(0xffffffffu, bad) && (threadIdx.x & 31) == 0) atomicOr(flags + l, 1);
}

__global__ void adam_tick_kernel(int L, const int* flags, long long* t) {
  int l = blockIdx.x * blockDim.x + threadIdx.x;
  if (l < L && !flags[l]) t[l] += 1;
}

__global__ void adam_kernel(long long P, float* __restrict__ p, const float* __restrict__ g, float* __restrict__ m,
                            float* __restrict__ v, const long long* t, const int* flags, float lr, double b1d,
                            double b2d, float eps) {
  const int l = blockIdx.y;
  if (flags[l]) return;  // rejected step: state untouched (optim.cpp:25)
  // 1 - beta from the f64 betas: (1.f - (float)0.999) carries a 1.3e-5 relative error
  const float b1 = (float)b1d, b2 = (float)b2d, ob1 = (float)(1.0 - b1d), ob2 = (float)(1.0 - b2d);
  __shared__ float c12[2];
  if (threadIdx.x == 0) {
    // bias corrections from the f64 betas, as std::pow in optim.cpp:30-31
    double tt = (double)t[l];
    c12[0] = (float)(1.0 - pow(b1d, tt));
    c12[1] = (float)(1.0 - pow(b2d, tt));
  }
  __syncthreads();
  const float c1 = c12[0], c2 = c12[1];
  const long long off = (long long)l * P;
  float4* p4 = reinterpret_cast<float4*>(p + off);
  const float4* g4 = reinterpret_cast<const float4*>(g + off);
  float4* m4 = reinterpret_cast<float4*>(m + off);
  float4* v4 = reinterpret_cast<float4*>(v + off);
  for (long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x; i < P / 4; i += (long long)gridDim.x * blockDim.x) {
    float4 gg = g4[i], mm = m4[i], vv = v4[i], pp = p4[i];
    float ga[4] = {gg.x, gg.y, gg.z, gg.w}, ma[4] = {mm.x, mm.y, mm.z, mm.w}, va[4] = {vv.x, vv.y, vv.z, vv.w},
          pa[4] = {pp.x, pp.y, pp.z, pp.w};
#pragma unroll
    for (int u = 0; u < 4; ++u) {
      ma[u] = b1 * ma[u] + ob1 * ga[u];
      va[u] = b2 * va[u] + ob2 * ga[u] * ga[u];
      pa[u] -= lr * (ma[u] / c1) / (sqrtf(va[u] / c2) + eps);
    }
    m4[i] = make_float4(ma[0], ma[1], ma[2], ma[3]);
    v4[i] = make_float4(va[0], va[1], va[2], va[3]);
    p4[i] = make_float4(pa[0], pa[1], pa[2], pa[3]);
  }
}

// ---- data movement ----
__global__ void gather_real_kernel(int B, const int* __restrict__ idx, const float* __restrict__ data,
                                   long long data_ls, long long sample, int Cp, int C, float* __restrict__ out) {
  const int l = blockIdx.z, b = blockIdx.y;
  const long long src = (long long)l * data_ls + (long long)idx[l * B + b] * sample;
  const long long dst = ((long long)l * B + b) * sample;
  // 32-bit index arithmetic (a sample is < 2^31 floats; the 64-bit modulo was
  // a software division per float4)
  const int n4 = (int)(sample / 4);
#pragma unroll 4
  for (int q = blockIdx.x * blockDim.x + threadIdx.x; q < n4; q += gridDim.x * blockDim.x) {
    float4 v = __ldg(reinterpret_cast<const float4*>(data + src) + q);
    int c0 = (4 * q) % Cp;
    float r[4] = {v.x, v.y, v.z, v.w};
#pragma unroll
    for (int u = 0; u < 4; ++u) r[u] = (c0 + u < C) ? r[u] * 2.f - 1.f : 0.f;
    reinterpret_cast<float4*>(out + dst)[q] = make_float4(r[0], r[1], r[2], r[3]);
  }
}

__global__ void nchw01_to_nhwc_kernel(long long N, int C, int H, int W, int Cp, const float* in, float* out, int map) {
  long long total = N * H * W * Cp;
  for (long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x; i < total; i += (long long)gridDim.x * blockDim.x) {
    int c = (int)(i % Cp);
    long long pix = i / Cp;
    int x = (int)(pix % W);
    long long t = pix / W;
    int y = (int)(t % H);
    long long n = t / H;
    float v = c < C ? in[((n * C + c) * H + y) * W + x] : 0.f;
    out[i] = (map && c < C) ? v * 2.f - 1.f : v;
  }
}

__global__ void nhwc_to_nchw01_kernel(long long N, int C, int H, int W, int Cp, const float* in, float* out) {
  long long total = N * C * H * W;
  for (long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x; i < total; i += (long long)gridDim.x * blockDim.x) {
    int x = (int)(i % W);
    long long t = i / W;
    int y = (int)(t % H);
    t /= H;
    int c = (int)(t % C);
    long long n = t / C;
    out[i] = (in[((n * H + y) * W + x) * Cp + c] + 1.f) * 0.5f;
  }
}

__global__ void fill_kernel(float* p, long long n, float v) {
  for (long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x; i < n; i += (long long)gridDim.x * blockDim.x)
    p[i] = v;
}

unsigned grid_for(long long work, int per_block, unsigned cap = 148 * 16) {
  long long g = (work + per_block - 1) / per_block;
  if (g < 1) g = 1;
  if (g > cap) g = cap;
  return (unsigned)g;
}

}  // namespace

int reduce_chunks(const ChannelMap& cm) { return (cm.R + red_rows(cm) - 1) / red_rows(cm); }
// sized for the smallest chunk, so any map with at most cm.R rows fits
size_t reduce_partial_floats(const ChannelMap& cm) { return (size_t)cm.L * ((cm.R + 31) / 32) * 3 * cm.Cp; }

cudaError_t launch_channel_reduce(const ChannelMap& cm, int mode, const float* x, const float* gy, const float* y,
                                  const float* mean, int act, float slope, float* partial, cudaStream_t st,
                                  float* g_out, BnCoef bc) {
  cudaEvent_t t0_ = timing_start(st);
  if (cm.Cp % 4) return cudaErrorInvalidValue;
  const int c4n = cm.Cp / 4, gpb = c4n < RED_NT ? c4n : RED_NT;
  dim3 grid(reduce_chunks(cm), (c4n + gpb - 1) / gpb, cm.L);
  const bool rec = mode == RED_BN_BWD && bc.istd != nullptr && sign_act(act);
#define PG_RED(M, A, R) channel_reduce_kernel<M, A, R><<<grid, RED_NT, 0, st>>>(cm, x, gy, y, mean, slope, partial, g_out, bc)
#define PG_RED_ACTS(M)                          \
  switch (act) {                                \
    case ACT_RELU: PG_RED(M, ACT_RELU, false); break;       \
    case ACT_LRELU: PG_RED(M, ACT_LRELU, false); break;     \
    case ACT_TANH: PG_RED(M, ACT_TANH, false); break;       \
    case ACT_SIGMOID: PG_RED(M, ACT_SIGMOID, false); break; \
    default: PG_RED(M, ACT_NONE, false); break;             \
  }
  switch (mode) {
    case RED_SUM: PG_RED(RED_SUM, ACT_NONE, false); break;
    case RED_SQDEV: PG_RED(RED_SQDEV, ACT_NONE, false); break;
    case RED_BN_BWD:
      if (rec && act == ACT_RELU) PG_RED(RED_BN_BWD, ACT_RELU, true);
      else if (rec) PG_RED(RED_BN_BWD, ACT_LRELU, true);
      else PG_RED_ACTS(RED_BN_BWD);
      break;
    case RED_ACT_G: PG_RED_ACTS(RED_ACT_G); break;
    default: return cudaErrorInvalidValue;
  }
#undef PG_RED_ACTS
#undef PG_RED
  cudaError_t r_ = launched();
  timing_stop(t0_, st, "hbm channel_reduce bytes=" + std::to_string((long long)((long long)cm.L * cm.R * cm.Cp * (mode == RED_ACT_G ? 12 : mode == RED_BN_BWD ? (rec ? 8 : 12) : 4))));
  return r_;
}

cudaError_t launch_bn_finalize_mean(const ChannelMap& cm, const float* partial, float* mean, cudaStream_t st) {
  int n = cm.L * cm.Cp;
  bn_finalize_mean_kernel<<<(n + 255) / 256, 256, 0, st>>>(cm, partial, mean);
  return launched();
}

cudaError_t launch_bn_finalize_var(const ChannelMap& cm, const float* partial, const float* mean, float* istd,
                                   float* running, long long run_ls, float eps, float momentum, int update_running,
                                   cudaStream_t st) {
  int n = cm.L * cm.Cp;
  bn_finalize_var_kernel<<<(n + 255) / 256, 256, 0, st>>>(cm, partial, mean, istd, running, run_ls, eps, momentum,
                                                          update_running);
  return launched();
}

cudaError_t launch_bn_eval_stats(const ChannelMap& cm, const float* running, long long run_ls, float eps, float* mean,
                                 float* istd, cudaStream_t st) {
  int n = cm.L * cm.Cp;
  bn_eval_stats_kernel<<<(n + 255) / 256, 256, 0, st>>>(cm, running, run_ls, eps, mean, istd);
  return launched();
}

cudaError_t launch_bn_apply(const ChannelMap& cm, const float* x, const float* mean, const float* istd,
                            const float* gamma_beta, long long gb_ls, int act, float slope, float* y, cudaStream_t st) {
  cudaEvent_t t0_ = timing_start(st);
  // few fat threads: each keeps its channel coefficients in registers and
  // streams ~16 float4 (8 blocks per SM over all labels)
  const long long per = (long long)cm.R * cm.Cp / 4;
  const unsigned cap = std::max(1u, 148u * 8u / (unsigned)std::max(1, cm.L));
  dim3 grid(grid_for(per, 256 * 16, cap), cm.L);
  switch (act) {
    case ACT_RELU: bn_apply_kernel<ACT_RELU><<<grid, 256, 0, st>>>(cm, x, mean, istd, gamma_beta, gb_ls, act, slope, y); break;
    case ACT_LRELU: bn_apply_kernel<ACT_LRELU><<<grid, 256, 0, st>>>(cm, x, mean, istd, gamma_beta, gb_ls, act, slope, y); break;
    case ACT_TANH: bn_apply_kernel<ACT_TANH><<<grid, 256, 0, st>>>(cm, x, mean, istd, gamma_beta, gb_ls, act, slope, y); break;
    case ACT_SIGMOID:
      bn_apply_kernel<ACT_SIGMOID><<<grid, 256, 0, st>>>(cm, x, mean, istd, gamma_beta, gb_ls, act, slope, y);
      break;
    default: bn_apply_kernel<ACT_NONE><<<grid, 256, 0, st>>>(cm, x, mean, istd, gamma_beta, gb_ls, act, slope, y); break;
  }
  cudaError_t r_ = launched();
  timing_stop(t0_, st, "hbm bn_apply bytes=" + std::to_string((long long)(8LL * cm.L * cm.R * cm.Cp)));
  return r_;
}

// lanes per channel: about 8 entries per lane, 4..32 (few entries: small blocks)
static int fin_lanes(const ChannelMap& cm) {
  int nl = 4;
  while (nl < FIN_MAX_LANES && nl * 8 < cm.nslot * cm.npack) nl <<= 1;
  return nl;
}

cudaError_t launch_bn_stats_finalize(const ChannelMap& cm, const float* stat, float* mean, float* istd, float* running,
                                     long long run_ls, float eps, float momentum, int update_running, cudaStream_t st) {
  if (cm.nslot <= 0) return cudaErrorInvalidValue;
  cudaEvent_t t0_ = timing_start(st);
  const dim3 grid((cm.Cp + 31) / 32, cm.L), block(32, fin_lanes(cm));
  if (cm.npack == 1)
    bn_stats_finalize_kernel<1><<<grid, block, 0, st>>>(cm, stat, mean, istd, running, run_ls, eps, momentum,
                                                        update_running);
  else if (cm.npack == 4)
    bn_stats_finalize_kernel<4><<<grid, block, 0, st>>>(cm, stat, mean, istd, running, run_ls, eps, momentum,
                                                        update_running);
  else
    bn_stats_finalize_kernel<0><<<grid, block, 0, st>>>(cm, stat, mean, istd, running, run_ls, eps, momentum,
                                                        update_running);
  cudaError_t r_ = launched();
  timing_stop(t0_, st, "hbm bn_stats_finalize bytes=" + std::to_string(16LL * cm.L * cm.nslot * cm.Cp * cm.npack));
  return r_;
}

cudaError_t launch_slot_sum(const ChannelMap& cm, const float* stat, float* out, cudaStream_t st) {
  if (cm.nslot <= 0) return cudaErrorInvalidValue;
  slot_sum_kernel<<<dim3((cm.Cp + 31) / 32, cm.L), dim3(32, 8), 0, st>>>(cm, stat, out);
  return launched();
}

cudaError_t launch_bn_bwd_finalize(const ChannelMap& cm, const float* partial, const float* istd,
                                   const float* gamma_beta, long long gb_ls, float* dgamma_beta, long long dgb_ls,
                                   float* dbias, long long dbias_ls, int accumulate, int train, float* coef,
                                   cudaStream_t st) {
  int n = cm.L * cm.Cp;
  bn_bwd_finalize_kernel<<<(n + 255) / 256, 256, 0, st>>>(cm, partial, istd, gamma_beta, gb_ls, dgamma_beta, dgb_ls,
                                                          dbias, dbias_ls, accumulate, train, coef);
  return launched();
}

cudaError_t launch_bn_bwd_apply(const ChannelMap& cm, const float* gy, const float* y, const float* x,
                                const float* mean, const float* coef, int act, float slope, float* gz,
                                cudaStream_t st, BnCoef bc) {
  cudaEvent_t t0_ = timing_start(st);
  const long long per = (long long)cm.R * cm.Cp / 4;
  const unsigned cap = std::max(1u, 148u * 8u / (unsigned)std::max(1, cm.L));
  dim3 grid(grid_for(per, 256 * 16, cap), cm.L);
  bn_bwd_apply_kernel<<<grid, 256, 0, st>>>(cm, gy, y, x, mean, coef, act, slope, gz, bc);
  cudaError_t r_ = launched();
  timing_stop(t0_, st, "hbm bn_bwd_apply bytes=" + std::to_string((long long)((bc.istd ? 12LL : 16LL) * cm.L * cm.R * cm.Cp)));
  return r_;
}

cudaError_t launch_act_bwd(const ChannelMap& cm, const float* gy, const float* y, int act, float slope, float* g,
                           cudaStream_t st) {
  cudaEvent_t t0_ = timing_start(st);
  const long long per = (long long)cm.R * cm.Cp / 4;
  const unsigned cap = std::max(1u, 148u * 8u / (unsigned)std::max(1, cm.L));
  dim3 grid(grid_for(per, 256 * 16, cap), cm.L);
  switch (act) {
    case ACT_RELU: act_bwd_kernel<ACT_RELU><<<grid, 256, 0, st>>>(cm, gy, y, slope, g); break;
    case ACT_LRELU: act_bwd_kernel<ACT_LRELU><<<grid, 256, 0, st>>>(cm, gy, y, slope, g); break;
    case ACT_TANH: act_bwd_kernel<ACT_TANH><<<grid, 256, 0, st>>>(cm, gy, y, slope, g); break;
    case ACT_SIGMOID: act_bwd_kernel<ACT_SIGMOID><<<grid, 256, 0, st>>>(cm, gy, y, slope, g); break;
    default: act_bwd_kernel<ACT_NONE><<<grid, 256, 0, st>>>(cm, gy, y, slope, g); break;
  }
  cudaError_t r_ = launched();
  timing_stop(t0_, st, "hbm act_bwd bytes=" + std::to_string((long long)(12LL * cm.L * cm.R * cm.Cp)));
  return r_;
}

cudaError_t launch_bias_finalize(const ChannelMap& cm, const float* partial, float* dbias, long long dbias_ls,
                                 int accumulate, cudaStream_t st) {
  int n = cm.L * cm.C;
  bias_finalize_kernel<<<(n + 255) / 256, 256, 0, st>>>(cm, partial, dbias, dbias_ls, accumulate);
  return launched();
}

static int pow2_at_least(int b) {
  int t = 32;
  while (t < b) t <<= 1;
  return t;
}

cudaError_t launch_loss_d(int L, int B, const float* p_real, const float* p_fake, int pstride, double clamp,
                          float* g_real, float* g_fake, double* report, cudaStream_t st) {
  int t = pow2_at_least(B);
  loss_d_kernel<<<L, t, t * sizeof(double), st>>>(B, p_real, p_fake, pstride, clamp, g_real, g_fake, report);
  return launched();
}

cudaError_t launch_loss_g(int L, int B, const float* p_fake, int pstride, double clamp, float* g, double* report,
                          cudaStream_t st) {
  int t = pow2_at_least(B);
  loss_g_kernel<<<L, t, t * sizeof(double), st>>>(B, p_fake, pstride, clamp, g, report);
  return launched();
}

cudaError_t launch_nonfinite_check(int L, long long P, const float* grads, int* flags, cudaStream_t st) {
  cudaEvent_t t0_ = timing_start(st);
  dim3 grid(grid_for(P / 4, 256, 64), L);
  nonfinite_kernel<<<grid, 256, 0, st>>>(P, grads, flags);
  cudaError_t r_ = launched();
  timing_stop(t0_, st, "hbm nonfinite bytes=" + std::to_string((long long)(4LL * L * P)));
  return r_;
}

cudaError_t launch_adam_tick(int L, const int* flags, long long* t, cudaStream_t st) {
  adam_tick_kernel<<<(L + 127) / 128, 128, 0, st>>>(L, flags, t);
  return launched();
}

cudaError_t launch_adam(int L, long long P, float* params, const float* grads, float* m, float* v,
                        const long long* t, const int* flags, float lr, double b1, double b2, float eps,
                        cudaStream_t st) {
  cudaEvent_t t0_ = timing_start(st);
  dim3 grid(grid_for(P / 4, 256, 256), L);
  adam_kernel<<<grid, 256, 0, st>>>(P, params, grads, m, v, t, flags, lr, b1, b2, eps);
  cudaError_t r_ = launched();
  timing_stop(t0_, st, "hbm adam bytes=" + std::to_string((long long)(28LL * L * P)));
  return r_;
}

cudaError_t launch_gather_real(int L, int B, const int* idx, const float* data, long long data_ls, long long sample,
                               int Cp, int C, float* out, cudaStream_t st) {
  cudaEvent_t t0_ = timing_start(st);
  dim3 grid(grid_for(sample / 4, 256 * 4, 16), B, L);  // ~4 float4 per thread
  gather_real_kernel<<<grid, 256, 0, st>>>(B, idx, data, data_ls, sample, Cp, C, out);
  cudaError_t r_ = launched();
  timing_stop(t0_, st, "hbm gather_real bytes=" + std::to_string((long long)(8LL * L * B * sample)));
  return r_;
}

cudaError_t launch_nchw01_to_nhwc(long long N, int C, int H, int W, int Cp, const float* in, float* out,
                                  cudaStream_t st, int map2x1) {
  nchw01_to_nhwc_kernel<<<grid_for(N * H * W * Cp, 256, 148 * 8), 256, 0, st>>>(N, C, H, W, Cp, in, out, map2x1);
  return launched();
}

cudaError_t launch_nhwc_to_nchw01(long long N, int C, int H, int W, int Cp, const float* in, float* out,
                                  cudaStream_t st) {
  nhwc_to_nchw01_kernel<<<grid_for(N * C * H * W, 256, 148 * 8), 256, 0, st>>>(N, C, H, W, Cp, in, out);
  return launched();
}

cudaError_t launch_fill(float* p, long long n, float v, cudaStream_t st) {
  fill_kernel<<<grid_for(n, 256, 148 * 8), 256, 0, st>>>(p, n, v);
  return launched();
}

// Parity instrumentation (not on the training path unless capture is enabled):
// the ReLU / LeakyReLU masks of an activation output map y [L][B][H][W][Cp],
// as bytes in the reference's [B][C][H][W] order, with act_bwd's convention
// (ReLU: y > 0, LeakyReLU: y >= 0 -- equal to the reference's x > 0 / x >= 0).
__global__ void mask_capture_kernel(int B, int H, int W, int C, int Cp, long long ls, const float* __restrict__ y,
                                    int leaky, unsigned char* __restrict__ out, long long out_ls) {
  const int l = blockIdx.y;
  const long long per = (long long)B * C * H * W;
  const float* yl = y + l * ls;
  unsigned char* ol = out + l * out_ls;
  for (long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x; i < per; i += (long long)gridDim.x * blockDim.x) {
    long long r = i;
    const int x = (int)(r % W);
    r /= W;
    const int yy = (int)(r % H);
    r /= H;
    const int c = (int)(r % C);
    const long long b = r / C;
    const float v = yl[((b * H + yy) * W + x) * Cp + c];
    ol[i] = leaky ? (v >= 0.f) : (v > 0.f);
  }
}

cudaError_t launch_mask_capture(int L, int B, int H, int W, int C, int Cp, long long ls, const float* y, int act,
                                unsigned char* out, long long out_ls, cudaStream_t st) {
  dim3 grid(grid_for((long long)B * C * H * W, 256, 256), L);
  mask_capture_kernel<<<grid, 256, 0, st>>>(B, H, W, C, Cp, ls, y, act == ACT_LRELU ? 1 : 0, out, out_ls);
  return launched();
}

}  // namespace pg
