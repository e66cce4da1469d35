// Device-resident network for a group of L labels that share one
// architecture: the B200 counterpart of partgan::Network / forward / backward
// (/root/reference/proj/include/partgan/network.hpp:20-107,
//  src/network.cpp:308-480).
//
// The reference layer list is compiled into fused *blocks*:
//     [Reshape] Linear [Reshape] [BatchNorm] [Activation]
// where Linear is Dense, Conv2d or ConvTranspose2d.  A block is one implicit
// GEMM (bias + activation in its epilogue when there is no BatchNorm), plus
// the BatchNorm statistics / apply kernels when there is one.  Reshapes next
// to a Dense are absorbed into a permutation of its weights, so every device
// map stays NHWC with channels padded to a multiple of 4.
//
// Parameters live in one [L][P] fp32 arena per network (weights in a
// GEMM-friendly layout, see import_params); gradients and Adam moments are
// arenas of the same shape, so Adam is one pass over contiguous memory.
// Import/export convert to and from the reference's flat f64 layout.
#pragma once

#include <cstdint>
#include <memory>
#include <stdexcept>
#include <string>
#include <vector>

#include "kernels.hpp"

namespace pg {

enum class LK { Dense, Conv, ConvT, BN, Upsample, Dropout, ReLU, LReLU, Tanh, Sigmoid, Reshape };

struct LayerSpec {
  LK kind = LK::ReLU;
  long in = 0, out = 0, k = 3, s = 1, p = 0;
  double eps = 1e-5, momentum = 0.1, slope = 0.2, rate = 0.5;
  long scale = 2;
  std::vector<long> target;
};

std::vector<LayerSpec> parse_layers(const std::string& text);
std::vector<long> parse_shape(const std::string& text);
long ref_param_count(const LayerSpec& l);
long ref_buffer_count(const LayerSpec& l);
std::vector<long> ref_out_shape(const LayerSpec& l, const std::vector<long>& in, size_t idx);
const char* layer_name(LK k);

inline long pad4(long x) { return (x + 3) / 4 * 4; }

// per-sample device map: H x W x Cp (C valid); flat features are H = W = 1.
struct Map {
  long H = 1, W = 1, C = 0, Cp = 0;
  long numel() const { return H * W * Cp; }
};

struct Block {
  LK lin = LK::Dense;
  LayerSpec L;                 // the linear layer
  bool has_bn = false;
  LayerSpec bn;
  int act = ACT_NONE;
  float slope = 0.f;
  bool in_from_chw = false;    // Reshape [C,H,W] -> [F] absorbed before a Dense
  bool out_to_chw = false;     // Reshape [F] -> [C,H,W] absorbed after a Dense
  std::vector<long> in_chw, out_chw;
  Map in, out;                 // device maps
  ConvGeo geo;                 // B filled per call
  // device arena offsets (floats, per label)
  long long off_w = 0, n_w = 0, off_b = 0, n_b = 0, off_bn = 0, off_run = 0;
  // reference offsets
  long ref_lin = 0, ref_bn = 0, ref_buf = 0;
  int first_layer = 0, last_layer = 0;
  bool bias_per_bn_channel() const { return has_bn && !out_to_chw; }
};

struct DeviceBuf {
  float* p = nullptr;
  size_t n = 0;
  DeviceBuf() = default;
  explicit DeviceBuf(size_t count);
  ~DeviceBuf();
  DeviceBuf(const DeviceBuf&) = delete;
  DeviceBuf& operator=(const DeviceBuf&) = delete;
  DeviceBuf(DeviceBuf&& o) noexcept : p(o.p), n(o.n) { o.p = nullptr; o.n = 0; }
  DeviceBuf& operator=(DeviceBuf&& o) noexcept;
};

struct Trace {
  // act[i] = input of block i (act[0] may alias an external buffer), act[nb] = output
  std::vector<float*> act;
  std::vector<DeviceBuf> own;   // owned activation buffers (index i >= 1)
  std::vector<DeviceBuf> pre;   // pre-BatchNorm linear output per block (BN blocks)
  std::vector<DeviceBuf> mean, istd;
  bool train = true;  // mode of the forward that filled it (backward's BatchNorm form)
};

class DevNet {
 public:
  DevNet(const std::string& spec, const std::vector<long>& in_shape, int L, int max_batch, int math);

  int L() const { return L_; }
  int blocks() const { return static_cast<int>(blocks_.size()); }
  const Block& block(int i) const { return blocks_[static_cast<size_t>(i)]; }
  const Map& in_map() const { return blocks_.front().in; }
  const Map& out_map() const { return blocks_.back().out; }
  long long P() const { return P_; }
  long ref_params() const { return ref_P_; }
  long ref_buffers() const { return ref_Bf_; }
  const std::vector<long>& ref_out_shape() const { return ref_shapes_.back(); }
  const std::vector<long>& ref_in_shape() const { return ref_shapes_.front(); }
  const std::vector<LayerSpec>& layers() const { return layers_; }
  int math() const { return math_; }
  void set_math(int m) { math_ = m; }

  // arenas [L][P] / [L][Bf]
  DeviceBuf params, grads, adam_m, adam_v, running;
  long long Bf() const { return Bf_; }

  // reference-layout (f64) <-> device arena (fp32) for one label.
  void import_params(const double* ref, float* dev_label) const;
  void export_params(const float* dev_label, double* ref) const;
  void import_buffers(const double* ref, float* dev_label) const;
  void export_buffers(const float* dev_label, double* ref) const;
  // initial parameters exactly as build_network draws them (network.cpp:308-343)
  std::vector<double> init_ref_params(uint64_t seed, double init_std) const;
  std::vector<double> init_ref_buffers() const;

  Trace make_trace(bool alias_input) const;
  // train: batch statistics (+ running update when update_running); eval: running stats.
  void forward(Trace& t, int B, bool train, bool update_running, cudaStream_t st);
  // gy: gradient w.r.t. the network output map [L][B][out]; writes param grads
  // into `grads` (accumulating when accumulate) unless param_grads is false;
  // writes the input gradient into gx when non-null.
  void backward(Trace& t, int B, const float* gy, bool param_grads, bool accumulate, float* gx, cudaStream_t st);

  size_t max_map_floats() const;  // largest [L][B_max][map] among all block maps

 private:
  int L_, Bmax_, math_;
  std::vector<LayerSpec> layers_;
  std::vector<std::vector<long>> ref_shapes_;
  std::vector<long> ref_off_, ref_boff_;
  std::vector<Block> blocks_;
  long long P_ = 0, Bf_ = 0;
  long ref_P_ = 0, ref_Bf_ = 0;
  DeviceBuf partial_, coef_, gscratch_[2], gz_, stat_;

  ConvGeo geo_for(const Block& b, int B) const;
  GemmArgs linear_args(const Block& b, int B, const float* x, float* y, bool with_epilogue) const;
  void linear_fwd(const Block& b, int B, const float* x, float* y, bool with_epilogue, cudaStream_t st);
  float* stat_buf(size_t floats, cudaStream_t st);  // grow-only buffer for fused GEMM statistics
  template <class F>
  void map_params(const Block& b, F f) const;  // f(ref_index, dev_index) for every real parameter
};

void check_cuda(cudaError_t e, const char* what);

}  // namespace pg
