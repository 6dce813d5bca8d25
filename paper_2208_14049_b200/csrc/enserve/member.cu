// DeviceMember: plans, weights and launches of one member on one GPU.
#include "enserve/member.hpp"

#include <cuda_bf16.h>

#include <algorithm>
#include <cmath>
#include <cstdlib>
#include <cstring>

#include "../cuda/aux_kernels.cuh"
#include "../cuda/conv_kernel.cuh"
#include "../cuda/conv_rows_kernel.cuh"
#include "../cuda/dense_kernel.cuh"
#include "../cuda/fp32_kernels.cuh"
#include "../cuda/mlp_kernel.cuh"
#include "../cuda/mlp_pair_kernel.cuh"
#include "../cuda/mlp_tmem_kernel.cuh"

namespace enserve {

namespace {

[[noreturn]] void fail_cuda(cudaError_t e, const char* what) {
  cudaGetLastError();
  throw DeviceError(std::string(what) + ": " + cudaGetErrorString(e));
}

#define M_CUDA(call)                                        \
  do {                                                      \
    cudaError_t m_err_ = (call);                            \
    if (m_err_ != cudaSuccess) fail_cuda(m_err_, #call);    \
  } while (0)

#define M_LAUNCH(call)                                                       \
  do {                                                                       \
    if ((call) != 0) fail_cuda(cudaGetLastError(), "kernel launch " #call); \
  } while (0)

struct OnDev {
  int prev = 0;
  explicit OnDev(int d) {
    cudaGetDevice(&prev);
    M_CUDA(cudaSetDevice(d));
  }
  ~OnDev() { cudaSetDevice(prev); }
};

bool env_is(const char* name, const char* value) {
  const char* v = std::getenv(name);
  return v && std::strcmp(v, value) == 0;
}

// Hidden dense layers: the SM-pair kernel (half of every W chunk per SM) unless
// ES_DENSE_KERNEL=single; the single-SM kernel when no pair plan exists.
bool plan_dense(int K, int N, es::DenseLayout* d) {
  if (!env_is("ES_DENSE_KERNEL", "single") && es::dense_pair_plan(K, N, true, d)) return true;
  return es::dense_plan(K, N, true, d);
}

}  // namespace

struct DeviceMember::Impl {
  ModelSpec model;
  int batch = 1;
  int C = 1;
  std::vector<std::pair<int, int>> dims;  // (fan_in, fan_out) per weight matrix
  // Dense: too wide for a fused head -- the hidden layer through the dense
  // kernel, the last layer in its logits mode.
  enum class Head { Synthetic, SwapAB, Tmem, Pair, Dense, Fp32 } head = Head::Synthetic;
  es::Mlp2Layout plan_swapab{};
  es::MlpTLayout plan_tmem{};
  es::MlpPLayout plan_pair{};
  std::vector<es::DenseLayout> dense;  // dense-kernel layers, in order
  std::vector<int> dense_layer;        // their weight-matrix index
  es::DenseLayout logits{};            // Head::Dense: the last layer
  bool cnn = false;
  es::ConvLayout conv{};  // CNN: the convolution stack (layers 0 and 1)
  // CNN-s shape: a samples-in-M kernel (conv_rows_kernel.cuh): 2 = the input
  // sweep (default), 1 = the row windows (ES_CONV_SCHEDULE=rows), 0 = neither.
  int conv_rows = 0;
  void* weights = nullptr;
  std::vector<std::size_t> w_off, b_off;  // per layer
  std::vector<float> conv_b1, conv_b2;      // CNN: conv biases, host copies
  // Outputs of the leading layers, bf16 [rows][width], indexed like X.
  std::vector<void*> act;
  std::vector<int> act_width;
  std::vector<std::size_t> act_rows;
  int act_elem = 2;  // bytes per activation: bf16, or fp32 (Head::Fp32)
};

DeviceMember::~DeviceMember() {
  if (!impl_) return;
  cudaSetDevice(device_);
  if (impl_->weights) cudaFree(impl_->weights);
  for (void* p : impl_->act) cudaFree(p);
  delete impl_;
}

std::string DeviceMember::schedule() const {
  if (!impl_) return "unloaded";
  switch (impl_->head) {
    case Impl::Head::Pair: return "pair";
    case Impl::Head::Tmem: return "tmem";
    case Impl::Head::SwapAB: return "swapab";
    case Impl::Head::Dense: return "dense";
    case Impl::Head::Fp32: return "fp32";
    default: return "synthetic";
  }
}

bool DeviceMember::fp32() const { return impl_ && impl_->head == Impl::Head::Fp32; }

bool DeviceMember::load(int device, const ModelSpec& model, int batch, bool fp32) {
  device_ = device;
  impl_ = new Impl();
  Impl& I = *impl_;
  I.model = model;
  I.batch = batch;
  I.C = model.output_width;
  if (model.arch.kind == MemberArch::Kind::Synthetic) return true;
  const MemberArch& a = model.arch;
  I.dims = a.layer_dims();
  const int L = static_cast<int>(I.dims.size());
  if (L < 2) throw SpecError(model.name + ": a member needs at least two layers");
  if (fp32) return load_fp32(device);
  if (a.kind == MemberArch::Kind::CNN) {
    // Leading layers: the fused convolution stack, bf16 [(S/P)^2 * c2] rows out.
    I.cnn = true;
    const char* cs = std::getenv("ES_CONV_SCHEDULE");  // tests: "tap" | "split" | "rows"
    const bool rows = cs && std::strcmp(cs, "rows") == 0;
    if (rows) cs = nullptr;
    const int sched = cs && std::strcmp(cs, "tap") == 0 ? 1 : cs && std::strcmp(cs, "split") == 0 ? 2 : 0;
    // Default for the CNN-s shape: samples in M (measured on B200);
    // "tap" / "split" select the positions-in-M kernel for comparison.
    I.conv_rows = !cs && es::conv_rows_supported(a.widths[0], a.widths[1], a.widths[2], a.widths[3])
                      ? (rows ? 1 : 2)
                      : 0;
    // ES_CONV_SCHEDULE=split falls back to tap where the shape has no split plan.
    if (!es::conv_plan(a.widths[0], a.widths[1], a.widths[2], a.widths[3], &I.conv, sched) &&
        !(sched == 2 && es::conv_plan(a.widths[0], a.widths[1], a.widths[2], a.widths[3], &I.conv, 1)))
      throw SpecError(model.name + ": CNN shape has no tile plan (patch 4, image side a "
                      "multiple of 4 up to 52, c1 in {32, 64, 128}, c2 a multiple of 32 up to 256)");
    I.act_width.push_back(I.dims[2].first);
  } else {
    // Leading layers: tcgen05 dense layers with a bf16 output.
    for (int l = 0; l < L - 2; ++l) {
      es::DenseLayout d;
      if (!plan_dense(I.dims[l].first, I.dims[l].second, &d))
        throw SpecError(model.name + ": leading layer " + std::to_string(I.dims[l].first) + "->" +
                        std::to_string(I.dims[l].second) +
                        " has no tile plan (input width a multiple of 8, output width a "
                        "multiple of 128 up to 512)");
      I.dense.push_back(d);
      I.dense_layer.push_back(l);
      I.act_width.push_back(I.dims[l].second);
    }
  }
  // Fused head over the last two layers.
  const int K = I.dims[L - 2].first, H = I.dims[L - 2].second, C = I.dims[L - 1].second;
  const char* pick = std::getenv("ES_MLP_KERNEL");
  const std::string want = pick ? pick : "";
  const bool pair_ok = (want.empty() || want == "pair") && es::mlpp_plan(K, H, C, batch, &I.plan_pair);
  const bool tmem_ok = (want.empty() || want == "tmem") && es::mlpt_plan(K, H, C, batch, &I.plan_tmem);
  // Measured on B200 (tools/time_members.py, 4M samples): the single-SM TMEM
  // schedule wins up to H = 384 (784-384-10: 2.64 vs 2.73 ms; 784-256-10:
  // 1.75 vs 1.76 ms; 1568-128-10: 2.29 vs 2.79 ms); SM pairs (half the W1
  // ingress per SM) from H = 512 up, and they alone cover hidden passes.
  if (pair_ok && (!tmem_ok || !want.empty() || H >= 512))
    I.head = Impl::Head::Pair;
  else if (tmem_ok)
    I.head = Impl::Head::Tmem;
  else if ((want.empty() || want == "swapab") && es::mlp2_plan(K, H, C, batch, &I.plan_swapab))
    I.head = Impl::Head::SwapAB;
  else if (want.empty() || want == "dense") {
    // Hidden layer wider than one SM's TMEM: no fused head.
    es::DenseLayout d;
    if (!plan_dense(K, H, &d) || !es::dense_logits_plan(H, C, &I.logits))
      throw SpecError(model.name + ": layers " + std::to_string(K) + "->" + std::to_string(H) +
                      "->" + std::to_string(C) + " have no tile plan");
    I.dense.push_back(d);
    I.dense_layer.push_back(L - 2);
    I.act_width.push_back(H);
    I.head = Impl::Head::Dense;
  } else {
    return false;  // the requested schedule does not fit one SM
  }

  OnDev on(device);
  auto up = [](std::size_t x) { return (x + 255) / 256 * 256; };
  std::size_t off = 0;
  for (int l = 0; l < L; ++l) {
    I.w_off.push_back(off);
    off += up(static_cast<std::size_t>(I.dims[l].first) * I.dims[l].second * 2);
    I.b_off.push_back(off);
    off += up(static_cast<std::size_t>(I.dims[l].second) * 4);
  }
  bytes_ = off;
  cudaError_t e = cudaMalloc(&I.weights, bytes_);
  if (e == cudaErrorMemoryAllocation) {
    cudaGetLastError();
    I.weights = nullptr;
    return false;
  }
  M_CUDA(e);
  uint8_t* base = static_cast<uint8_t*>(I.weights);
  for (int l = 0; l < L; ++l) {
    const int fi = I.dims[l].first, fo = I.dims[l].second;
    const float limit = static_cast<float>(std::sqrt(6.0 / static_cast<double>(fi + fo)));
    M_LAUNCH(es::generate_dense_layer(a.weight_seed, l, fi, fo, limit,
                                      reinterpret_cast<__nv_bfloat16*>(base + I.w_off[l]),
                                      reinterpret_cast<float*>(base + I.b_off[l]), 0));
  }
  I.act.assign(I.act_width.size(), nullptr);
  I.act_rows.assign(I.act_width.size(), 0);
  M_CUDA(cudaDeviceSynchronize());
  if (I.cnn) {  // conv2 bias travels by value in the launch parameters (conv_kernel.cuh)
    I.conv_b2.resize(static_cast<std::size_t>(I.dims[1].second));
    M_CUDA(cudaMemcpy(I.conv_b2.data(), base + I.b_off[1], I.conv_b2.size() * sizeof(float),
                      cudaMemcpyDeviceToHost));
    I.conv_b1.resize(static_cast<std::size_t>(I.dims[0].second));
    M_CUDA(cudaMemcpy(I.conv_b1.data(), base + I.b_off[0], I.conv_b1.size() * sizeof(float),
                      cudaMemcpyDeviceToHost));
  }
  return true;
}

std::vector<std::string> DeviceMember::kernel_names() const {
  std::vector<std::string> n;
  if (!impl_) return n;
  const Impl& I = *impl_;
  if (I.head == Impl::Head::Synthetic) return {"synthetic_member_kernel"};
  if (I.head == Impl::Head::Fp32) {
    if (I.cnn) n.push_back("f32_conv_kernel");
    for (std::size_t l = I.cnn ? 2 : 0; l < I.dims.size(); ++l) n.push_back("f32_dense_kernel");
    return n;
  }
  if (I.cnn)
    n.push_back(I.conv_rows == 2 ? "conv_sweep_sm100" : I.conv_rows ? "conv_rows_sm100" : I.conv.split ? "conv_stack_sm100[split]" : "conv_stack_sm100[tap]");
  for (const auto& d : I.dense) n.push_back(d.pair ? "dense_pair_sm100" : "dense_sm100");
  if (env_is("ES_MEMBER_KERNEL", "simt") && I.head != Impl::Head::Dense) {
    n.push_back("mlp2_simt_kernel");
    return n;
  }
  switch (I.head) {
    case Impl::Head::Pair: n.push_back("member_mlp2_pair_sm100"); break;
    case Impl::Head::Tmem: n.push_back("member_mlp2_tmem_sm100"); break;
    case Impl::Head::SwapAB: n.push_back("member_mlp2_sm100"); break;
    default: n.push_back("dense_sm100[logits]"); break;
  }
  return n;
}

bool DeviceMember::supports_claim() const {
  if (!impl_) return false;
  if (env_is("ES_MEMBER_KERNEL", "simt")) return false;
  return impl_->head != Impl::Head::SwapAB;
}

int DeviceMember::forward(const void* x, long long nb, int seg_size, long long s0, long long s1,
                          float* out, int grid, cudaStream_t stream, const cudaEvent_t* marks,
                          const es::ClaimedRun* claim) {
  Impl& I = *impl_;
  if (s1 <= s0 || nb == 0) return 0;
  if (claim && !supports_claim()) throw Error(I.model.name + ": schedule cannot follow a claim");
  auto mark = [&](int i) {
    if (marks) M_CUDA(cudaEventRecord(marks[i], stream));
  };
  if (I.head == Impl::Head::Synthetic) {
    M_LAUNCH(es::synthetic_member_launch(I.model.id, I.C, seg_size, s0, s1, nb, out, stream, claim));
    mark(0);
    return 1;
  }
  const uint8_t* base = static_cast<const uint8_t*>(I.weights);
  const int L = static_cast<int>(I.dims.size());
  const long long r0 = s0 * seg_size, r1 = std::min<long long>(s1 * seg_size, nb);
  int launches = 0;
  const void* cur = x;
  for (std::size_t l = 0; l < I.act.size(); ++l) {
    if (I.act_rows[l] < static_cast<std::size_t>(nb)) {
      cudaFree(I.act[l]);
      I.act[l] = nullptr;
      M_CUDA(cudaMalloc(&I.act[l], static_cast<std::size_t>(nb) * I.act_width[l] * I.act_elem));
      I.act_rows[l] = static_cast<std::size_t>(nb);
    }
  }
  if (I.head == Impl::Head::Fp32)
    return forward_fp32(static_cast<const float*>(x), nb, r0, r1, out, grid, stream, marks, claim);
  if (I.cnn && I.conv_rows) {
    es::ConvRowsArgs c;
    c.row_begin = r0;
    c.row_end = r1;
    c.claim = claim;
    c.w1 = base + I.w_off[0];
    c.w2 = base + I.w_off[1];
    std::copy(I.conv_b1.begin(), I.conv_b1.end(), c.b1c);
    std::copy(I.conv_b2.begin(), I.conv_b2.end(), c.b2c);
    c.out = I.act[0];
    M_LAUNCH(I.conv_rows == 2 ? es::conv_sweep_launch(c, cur, nb, grid, stream)
                              : es::conv_rows_launch(c, cur, nb, grid, stream));
    mark(launches++);
    cur = I.act[0];
  } else if (I.cnn) {
    es::ConvArgs c;
    c.L = I.conv;
    c.row_begin = r0;
    c.row_end = r1;
    c.claim = claim;
    c.w1 = base + I.w_off[0];
    c.b1 = reinterpret_cast<const float*>(base + I.b_off[0]);
    c.w2 = base + I.w_off[1];
    c.b2 = reinterpret_cast<const float*>(base + I.b_off[1]);
    std::copy(I.conv_b2.begin(), I.conv_b2.end(), c.b2c);
    c.out = I.act[0];
    M_LAUNCH(es::conv_launch(c, cur, nb, grid, stream));
    mark(launches++);
    cur = I.act[0];
  }
  for (std::size_t i = 0; i < I.dense.size(); ++i) {
    const int l = I.dense_layer[i];
    void* y = I.act[i + (I.cnn ? 1 : 0)];
    es::DenseArgs d;
    d.L = I.dense[i];
    d.row_begin = r0;
    d.row_end = r1;
    d.claim = claim;
    d.bias = reinterpret_cast<const float*>(base + I.b_off[l]);
    M_LAUNCH(d.L.pair ? es::dense_pair_launch(d, cur, nb, base + I.w_off[l], y, grid, stream)
                      : es::dense_launch(d, cur, nb, base + I.w_off[l], y, grid, stream));
    mark(launches++);
    cur = y;
  }
  if (I.head == Impl::Head::Dense) {
    es::DenseArgs d;
    d.L = I.logits;
    d.row_begin = r0;
    d.row_end = r1;
    d.claim = claim;
    d.bias = reinterpret_cast<const float*>(base + I.b_off[L - 1]);
    d.logits = out;
    M_LAUNCH(es::dense_launch(d, cur, nb, base + I.w_off[L - 1], nullptr, grid, stream));
    mark(launches);
    return launches + 1;
  }
  const int h = L - 2;  // head layers h, h+1
  const float* b1 = reinterpret_cast<const float*>(base + I.b_off[h]);
  const float* b2 = reinterpret_cast<const float*>(base + I.b_off[h + 1]);
  const void* w1 = base + I.w_off[h];
  const void* w2 = base + I.w_off[h + 1];
  if (env_is("ES_MEMBER_KERNEL", "simt")) {
    M_LAUNCH(es::mlp2_simt_launch(static_cast<const __nv_bfloat16*>(cur), nb, I.dims[h].first,
                                  static_cast<const __nv_bfloat16*>(w1), b1, I.dims[h].second,
                                  static_cast<const __nv_bfloat16*>(w2), b2, I.C, r0, r1, out,
                                  stream));
    mark(launches);
    return launches + 1;
  }
  switch (I.head) {
    case Impl::Head::Pair: {
      es::MlpPArgs p;
      p.L = I.plan_pair;
      p.b = I.batch;
      p.seg_size = seg_size;
      p.seg_begin = s0;
      p.seg_end = s1;
      p.nb = nb;
      p.bias1 = b1;
      p.bias2 = b2;
      p.out = out;
      p.claim = claim;
      M_LAUNCH(es::mlpp_launch(p, cur, w1, w2, grid, stream));
      break;
    }
    case Impl::Head::Tmem: {
      es::MlpTArgs t;
      t.L = I.plan_tmem;
      t.b = I.batch;
      t.seg_size = seg_size;
      t.seg_begin = s0;
      t.seg_end = s1;
      t.nb = nb;
      t.bias1 = b1;
      t.bias2 = b2;
      t.out = out;
      t.claim = claim;
      M_LAUNCH(es::mlpt_launch(t, cur, w1, w2, grid, stream));
      break;
    }
    default: {
      es::Mlp2Args s;
      s.L = I.plan_swapab;
      s.b = I.batch;
      s.seg_size = seg_size;
      s.seg_begin = s0;
      s.seg_end = s1;
      s.nb = nb;
      s.bias1 = b1;
      s.bias2 = b2;
      s.out = out;
      M_LAUNCH(es::mlp2_launch(s, cur, w1, w2, grid, stream));
      break;
    }
  }
  mark(launches);
  return launches + 1;
}

bool DeviceMember::load_fp32(int device) {
  Impl& I = *impl_;
  const MemberArch& a = I.model.arch;
  const int L = static_cast<int>(I.dims.size());
  I.head = Impl::Head::Fp32;
  I.act_elem = 4;
  if (a.kind == MemberArch::Kind::CNN) {
    I.cnn = true;
    if (!es::f32_conv_supported(a.widths[0], a.widths[1], a.widths[2], a.widths[3]))
      throw SpecError(I.model.name + ": CNN shape too large for the fp32 convolution kernel");
    for (int l = 2; l < L - 1; ++l) I.act_width.push_back(I.dims[l].first);
    I.act_width.push_back(I.dims[L - 1].first);
  } else {
    for (int l = 0; l < L - 1; ++l) I.act_width.push_back(I.dims[l].second);
  }
  OnDev on(device);
  auto up = [](std::size_t x) { return (x + 255) / 256 * 256; };
  std::size_t off = 0;
  for (int l = 0; l < L; ++l) {
    I.w_off.push_back(off);
    off += up(static_cast<std::size_t>(I.dims[l].first) * I.dims[l].second * 4);
    I.b_off.push_back(off);
    off += up(static_cast<std::size_t>(I.dims[l].second) * 4);
  }
  bytes_ = off;
  cudaError_t e = cudaMalloc(&I.weights, bytes_);
  if (e == cudaErrorMemoryAllocation) {
    cudaGetLastError();
    I.weights = nullptr;
    return false;
  }
  M_CUDA(e);
  uint8_t* base = static_cast<uint8_t*>(I.weights);
  for (int l = 0; l < L; ++l) {
    const int fi = I.dims[l].first, fo = I.dims[l].second;
    const float limit = static_cast<float>(std::sqrt(6.0 / static_cast<double>(fi + fo)));
    M_LAUNCH(es::generate_dense_layer_f32(a.weight_seed, l, fi, fo, limit,
                                          reinterpret_cast<float*>(base + I.w_off[l]),
                                          reinterpret_cast<float*>(base + I.b_off[l]), 0));
  }
  I.act.assign(I.act_width.size(), nullptr);
  I.act_rows.assign(I.act_width.size(), 0);
  M_CUDA(cudaDeviceSynchronize());
  return true;
}

// fp32 chain: [conv stack] then every dense layer (ReLU but the last), the
// last writing fp32 logits at the rows' offsets.
int DeviceMember::forward_fp32(const float* x, long long nb, long long r0, long long r1, float* out,
                               int grid, cudaStream_t stream, const cudaEvent_t* marks,
                               const es::ClaimedRun* claim) {
  Impl& I = *impl_;
  const uint8_t* base = static_cast<const uint8_t*>(I.weights);
  const int L = static_cast<int>(I.dims.size());
  auto W = [&](int l) { return reinterpret_cast<const float*>(base + I.w_off[l]); };
  auto B = [&](int l) { return reinterpret_cast<const float*>(base + I.b_off[l]); };
  int launches = 0;
  const float* cur = x;
  int l = 0;
  if (I.cnn) {
    const MemberArch& a = I.model.arch;
    es::F32ConvArgs c;
    c.x = x;
    c.w1 = W(0);
    c.b1 = B(0);
    c.w2 = W(1);
    c.b2 = B(1);
    c.out = static_cast<float*>(I.act[0]);
    c.S = a.widths[0];
    c.P = a.widths[1];
    c.c1 = a.widths[2];
    c.c2 = a.widths[3];
    c.row_begin = r0;
    c.row_end = r1;
    c.claim = claim;
    M_LAUNCH(es::f32_conv_launch(c, grid, stream));
    if (marks) M_CUDA(cudaEventRecord(marks[launches], stream));
    ++launches;
    cur = c.out;
    l = 2;
  }
  for (; l < L; ++l) {
    es::F32DenseArgs d;
    d.x = cur;
    d.w = W(l);
    d.b = B(l);
    d.K = I.dims[l].first;
    d.N = I.dims[l].second;
    d.relu = l < L - 1;
    d.y = l == L - 1 ? out : static_cast<float*>(I.act[I.cnn ? l - 1 : l]);
    d.row_begin = r0;
    d.row_end = r1;
    d.claim = claim;
    M_LAUNCH(es::f32_dense_launch(d, grid, stream));
    if (marks) M_CUDA(cudaEventRecord(marks[launches], stream));
    ++launches;
    cur = d.y;
  }
  return launches;
}

}  // namespace enserve
