// The drop-in classes of include/p2r/{tensor,model,optim}.hpp: the reference's
// Tensor / GradTape / primitives / Model / AdamW / LrSchedule / moe_dispatch
// (/root/reference/proj/core/include/p2r/*.hpp) over this build's engine and
// kernels. Primitives upload their operands, run the fp32 kernels of
// csrc/prims.cu and download the result (the reference's host-memory tensor
// semantics); the model layer keeps activations and parameters on the device and
// copies them to the host only when a caller reads them.
#include <cuda_runtime.h>

#include <algorithm>
#include <cmath>
#include <cstring>
#include <map>
#include <mutex>
#include <stdexcept>

#include "p2r/engine.hpp"
#include "p2r/optim.hpp"
#include "p2r_cuda.h"

namespace p2r {

// ---------------------------------------------------------------- device views
// A device-resident tensor value: an engine activation (kind 1), the logits (2),
// the loss (3) or a parameter (4). The host copy is cached per engine version.
struct DeviceView {
  Engine* engine = nullptr;
  std::shared_ptr<void> keep;  // keeps the engine alive
  const float* ptr = nullptr;
  int rows = 0, cols = 0, ld = 0;
  int kind = 0;
  int param = -1;  // kind 4: engine parameter index
  mutable std::uint64_t host_version = 0;
  bool host_dirty = false;  // kind 4: the host copy was handed out writable
};

namespace {
enum { kAct = 1, kLogits = 2, kLoss = 3, kParam = 4 };

std::size_t count_of(const std::vector<int>& shape) {
  std::size_t n = 1;
  for (int d : shape) {
    if (d < 0) throw std::invalid_argument("tensor: negative dimension");
    n *= static_cast<std::size_t>(d);
  }
  return n;
}

void download(const DeviceView& v, std::vector<float>& host) {
  host.resize(static_cast<std::size_t>(v.rows) * v.cols);
  cuda_check(cudaDeviceSynchronize(), "sync");
  if (v.kind == kParam) {
    v.engine->get_param(v.param, host.data());
  } else {
    cuda_check(cudaMemcpy2D(host.data(), static_cast<std::size_t>(v.cols) * 4, v.ptr, static_cast<std::size_t>(v.ld) * 4,
                            static_cast<std::size_t>(v.cols) * 4, v.rows, cudaMemcpyDeviceToHost),
               "d2h tensor");
  }
}

// ---- device scratch for the primitive layer
struct Dev {
  void* p = nullptr;
  std::size_t bytes = 0;
  Dev() = default;
  explicit Dev(std::size_t n) : bytes(n) {
    if (n) cuda_check(cudaMalloc(&p, n), "cudaMalloc");
  }
  ~Dev() {
    if (p) cudaFree(p);
  }
  Dev(const Dev&) = delete;
  Dev& operator=(const Dev&) = delete;
  Dev(Dev&& o) noexcept : p(o.p), bytes(o.bytes) {
    o.p = nullptr;
    o.bytes = 0;
  }
  float* f() const { return static_cast<float*>(p); }
  int* i() const { return static_cast<int*>(p); }
};

Dev up(const float* h, std::size_t n) {
  Dev d(std::max<std::size_t>(n, 1) * 4);
  if (n) cuda_check(cudaMemcpy(d.p, h, n * 4, cudaMemcpyHostToDevice), "h2d");
  return d;
}
Dev up_i(const int* h, std::size_t n) {
  Dev d(std::max<std::size_t>(n, 1) * 4);
  if (n) cuda_check(cudaMemcpy(d.p, h, n * 4, cudaMemcpyHostToDevice), "h2d");
  return d;
}
Dev up_u8(const std::uint8_t* h, std::size_t n) {
  Dev d(std::max<std::size_t>(n, 1));
  if (n) cuda_check(cudaMemcpy(d.p, h, n, cudaMemcpyHostToDevice), "h2d");
  return d;
}
Dev zeros_dev(std::size_t n) {
  Dev d(std::max<std::size_t>(n, 1) * 4);
  cuda_check(cudaMemset(d.p, 0, std::max<std::size_t>(n, 1) * 4), "memset");
  return d;
}
void down(const Dev& d, float* h, std::size_t n) {
  if (n) cuda_check(cudaMemcpy(h, d.p, n * 4, cudaMemcpyDeviceToHost), "d2h");
}
void ok(int st, const char* what) { p2r_check(st, what); }

void require_2d(const Tensor& t, const char* op) {
  if (t.ndim() != 2) throw std::invalid_argument(std::string(op) + ": expected 2-D tensor");
}

// the gradient buffer of `t` gets `g` added on the device. Tape closures hold
// (const) shallow copies; a tensor that requires grad carries its shared gradient
// buffer from creation, so writing through the copy reaches the caller's tensor.
void add_grad(const Tensor& tc, const Dev& g, std::size_t n) {
  Tensor& t = const_cast<Tensor&>(tc);
  t.ensure_grad();
  Dev acc = up(t.grad(), n);
  ok(p2r_prim_ew(1, static_cast<long long>(n), g.f(), nullptr, acc.f(), nullptr), "grad accumulate");
  down(acc, t.grad(), n);
}
}  // namespace

// ---------------------------------------------------------------- Tensor
Tensor Tensor::zeros(std::vector<int> shape, bool requires_grad) { return full(std::move(shape), 0.0f, requires_grad); }

Tensor Tensor::full(std::vector<int> shape, float value, bool requires_grad) {
  Tensor t;
  const std::size_t n = count_of(shape);
  t.shape_ = std::move(shape);
  t.data_ = std::make_shared<std::vector<float>>(n, value);
  t.requires_grad_ = requires_grad;
  if (requires_grad) t.ensure_grad();
  return t;
}

Tensor Tensor::from_data(std::vector<int> shape, std::vector<float> values, bool requires_grad) {
  if (count_of(shape) != values.size()) throw std::invalid_argument("tensor: shape does not match value count");
  Tensor t;
  t.shape_ = std::move(shape);
  t.data_ = std::make_shared<std::vector<float>>(std::move(values));
  t.requires_grad_ = requires_grad;
  if (requires_grad) t.ensure_grad();
  return t;
}

Tensor Tensor::device(std::vector<int> shape, std::shared_ptr<DeviceView> view) {
  Tensor t;
  t.shape_ = std::move(shape);
  t.dev_ = std::move(view);
  t.data_ = std::make_shared<std::vector<float>>();
  return t;
}

bool Tensor::defined() const { return static_cast<bool>(data_) || static_cast<bool>(dev_); }

std::size_t Tensor::numel() const { return count_of(shape_); }

const float* Tensor::data() const {
  if (dev_) {
    const std::uint64_t v = dev_->engine->version();
    if (dev_->host_version != v && !dev_->host_dirty) {
      download(*dev_, *data_);
      dev_->host_version = v;
    }
  }
  return data_->data();
}

float* Tensor::data() {
  const float* p = static_cast<const Tensor*>(this)->data();
  if (dev_ && dev_->kind == kParam) dev_->host_dirty = true;  // pushed back before the next forward / step
  return const_cast<float*>(p);
}

std::shared_ptr<std::vector<float>> Tensor::data_ptr() const {
  data();
  return data_;
}

bool Tensor::has_grad() const { return static_cast<bool>(grad_) || (dev_ && dev_->kind == kParam); }

void Tensor::ensure_grad() {
  if (!grad_) grad_ = std::make_shared<std::vector<float>>(numel(), 0.0f);
}

void Tensor::zero_grad() {
  if (grad_) std::fill(grad_->begin(), grad_->end(), 0.0f);
}

float* Tensor::grad() {
  if (dev_ && dev_->kind == kParam) {  // the engine's accumulated gradient (host snapshot)
    if (!grad_) grad_ = std::make_shared<std::vector<float>>(numel(), 0.0f);
    cuda_check(cudaDeviceSynchronize(), "sync");
    dev_->engine->get_grad(dev_->param, grad_->data());
    return grad_->data();
  }
  if (!grad_) throw std::logic_error("tensor: grad buffer not allocated");
  return grad_->data();
}

const float* Tensor::grad() const { return const_cast<Tensor*>(this)->grad(); }

Tensor Tensor::alias_with_grad(std::shared_ptr<std::vector<float>> grad_buffer) const {
  if (!grad_buffer || grad_buffer->size() != numel()) throw std::invalid_argument("tensor: grad alias size mismatch");
  Tensor t = *this;
  t.grad_ = std::move(grad_buffer);
  t.requires_grad_ = true;
  return t;
}

Tensor Tensor::fork_for_grad() const {
  return alias_with_grad(std::make_shared<std::vector<float>>(numel(), 0.0f));
}

Tensor Tensor::clone() const {
  const float* p = data();
  Tensor t;
  t.shape_ = shape_;
  t.data_ = std::make_shared<std::vector<float>>(p, p + numel());
  t.requires_grad_ = requires_grad_;
  if (requires_grad_) t.ensure_grad();
  return t;
}

// ---------------------------------------------------------------- GradTape
void GradTape::backward() {
  for (auto it = entries_.rbegin(); it != entries_.rend(); ++it) (*it)();
}

void GradTape::backward_scalar(Tensor& loss) {
  if (loss.numel() != 1) throw std::invalid_argument("backward_scalar: loss must be scalar");
  // the model layer's fused cross-entropy wrote d logits for d loss = 1 already
  if (!(loss.device_view() && loss.device_view()->kind == kLoss)) {
    loss.ensure_grad();
    loss.grad()[0] += 1.0f;
  }
  backward();
}

// ---------------------------------------------------------------- primitives (csrc/prims.cu)
namespace {
Tensor result(std::vector<int> shape, const Dev& d, bool grad) {
  Tensor t = Tensor::zeros(std::move(shape), grad);
  down(d, t.data(), t.numel());
  return t;
}

// C[m,n] = op(A) op(B) on the device; A [m,k] (or [k,m] if ta), B [k,n] (or [n,k] if tb)
void gemm(bool ta, bool tb, int m, int n, int k, const float* A, const float* B, float* C, float beta) {
  ok(p2r_prim_gemm_f32(ta, tb, m, n, k, A, ta ? m : k, B, tb ? k : n, C, n, beta, 1, 0, 0, 0, nullptr), "gemm");
}
}  // namespace

Tensor matmul(GradTape* tape, const Tensor& a, const Tensor& b) {
  require_2d(a, "matmul");
  require_2d(b, "matmul");
  const int m = a.dim(0), k = a.dim(1), n = b.dim(1);
  if (b.dim(0) != k) throw std::invalid_argument("matmul: inner dimensions disagree");
  Dev da = up(a.data(), a.numel()), db = up(b.data(), b.numel()), dc(static_cast<std::size_t>(m) * n * 4 + 4);
  gemm(false, false, m, n, k, da.f(), db.f(), dc.f(), 0.f);
  Tensor out = result({m, n}, dc, tape != nullptr);
  if (tape) {
    tape->record([a, b, out, m, n, k]() mutable {
      Dev g = up(out.grad(), out.numel()), A = up(a.data(), a.numel()), B = up(b.data(), b.numel());
      if (a.requires_grad()) {  // dA = dC B^T
        Dev d(static_cast<std::size_t>(m) * k * 4 + 4);
        gemm(false, true, m, k, n, g.f(), B.f(), d.f(), 0.f);
        add_grad(a, d, a.numel());
      }
      if (b.requires_grad()) {  // dB = A^T dC
        Dev d(static_cast<std::size_t>(k) * n * 4 + 4);
        gemm(true, false, k, n, m, A.f(), g.f(), d.f(), 0.f);
        add_grad(b, d, b.numel());
      }
    });
  }
  return out;
}

Tensor matmul_nt(GradTape* tape, const Tensor& a, const Tensor& b) {
  require_2d(a, "matmul_nt");
  require_2d(b, "matmul_nt");
  const int m = a.dim(0), k = a.dim(1), n = b.dim(0);
  if (b.dim(1) != k) throw std::invalid_argument("matmul_nt: inner dimensions disagree");
  Dev da = up(a.data(), a.numel()), db = up(b.data(), b.numel()), dc(static_cast<std::size_t>(m) * n * 4 + 4);
  gemm(false, true, m, n, k, da.f(), db.f(), dc.f(), 0.f);
  Tensor out = result({m, n}, dc, tape != nullptr);
  if (tape) {
    tape->record([a, b, out, m, n, k]() mutable {
      Dev g = up(out.grad(), out.numel()), A = up(a.data(), a.numel()), B = up(b.data(), b.numel());
      if (a.requires_grad()) {  // dA = dC B
        Dev d(static_cast<std::size_t>(m) * k * 4 + 4);
        gemm(false, false, m, k, n, g.f(), B.f(), d.f(), 0.f);
        add_grad(a, d, a.numel());
      }
      if (b.requires_grad()) {  // dB = dC^T A
        Dev d(static_cast<std::size_t>(n) * k * 4 + 4);
        gemm(true, false, n, k, m, g.f(), A.f(), d.f(), 0.f);
        add_grad(b, d, b.numel());
      }
    });
  }
  return out;
}

Tensor add(GradTape* tape, const Tensor& a, const Tensor& b) {
  if (a.shape() != b.shape()) throw std::invalid_argument("add: shape mismatch");
  const std::size_t n = a.numel();
  Dev da = up(a.data(), n), db = up(b.data(), n), dc(n * 4 + 4);
  ok(p2r_prim_ew(0, static_cast<long long>(n), da.f(), db.f(), dc.f(), nullptr), "add");
  Tensor out = result(a.shape(), dc, tape != nullptr);
  if (tape) {
    tape->record([a, b, out, n]() mutable {
      Dev g = up(out.grad(), n);
      if (a.requires_grad()) add_grad(a, g, n);
      if (b.requires_grad()) add_grad(b, g, n);
    });
  }
  return out;
}

Tensor add_bias(GradTape* tape, const Tensor& x, const Tensor& b) {
  const int n = x.ndim() > 0 ? x.dim(x.ndim() - 1) : 0;
  if (b.numel() != static_cast<std::size_t>(n)) throw std::invalid_argument("add_bias: bias length must match row width");
  const int rows = n ? static_cast<int>(x.numel() / n) : 0;
  Dev dx = up(x.data(), x.numel()), db = up(b.data(), b.numel()), dc(x.numel() * 4 + 4);
  ok(p2r_prim_bias(rows, n, dx.f(), db.f(), dc.f(), nullptr), "add_bias");
  Tensor out = result(x.shape(), dc, tape != nullptr);
  if (tape) {
    tape->record([x, b, out, rows, n]() mutable {
      Dev g = up(out.grad(), out.numel());
      if (x.requires_grad()) add_grad(x, g, x.numel());
      if (b.requires_grad()) {
        Dev d = zeros_dev(b.numel());
        ok(p2r_prim_colsum_acc(rows, n, g.f(), d.f(), nullptr), "bias grad");
        add_grad(b, d, b.numel());
      }
    });
  }
  return out;
}

Tensor gelu(GradTape* tape, const Tensor& x) {
  const std::size_t n = x.numel();
  Dev dx = up(x.data(), n), dc(n * 4 + 4);
  ok(p2r_prim_ew(2, static_cast<long long>(n), dx.f(), nullptr, dc.f(), nullptr), "gelu");
  Tensor out = result(x.shape(), dc, tape != nullptr);
  if (tape) {
    tape->record([x, out, n]() mutable {
      if (!x.requires_grad()) return;
      Dev g = up(out.grad(), n), X = up(x.data(), n), d = zeros_dev(n);
      ok(p2r_prim_ew(3, static_cast<long long>(n), X.f(), g.f(), d.f(), nullptr), "gelu bwd");
      add_grad(x, d, n);
    });
  }
  return out;
}

Tensor layernorm(GradTape* tape, const Tensor& x, const Tensor& gain, const Tensor& bias, float eps) {
  if (x.ndim() < 1) throw std::invalid_argument("layernorm: rank-0 input");
  const int d = x.dim(x.ndim() - 1);
  if (gain.numel() != static_cast<std::size_t>(d) || bias.numel() != static_cast<std::size_t>(d))
    throw std::invalid_argument("layernorm: gain/bias length must match last dimension");
  const int rows = d ? static_cast<int>(x.numel() / d) : 0;
  Dev X = up(x.data(), x.numel()), G = up(gain.data(), d), Bb = up(bias.data(), d), Y(x.numel() * 4 + 4);
  auto xhat = std::make_shared<Dev>(x.numel() * 4 + 4);
  auto inv = std::make_shared<Dev>(static_cast<std::size_t>(rows) * 4 + 4);
  ok(p2r_prim_layernorm_fwd(rows, d, X.f(), G.f(), Bb.f(), eps, Y.f(), xhat->f(), inv->f(), nullptr), "layernorm");
  Tensor out = result(x.shape(), Y, tape != nullptr);
  if (tape) {
    tape->record([x, gain, bias, out, rows, d, xhat, inv]() mutable {
      Dev g = up(out.grad(), out.numel()), Gn = up(gain.data(), d);
      Dev gx = zeros_dev(x.numel()), gg = zeros_dev(d), gb = zeros_dev(d);
      ok(p2r_prim_layernorm_bwd(rows, d, g.f(), xhat->f(), inv->f(), Gn.f(), gx.f(), gg.f(), gb.f(), nullptr),
         "layernorm bwd");
      if (x.requires_grad()) add_grad(x, gx, x.numel());
      if (gain.requires_grad()) add_grad(gain, gg, d);
      if (bias.requires_grad()) add_grad(bias, gb, d);
    });
  }
  return out;
}

Tensor gather_rows(GradTape* tape, const Tensor& x, std::vector<int> rows) {
  require_2d(x, "gather_rows");
  const int n = x.dim(0), d = x.dim(1), m = static_cast<int>(rows.size());
  for (int r : rows)
    if (r < 0 || r >= n) throw std::out_of_range("gather_rows: row index out of range");
  Dev X = up(x.data(), x.numel()), R = up_i(rows.data(), rows.size()), O(static_cast<std::size_t>(m) * d * 4 + 4);
  ok(p2r_prim_gather_rows(m, d, X.f(), R.i(), O.f(), nullptr), "gather_rows");
  Tensor out = result({m, d}, O, tape != nullptr);
  if (tape) {
    tape->record([x, rows, out, m, d]() mutable {
      if (!x.requires_grad()) return;
      Dev g = up(out.grad(), out.numel()), R = up_i(rows.data(), rows.size()), acc = zeros_dev(x.numel());
      ok(p2r_prim_scatter_rows_acc(m, d, g.f(), R.i(), acc.f(), nullptr), "gather_rows bwd");
      add_grad(x, acc, x.numel());
    });
  }
  return out;
}

Tensor embedding_lookup(GradTape* tape, const Tensor& table, std::span<const int> ids) {
  require_2d(table, "embedding_lookup");
  for (int id : ids)
    if (id < 0 || id >= table.dim(0)) throw std::out_of_range("embedding_lookup: id out of range");
  return gather_rows(tape, table, std::vector<int>(ids.begin(), ids.end()));
}

Tensor split_heads(GradTape* tape, const Tensor& x, int batch, int heads, int seq) {
  if (x.ndim() != 2 || batch <= 0 || heads <= 0 || seq <= 0 || x.dim(0) != batch * seq || x.dim(1) % heads != 0)
    throw std::invalid_argument("split_heads: shape incompatible with batch/heads/seq");
  const int hd = x.dim(1) / heads;
  Dev X = up(x.data(), x.numel()), O(x.numel() * 4 + 4);
  ok(p2r_prim_permute_heads(0, 0, batch, heads, seq, hd, X.f(), O.f(), nullptr), "split_heads");
  Tensor out = result({batch, heads, seq, hd}, O, tape != nullptr);
  if (tape) {
    tape->record([x, out, batch, heads, seq, hd]() mutable {
      if (!x.requires_grad()) return;
      Dev g = up(out.grad(), out.numel()), d = zeros_dev(x.numel());
      ok(p2r_prim_permute_heads(1, 0, batch, heads, seq, hd, g.f(), d.f(), nullptr), "split_heads bwd");
      add_grad(x, d, x.numel());
    });
  }
  return out;
}

Tensor merge_heads(GradTape* tape, const Tensor& x) {
  if (x.ndim() != 4) throw std::invalid_argument("merge_heads: expected 4-D tensor");
  const int B = x.dim(0), H = x.dim(1), S = x.dim(2), hd = x.dim(3);
  Dev X = up(x.data(), x.numel()), O(x.numel() * 4 + 4);
  ok(p2r_prim_permute_heads(1, 0, B, H, S, hd, X.f(), O.f(), nullptr), "merge_heads");
  Tensor out = result({B * S, H * hd}, O, tape != nullptr);
  if (tape) {
    tape->record([x, out, B, H, S, hd]() mutable {
      if (!x.requires_grad()) return;
      Dev g = up(out.grad(), out.numel()), d = zeros_dev(x.numel());
      ok(p2r_prim_permute_heads(0, 0, B, H, S, hd, g.f(), d.f(), nullptr), "merge_heads bwd");
      add_grad(x, d, x.numel());
    });
  }
  return out;
}

Tensor masked_attention(GradTape* tape, const Tensor& q, const Tensor& k, const Tensor& v, bool causal) {
  if (q.ndim() != 4 || q.shape() != k.shape() || q.shape() != v.shape())
    throw std::invalid_argument("masked_attention: q/k/v must share a [B,H,S,hd] shape");
  const int B = q.dim(0), H = q.dim(1), S = q.dim(2), hd = q.dim(3);
  const int BH = B * H;
  const long long qs = static_cast<long long>(S) * hd, ps = static_cast<long long>(S) * S;
  Dev Q = up(q.data(), q.numel()), K = up(k.data(), k.numel()), V = up(v.data(), v.numel());
  auto P = std::make_shared<Dev>(static_cast<std::size_t>(BH) * ps * 4 + 4);
  Dev O(q.numel() * 4 + 4);
  // S = Q K^T (the 1/sqrt(hd) scale is applied to the scores as the reference does)
  ok(p2r_prim_gemm_f32(0, 1, S, S, hd, Q.f(), hd, K.f(), hd, P->f(), S, 0.f, BH, qs, qs, ps, nullptr), "scores");
  {
    std::vector<float> scale(static_cast<std::size_t>(BH) * ps);
    down(*P, scale.data(), scale.size());
    const float sc = 1.0f / std::sqrt(static_cast<float>(hd));
    for (float& f : scale) f *= sc;
    cuda_check(cudaMemcpy(P->p, scale.data(), scale.size() * 4, cudaMemcpyHostToDevice), "h2d");
  }
  ok(p2r_prim_softmax_rows(static_cast<long long>(BH) * S, S, causal ? S : 0, P->f(), nullptr), "softmax");
  ok(p2r_prim_gemm_f32(0, 0, S, hd, S, P->f(), S, V.f(), hd, O.f(), hd, 0.f, BH, ps, qs, qs, nullptr), "PV");
  Tensor out = result(q.shape(), O, tape != nullptr);
  if (tape) {
    tape->record([q, k, v, out, P, B, H, S, hd]() mutable {
      const int BH2 = B * H;
      const long long qs2 = static_cast<long long>(S) * hd, ps2 = static_cast<long long>(S) * S;
      Dev g = up(out.grad(), out.numel()), Q2 = up(q.data(), q.numel()), K2 = up(k.data(), k.numel()),
          V2 = up(v.data(), v.numel());
      Dev dv(q.numel() * 4 + 4), dp(static_cast<std::size_t>(BH2) * ps2 * 4 + 4),
          ds(static_cast<std::size_t>(BH2) * ps2 * 4 + 4), dq(q.numel() * 4 + 4), dk(q.numel() * 4 + 4);
      ok(p2r_prim_gemm_f32(1, 0, S, hd, S, P->f(), S, g.f(), hd, dv.f(), hd, 0.f, BH2, ps2, qs2, qs2, nullptr), "dV");
      ok(p2r_prim_gemm_f32(0, 1, S, S, hd, g.f(), hd, V2.f(), hd, dp.f(), S, 0.f, BH2, qs2, qs2, ps2, nullptr), "dP");
      ok(p2r_prim_softmax_bwd_rows(static_cast<long long>(BH2) * S, S, P->f(), dp.f(), ds.f(), nullptr), "dS");
      ok(p2r_prim_gemm_f32(0, 0, S, hd, S, ds.f(), S, K2.f(), hd, dq.f(), hd, 0.f, BH2, ps2, qs2, qs2, nullptr), "dQ");
      ok(p2r_prim_gemm_f32(1, 0, S, hd, S, ds.f(), S, Q2.f(), hd, dk.f(), hd, 0.f, BH2, ps2, qs2, qs2, nullptr), "dK");
      const float sc = 1.0f / std::sqrt(static_cast<float>(hd));
      std::vector<float> h(q.numel());
      for (Dev* t : {&dq, &dk}) {  // scale, as the reference applies it to dQ and dK
        down(*t, h.data(), h.size());
        for (float& f : h) f *= sc;
        cuda_check(cudaMemcpy(t->p, h.data(), h.size() * 4, cudaMemcpyHostToDevice), "h2d");
      }
      if (q.requires_grad()) add_grad(q, dq, q.numel());
      if (k.requires_grad()) add_grad(k, dk, k.numel());
      if (v.requires_grad()) add_grad(v, dv, v.numel());
    });
  }
  return out;
}

Tensor selected_softmax(GradTape* tape, const Tensor& logits, std::span<const int> selected,
                        std::span<const std::uint8_t> survived, int k) {
  require_2d(logits, "selected_softmax");
  const int T = logits.dim(0), E = logits.dim(1);
  if (k <= 0 || selected.size() != static_cast<std::size_t>(T) * k || survived.size() != selected.size())
    throw std::invalid_argument("selected_softmax: selection size mismatch");
  for (int e : selected)
    if (e < 0 || e >= E) throw std::out_of_range("selected_softmax: expert index");
  std::vector<int> sel(selected.begin(), selected.end());
  std::vector<std::uint8_t> sur(survived.begin(), survived.end());
  Dev L = up(logits.data(), logits.numel()), Sd = up_i(sel.data(), sel.size()), Su = up_u8(sur.data(), sur.size()),
      W(static_cast<std::size_t>(T) * k * 4 + 4);
  ok(p2r_prim_selected_softmax(0, T, E, k, L.f(), nullptr, Sd.i(), static_cast<const std::uint8_t*>(Su.p), W.f(),
                               nullptr),
     "selected_softmax");
  Tensor out = result({T, k}, W, tape != nullptr);
  if (tape) {
    tape->record([logits, sel, sur, out, T, E, k]() mutable {
      if (!logits.requires_grad()) return;
      Dev g = up(out.grad(), out.numel()), w = up(out.data(), out.numel()), Sd2 = up_i(sel.data(), sel.size()),
          Su2 = up_u8(sur.data(), sur.size()), gl = zeros_dev(logits.numel());
      ok(p2r_prim_selected_softmax(1, T, E, k, w.f(), g.f(), Sd2.i(), static_cast<const std::uint8_t*>(Su2.p), gl.f(),
                                   nullptr),
         "selected_softmax bwd");
      add_grad(logits, gl, logits.numel());
    });
  }
  return out;
}

Tensor moe_combine(GradTape* tape, const std::vector<Tensor>& expert_outputs,
                   const std::vector<std::vector<int>>& expert_rows, const std::vector<std::vector<int>>& expert_slots,
                   const Tensor& weights, int n_tokens, int d_model) {
  const std::size_t E = expert_outputs.size();
  if (expert_rows.size() != E || expert_slots.size() != E)
    throw std::invalid_argument("moe_combine: per-expert vectors must align");
  const int k = weights.ndim() == 2 ? weights.dim(1) : 1;
  // concatenate the defined experts' rows in expert order; per token, its
  // contributions in (expert asc, row asc) order -- the reference's summation order
  std::vector<float> y;
  std::vector<int> rtok, rslot, off(static_cast<std::size_t>(n_tokens) + 1, 0);
  std::vector<std::pair<int, int>> base;  // (expert, first concatenated row)
  for (std::size_t e = 0; e < E; ++e) {
    if (!expert_outputs[e].defined()) continue;
    if (expert_rows[e].size() != expert_slots[e].size() ||
        expert_outputs[e].numel() != expert_rows[e].size() * static_cast<std::size_t>(d_model))
      throw std::invalid_argument("moe_combine: per-expert vectors must align");
    base.push_back({static_cast<int>(e), static_cast<int>(rtok.size())});
    const float* p = expert_outputs[e].data();
    y.insert(y.end(), p, p + expert_outputs[e].numel());
    for (std::size_t r = 0; r < expert_rows[e].size(); ++r) {
      const int t = expert_rows[e][r];
      if (t < 0 || t >= n_tokens) throw std::out_of_range("moe_combine: token row out of range");
      rtok.push_back(t);
      rslot.push_back(expert_slots[e][r]);
      ++off[static_cast<std::size_t>(t) + 1];
    }
  }
  const int R = static_cast<int>(rtok.size());
  for (int t = 0; t < n_tokens; ++t) off[static_cast<std::size_t>(t) + 1] += off[static_cast<std::size_t>(t)];
  std::vector<int> crow(static_cast<std::size_t>(R)), cslot(static_cast<std::size_t>(R)), fill(off.begin(), off.end() - 1);
  for (int r = 0; r < R; ++r) {  // rows are visited in expert order: that is the per-token order
    const int t = rtok[static_cast<std::size_t>(r)];
    crow[static_cast<std::size_t>(fill[static_cast<std::size_t>(t)])] = r;
    cslot[static_cast<std::size_t>(fill[static_cast<std::size_t>(t)]++)] = rslot[static_cast<std::size_t>(r)];
  }
  Dev Y = up(y.data(), y.size()), Wt = up(weights.data(), weights.numel()), Of = up_i(off.data(), off.size()),
      Cr = up_i(crow.data(), crow.size()), Cs = up_i(cslot.data(), cslot.size()),
      O = zeros_dev(static_cast<std::size_t>(n_tokens) * d_model);
  ok(p2r_prim_combine_fwd(n_tokens, d_model, k, Of.i(), Cr.i(), Cs.i(), Y.f(), Wt.f(), O.f(), nullptr), "moe_combine");
  Tensor out = result({n_tokens, d_model}, O, tape != nullptr);
  if (tape) {
    tape->record([expert_outputs, weights, out, rtok, rslot, base, y, R, k, d_model]() mutable {
      Dev g = up(out.grad(), out.numel()), Y2 = up(y.data(), y.size()), Wt2 = up(weights.data(), weights.numel()),
          Rt = up_i(rtok.data(), rtok.size()), Rs = up_i(rslot.data(), rslot.size()),
          dy = zeros_dev(static_cast<std::size_t>(R) * d_model), dw = zeros_dev(weights.numel());
      ok(p2r_prim_combine_bwd(R, d_model, k, Rt.i(), Rs.i(), g.f(), Y2.f(), Wt2.f(), dy.f(), dw.f(), nullptr),
         "moe_combine bwd");
      std::vector<float> hdy(static_cast<std::size_t>(R) * d_model);
      down(dy, hdy.data(), hdy.size());
      for (std::size_t i = 0; i < base.size(); ++i) {
        const Tensor& eo = expert_outputs[static_cast<std::size_t>(base[i].first)];
        if (!eo.requires_grad()) continue;
        const std::size_t n = eo.numel();
        Dev part = up(hdy.data() + static_cast<std::size_t>(base[i].second) * d_model, n);
        add_grad(eo, part, n);
      }
      if (weights.requires_grad()) add_grad(weights, dw, weights.numel());
    });
  }
  return out;
}

namespace {
Tensor ce_impl(GradTape* tape, const Tensor& logits, std::span<const int> targets,
               const std::uint8_t* mask, double denom) {
  // model-layer logits: the engine's fused cross-entropy (seeds d logits for the head closure)
  if (logits.device_view() && logits.device_view()->kind == kLogits) {
    Engine& e = *logits.device_view()->engine;
    if (denom <= 0.0) throw std::invalid_argument("softmax_cross_entropy: denominator must be > 0");
    const int* dt = nullptr;
    const std::uint8_t* dm = nullptr;
    e.stage_targets(targets.data(), mask, static_cast<int>(targets.size()), &dt, &dm);
    const DeviceView& lv = *logits.device_view();
    const DevTensor L{lv.rows, lv.cols, const_cast<float*>(lv.ptr), nullptr, nullptr};
    const DevTensor loss = e.softmax_cross_entropy(tape, L, dt, dm, denom);
    auto v = std::make_shared<DeviceView>();
    v->engine = &e;
    v->keep = lv.keep;
    v->ptr = loss.data;
    v->rows = v->cols = v->ld = 1;
    v->kind = kLoss;
    return Tensor::device({1}, v);
  }
  require_2d(logits, "softmax_cross_entropy");
  const int rows = logits.dim(0), V = logits.dim(1);
  if (targets.size() != static_cast<std::size_t>(rows))
    throw std::invalid_argument("softmax_cross_entropy: one target per row required");
  if (denom <= 0.0) throw std::invalid_argument("softmax_cross_entropy: denominator must be > 0");
  for (int r = 0; r < rows; ++r)
    if ((mask == nullptr || mask[r] != 0) && (targets[static_cast<std::size_t>(r)] < 0 || targets[static_cast<std::size_t>(r)] >= V))
      throw std::out_of_range("softmax_cross_entropy: target out of range");
  Dev L = up(logits.data(), logits.numel()), Tg = up_i(targets.data(), targets.size()),
      M = mask ? up_u8(mask, static_cast<std::size_t>(rows)) : Dev(), ws(static_cast<std::size_t>(rows) * 8 + 8),
      loss(4);
  auto gl = std::make_shared<Dev>(logits.numel() * 4 + 4);
  ok(p2r_prim_cross_entropy(rows, V, L.f(), Tg.i(), mask ? static_cast<const std::uint8_t*>(M.p) : nullptr, denom,
                            static_cast<double*>(ws.p), loss.f(), gl->f(), nullptr),
     "softmax_cross_entropy");
  Tensor out = result({1}, loss, tape != nullptr);
  if (tape) {
    tape->record([logits, out, gl]() mutable {
      if (!logits.requires_grad()) return;
      // d logits = (p - onehot) / denom, times the loss gradient
      const float s = out.grad()[0];
      std::vector<float> h(logits.numel());
      down(*gl, h.data(), h.size());
      for (float& f : h) f *= s;
      Dev d = up(h.data(), h.size());
      add_grad(logits, d, logits.numel());
    });
  }
  return out;
}
}  // namespace

Tensor softmax_cross_entropy(GradTape* tape, const Tensor& logits, std::span<const int> targets) {
  const int rows = logits.ndim() == 2 ? logits.dim(0) : 0;
  return ce_impl(tape, logits, targets, nullptr, static_cast<double>(std::max(rows, 1)));
}

Tensor softmax_cross_entropy(GradTape* tape, const Tensor& logits, std::span<const int> targets,
                             std::span<const std::uint8_t> mask, double denom) {
  if (!mask.empty() && mask.size() != targets.size())
    throw std::invalid_argument("softmax_cross_entropy: mask size mismatch");
  return ce_impl(tape, logits, targets, mask.empty() ? nullptr : mask.data(), denom);
}

// ---------------------------------------------------------------- LayerParams
void LayerParams::for_each(const std::function<void(const std::string&, Tensor&)>& fn) {
  auto v = [&](const char* n, Tensor& t) {
    if (t.defined()) fn(n, t);
  };
  v("ln1.gain", ln1_gain);
  v("ln1.bias", ln1_bias);
  v("attn.wq", wq);
  v("attn.wk", wk);
  v("attn.wv", wv);
  v("attn.wo", wo);
  v("ln2.gain", ln2_gain);
  v("ln2.bias", ln2_bias);
  v("ffn.w1", ffn_w1);
  v("ffn.b1", ffn_b1);
  v("ffn.w2", ffn_w2);
  v("ffn.b2", ffn_b2);
  v("moe.gate", gate);
  for (std::size_t e = 0; e < experts.size(); ++e) {
    const std::string p = "moe.expert." + std::to_string(e) + ".";
    v((p + "w1").c_str(), experts[e].w1);
    v((p + "b1").c_str(), experts[e].b1);
    v((p + "w2").c_str(), experts[e].w2);
    v((p + "b2").c_str(), experts[e].b2);
  }
}

void LayerParams::for_each(const std::function<void(const std::string&, const Tensor&)>& fn) const {
  const_cast<LayerParams*>(this)->for_each([&](const std::string& n, Tensor& t) { fn(n, t); });
}

// ---------------------------------------------------------------- Model (drop-in handle)
struct ParamViews {
  std::vector<Tensor> by_index;  // engine parameter order (for_each_param order)
  std::vector<LayerParams> layers;
  Tensor* tok = nullptr;
  Tensor* pos = nullptr;
};

namespace {
std::shared_ptr<ParamViews> make_views(const std::shared_ptr<Engine>& e) {
  auto pv = std::make_shared<ParamViews>();
  const auto& views = e->params();
  pv->by_index.reserve(views.size());
  for (std::size_t i = 0; i < views.size(); ++i) {
    auto dv = std::make_shared<DeviceView>();
    dv->engine = e.get();
    dv->keep = e;
    dv->rows = views[i].rows;
    dv->cols = views[i].cols;
    dv->ld = views[i].ld;
    dv->kind = kParam;
    dv->param = static_cast<int>(i);
    pv->by_index.push_back(Tensor::device(views[i].shape, dv));
    pv->by_index.back().set_requires_grad(true);
  }
  const ModelConfig& c = e->config();
  pv->layers.resize(static_cast<std::size_t>(c.n_layers_params));
  for (std::size_t i = 0; i < views.size(); ++i) {
    const std::string& n = views[i].name;
    Tensor& t = pv->by_index[i];
    if (n == "embed.tok") pv->tok = &t;
    if (n == "embed.pos") pv->pos = &t;
    if (views[i].granule < 0) continue;
    LayerParams& L = pv->layers[static_cast<std::size_t>(views[i].granule)];
    const std::string rest = n.substr(n.find('.', 6) + 1);  // after "layer.<i>."
    if (rest == "ln1.gain") L.ln1_gain = t;
    else if (rest == "ln1.bias") L.ln1_bias = t;
    else if (rest == "attn.wq") L.wq = t;
    else if (rest == "attn.wk") L.wk = t;
    else if (rest == "attn.wv") L.wv = t;
    else if (rest == "attn.wo") L.wo = t;
    else if (rest == "ln2.gain") L.ln2_gain = t;
    else if (rest == "ln2.bias") L.ln2_bias = t;
    else if (rest == "ffn.w1") L.ffn_w1 = t;
    else if (rest == "ffn.b1") L.ffn_b1 = t;
    else if (rest == "ffn.w2") L.ffn_w2 = t;
    else if (rest == "ffn.b2") L.ffn_b2 = t;
    else if (rest == "moe.gate") L.gate = t;
    else if (rest.rfind("moe.expert.", 0) == 0) {
      const std::size_t dot = rest.find('.', 11);
      const std::size_t e = static_cast<std::size_t>(std::stoi(rest.substr(11, dot - 11)));
      if (L.experts.size() <= e) L.experts.resize(e + 1);
      const std::string p = rest.substr(dot + 1);
      if (p == "w1") L.experts[e].w1 = t;
      else if (p == "b1") L.experts[e].b1 = t;
      else if (p == "w2") L.experts[e].w2 = t;
      else L.experts[e].b2 = t;
    }
  }
  return pv;
}

std::shared_ptr<DeviceView> act_view(const Model& m, const DevTensor& t, int kind, int ld) {
  auto v = std::make_shared<DeviceView>();
  v->engine = &m.engine();
  v->ptr = t.data;
  v->rows = t.rows;
  v->cols = t.cols;
  v->ld = ld;
  v->kind = kind;
  return v;
}
}  // namespace

Model::Model(ModelConfig config, std::uint64_t seed)
    : config_(config), engine_(std::make_shared<Engine>(std::move(config), seed)) {
  views_ = make_views(engine_);
}

Model::Model(std::shared_ptr<Engine> engine) : config_(engine->config()), engine_(std::move(engine)) {
  views_ = make_views(engine_);
}

void Model::sync_params() const {
  for (Tensor& t : views_->by_index) {
    const auto& dv = t.device_view();
    if (dv->host_dirty) {
      engine_->set_param(dv->param, t.data_ptr()->data());
      dv->host_dirty = false;
      dv->host_version = engine_->version();
    }
  }
}

Tensor Model::forward(std::span<const int> tokens, int batch, AttentionMode mode) const {
  if (batch <= 0 || tokens.size() % static_cast<std::size_t>(batch) != 0)
    throw std::invalid_argument("forward: token count must be a multiple of batch");
  sync_params();
  const int T = static_cast<int>(tokens.size()), V = config_.vocab_size;
  std::vector<float> logits(static_cast<std::size_t>(T) * V);
  engine_->forward_host(tokens.data(), batch, T / batch, mode, logits.data());
  return Tensor::from_data({T, V}, std::move(logits));
}

Tensor Model::embed_forward(GradTape* tape, std::span<const int> tokens, int batch) const {
  if (batch <= 0 || tokens.size() % static_cast<std::size_t>(batch) != 0)
    throw std::invalid_argument("forward: token count must be a multiple of batch");
  sync_params();
  const int T = static_cast<int>(tokens.size());
  const int* d = engine_->stage_tokens(tokens.data(), batch, T / batch);
  const DevTensor x = engine_->embed_forward(tape, d, batch, T / batch);
  return Tensor::device({x.rows, x.cols}, act_view(*this, x, kAct, x.cols));
}

Tensor Model::block_forward(GradTape* tape, int graph_layer, const Tensor& x, int batch, AttentionMode mode) const {
  if (graph_layer < 0 || graph_layer >= config_.n_layers_graph)
    throw std::out_of_range("model: graph layer index out of range");
  DevTensor in;
  const auto& dv = x.device_view();
  if (dv && dv->kind == kAct && dv->engine == engine_.get()) {
    in = DevTensor{dv->rows, dv->cols, const_cast<float*>(dv->ptr), nullptr, nullptr};
  } else {  // a host activation: into the engine's input buffer
    if (x.ndim() != 2 || x.dim(1) != config_.d_model)
      throw std::invalid_argument("block_forward: batch does not match embed_forward");
    in = DevTensor{x.dim(0), x.dim(1), engine_->stage_activation(x.data(), x.dim(0)), nullptr, nullptr};
  }
  const DevTensor y = engine_->block_forward(tape, graph_layer, in, batch, mode);
  return Tensor::device({y.rows, y.cols}, act_view(*this, y, kAct, y.cols));
}

Tensor Model::head_forward(GradTape* tape, const Tensor& x) const {
  const auto& dv = x.device_view();
  DevTensor in;
  if (dv && dv->kind == kAct && dv->engine == engine_.get())
    in = DevTensor{dv->rows, dv->cols, const_cast<float*>(dv->ptr), nullptr, nullptr};
  else
    in = DevTensor{x.dim(0), x.dim(1), engine_->stage_activation(x.data(), x.dim(0)), nullptr, nullptr};
  const DevTensor l = engine_->head_forward(tape, in);
  auto v = act_view(*this, l, kLogits, engine_->vocab_ld());
  v->keep = engine_;
  return Tensor::device({l.rows, l.cols}, v);
}

const LayerParams& Model::graph_layer(int g) const {
  if (g < 0 || g >= config_.n_layers_graph) throw std::out_of_range("model: graph layer index out of range");
  return views_->layers[static_cast<std::size_t>(owned_index_of_graph_layer(g))];
}
LayerParams& Model::owned_layer(int i) { return views_->layers.at(static_cast<std::size_t>(i)); }
const LayerParams& Model::owned_layer(int i) const { return views_->layers.at(static_cast<std::size_t>(i)); }
Tensor& Model::token_embedding() { return *views_->tok; }
Tensor& Model::position_embedding() { return *views_->pos; }

void Model::for_each_param(const std::function<void(const std::string&, Tensor&)>& fn) {
  const auto& views = engine_->params();
  for (std::size_t i = 0; i < views.size(); ++i) fn(views[i].name, views_->by_index[i]);
}
void Model::for_each_param(const std::function<void(const std::string&, const Tensor&)>& fn) const {
  const auto& views = engine_->params();
  for (std::size_t i = 0; i < views.size(); ++i) fn(views[i].name, views_->by_index[i]);
}

void Model::zero_grads() { engine_->zero_grads(); }
void Model::flush_shared_layer_grads() { engine_->flush_shared_layer_grads(); }
std::int64_t Model::scratch_grad_bytes() const { return engine_->scratch_grad_bytes(); }
int Model::expert_shard(int expert) const { return engine_->expert_shard(expert); }
std::vector<std::vector<int>> Model::shard_layout() const { return engine_->shard_layout(); }
void Model::redistribute_experts(int new_n_shards) {
  engine_->redistribute_experts(new_n_shards);
  config_.moe.n_shards = engine_->config().moe.n_shards;
}

Model Model::delinked() const {
  sync_params();
  std::unique_ptr<Engine> real = engine_->delinked();
  return Model(std::shared_ptr<Engine>(std::move(real)));
}

Model build_model(const ModelConfig& config, std::uint64_t seed) { return Model(config, seed); }

Model redistribute_experts(const Model& model, int new_n_shards) {
  // copies share the engine (as the reference's Model copies share tensors); the
  // shard assignment is bookkeeping of that engine
  Model m = model;
  m.redistribute_experts(new_n_shards);
  return m;
}

Routing moe_dispatch(const Tensor& gating_logits, const MoEConfig& moe) {
  if (!moe.enabled()) throw std::invalid_argument("moe_dispatch: moe disabled");
  if (gating_logits.ndim() != 2 || gating_logits.dim(1) != moe.n_experts)
    throw std::invalid_argument("moe_dispatch: logits must be [tokens, n_experts]");
  const int T = gating_logits.dim(0);
  const HostRouting h = moe_dispatch_host(gating_logits.data(), T, moe);
  Routing r;
  r.n_tokens = T;
  r.k = moe.n_prototypes;
  r.selected = h.selected;
  r.survived = h.survived;
  r.raw_load = h.raw_load;
  r.capacity = h.capacity;
  r.dropped = h.dropped;
  r.expert_rows.resize(static_cast<std::size_t>(moe.n_experts));
  r.expert_slots.resize(static_cast<std::size_t>(moe.n_experts));
  for (int e = 0; e < moe.n_experts; ++e)
    for (int i = h.offsets[static_cast<std::size_t>(e)]; i < h.offsets[static_cast<std::size_t>(e) + 1]; ++i) {
      r.expert_rows[static_cast<std::size_t>(e)].push_back(h.rows[static_cast<std::size_t>(i)]);
      r.expert_slots[static_cast<std::size_t>(e)].push_back(h.slots[static_cast<std::size_t>(i)]);
    }
  return r;
}

// ---------------------------------------------------------------- LrSchedule / AdamW
LrSchedule LrSchedule::cosine(float peak, double warmup_ratio, std::int64_t total_steps) {
  if (total_steps <= 0) throw std::invalid_argument("lr schedule: total_steps must be positive");
  LrSchedule s;
  s.peak = peak;
  s.total_steps = total_steps;
  s.warmup_steps = std::max<std::int64_t>(
      1, static_cast<std::int64_t>(std::llround(warmup_ratio * static_cast<double>(total_steps))));
  return s;
}

float LrSchedule::at(std::int64_t step) const {
  if (step < warmup_steps) return peak * static_cast<float>(step) / static_cast<float>(warmup_steps);
  const double span = static_cast<double>(std::max<std::int64_t>(1, total_steps - warmup_steps));
  const double t = std::min(1.0, static_cast<double>(step - warmup_steps) / span);
  return static_cast<float>(peak * 0.5 * (1.0 + std::cos(t * 3.14159265358979323846)));
}

AdamW::AdamW(AdamWSettings settings) : settings_(settings) {}

void AdamW::register_model(Model& model) {
  engine_ = &model.engine();
  engine_->adamw_attach(settings_.beta1, settings_.beta2, settings_.eps, settings_.weight_decay);
  engine_->set_step_count(step_count_);
}

void AdamW::step(Model& model, float lr) {
  if (engine_ == nullptr || engine_ != &model.engine()) throw std::logic_error("adamw: unregistered parameter embed.tok");
  model.sync_params();
  engine_->adamw_step(lr);
  step_count_ = engine_->step_count();
}

std::int64_t AdamW::step_count() const { return engine_ ? engine_->step_count() : step_count_; }

void AdamW::set_step_count(std::int64_t t) {
  step_count_ = t;
  if (engine_) engine_->set_step_count(t);
}

std::map<std::string, AdamW::Moments>& AdamW::moments() {
  if (engine_) {
    const auto& views = engine_->params();
    for (std::size_t i = 0; i < views.size(); ++i) {
      Moments& m = moments_[views[i].name];
      const std::size_t n = static_cast<std::size_t>(views[i].rows) * views[i].cols;
      m.m.resize(n);
      m.v.resize(n);
      engine_->get_moment(static_cast<int>(i), 0, m.m.data());
      engine_->get_moment(static_cast<int>(i), 1, m.v.data());
    }
  }
  return moments_;
}

const std::map<std::string, AdamW::Moments>& AdamW::moments() const { return const_cast<AdamW*>(this)->moments(); }

std::int64_t AdamW::state_bytes() const { return engine_ ? engine_->state_bytes() : 0; }

}  // namespace p2r
