// Granular CPU offloading (§4.2; the reference's
// offload.cpp is absent, so this follows the spec's Fn / Bn / An phase model).
//
// SLOW layer granules live in pinned host DRAM (fp32 master + bf16 shadow +
// AdamW moments). A ring of HBM staging slots (each one granule of p32, grad,
// m, v, bf16) is fed by cudaMemcpyAsync on a dedicated H2D stream and drained
// by a D2H stream, event-synchronised with the compute stream. The step's SLOW
// uses (forward ascending, then backward descending) are staged as far ahead as
// the ring allows, so backward granules load during the H2D-light forward:
//   Fn : H2D bf16 shadow + the fp32 vectors / MoE gate (default), or (master
//        form: P2R_OFFLOAD_FN_MASTER=1 or P2R_OFFLOAD_FN_SHADOW=0) the fp32 master
//   Bn : H2D fp32 master (+ m, v) in the micro-step that applies AdamW (the bf16
//        operand is re-derived on the device); accumulating micro-steps load the
//        Fn form plus the parked partial gradients
//   An : AdamW for the granule on the GPU right after its backward, then D2H
//        write-back of p32 + m + v (+ the bf16 shadow in the shadow form), or
//        of the grads when no optimizer is attached / the window continues.
// FAST granules stay resident; the placement comes from plan_offload.
#include <cuda_runtime.h>

#include <algorithm>
#include <cstdlib>
#include <cmath>
#include <cstring>
#include <limits>

#include "offload_state.hpp"
#include "p2r_cuda.h"

namespace p2r {

float* offload_slot_ptr(const OffloadState& st, int owned, int kind) {
  const int s = st.slot_of[static_cast<std::size_t>(owned)];
  if (s < 0) throw std::logic_error("offload: SLOW granule used while not staged");
  const OffloadSlot& sl = st.slots[static_cast<std::size_t>(s)];
  switch (kind) {
    case 0: return sl.p32.as<float>();
    case 1: return sl.g32.as<float>();
    case 2: return sl.m.as<float>();
    case 3: return sl.v.as<float>();
    default: return reinterpret_cast<float*>(sl.p16.as<std::uint16_t>());
  }
}

void host_cast_bf16(const float* src, std::uint16_t* dst, long long n) {
  for (long long i = 0; i < n; ++i) {
    std::uint32_t u;
    std::memcpy(&u, src + i, 4);
    if ((u & 0x7fffffffu) > 0x7f800000u) {  // NaN: keep quiet NaN
      dst[i] = static_cast<std::uint16_t>((u >> 16) | 0x40u);
      continue;
    }
    const std::uint32_t r = u + 0x7fffu + ((u >> 16) & 1u);
    dst[i] = static_cast<std::uint16_t>(r >> 16);
  }
}

// ---------------------------------------------------------------- planner
double predict_step_time(const std::vector<std::int64_t>& layer_bytes, const std::vector<int>& slow,
                         double bandwidth, double compute_s, double latency_s) {
  double moved = 0;
  int n = 0;
  for (std::size_t i = 0; i < layer_bytes.size(); ++i)
    if (slow[i]) {
      moved += 4.0 * static_cast<double>(layer_bytes[i]);  // Fn + Bn + grad + write-back
      n += 4;
    }
  return compute_s + moved / bandwidth + n * latency_s;
}

double predict_step_time_overlap(const std::vector<std::int64_t>& layer_params,
                                 const std::vector<std::int64_t>& vector_params, const std::vector<int>& slow,
                                 const OffloadCost& c) {
  const std::size_t L = layer_params.size();
  if (slow.size() != L || (!vector_params.empty() && vector_params.size() != L))
    throw std::invalid_argument("predict_step_time_overlap: layer / placement size mismatch");
  const double M = static_cast<double>(std::max(1, c.micro_steps));
  double h2d_f = 0, h2d_b = 0, h2d_bn = 0, h2d_bf = 0, d2h = 0, d2h_f = 0, fill = -1, drain = 0;
  int n_slow = 0;
  for (std::size_t i = 0; i < L; ++i)
    if (slow[i]) {
      ++n_slow;
      const double P = static_cast<double>(layer_params[i]);
      const double vec = vector_params.empty() ? 0.0 : static_cast<double>(vector_params[i]);
      // forward: bf16 shadow + the fp32 vectors it reads, or the whole fp32 master
      const double f = c.fn_master ? 4.0 * P : 2.0 * P + 4.0 * vec;
      const double w = c.fn_master ? 12.0 * P : 14.0 * P;  // updated p, m, v (+ bf16 shadow)
      h2d_f += f;                   // per micro-step
      h2d_b += 4.0 * P;             // last micro-step: fp32 master (bf16 re-derived on the device)
      h2d_bn += c.fn_master ? 4.0 * P : f;  // accumulating micro-steps: what the forward loads
      h2d_bf += 8.0 * P;            // last micro-step: m + v
      d2h_f += w;                   // last micro-step: write-back
      d2h += 4.0 * P;               // earlier micro-steps: partial gradients parked ...
      if (fill < 0) {
        // the lowest SLOW layer: its Fn load opens the step behind the forward of the
        // layers below it, its write-back closes it behind their backward
        fill = std::max(0.0, f / c.h2d_bw - c.fwd_s * static_cast<double>(i));
        drain = std::max(0.0, w / c.d2h_bw - c.bwd_s * static_cast<double>(i));
      }
    }
  const double cf = c.fwd_s * static_cast<double>(L);
  const double cb = c.bwd_s * static_cast<double>(L) + (c.recompute ? c.fwd_s * n_slow : 0.0);
  // micro-steps 1 .. M-1 park the partial grads (D2H 4P); from the 2nd on they are
  // reloaded with the Bn load (H2D another 4P); the last loads the master, moments,
  // and writes back
  double phases = 0, h2d_all = 0;
  for (int m = 1; m <= static_cast<int>(M); ++m) {
    const bool last = m == static_cast<int>(M);
    const double hb = (last ? h2d_b + h2d_bf : h2d_bn) + (m > 1 ? h2d_b : 0.0);
    h2d_all += h2d_f + hb;
    const double db = last ? d2h_f : d2h;
    phases += std::max(cf, h2d_f / c.h2d_bw) + std::max({cb, hb / c.h2d_bw, db / c.d2h_bw});
  }
  // the ring prefetches backward granules during the forward, so the H2D stream can
  // also be the bound as a whole: every load, plus the exposed first load and last write-back
  const double stream = fill < 0 ? 0.0 : h2d_all / c.h2d_bw + fill + drain;
  return std::max(phases, stream);
}

std::vector<int> plan_offload_overlap(const std::vector<std::int64_t>& layer_params, std::int64_t budget,
                                      const OffloadCost& c) {
  const int n = static_cast<int>(layer_params.size());
  std::int64_t total = 0, largest = 0;
  for (auto p : layer_params) {
    total += 18 * p;
    largest = std::max<std::int64_t>(largest, 18 * p);
  }
  if (budget < largest) throw std::runtime_error("plan_offload: no feasible plan (a single layer exceeds the budget)");
  // once anything is SLOW the engine also holds `ring_slots` HBM staging slots of the
  // largest granule: they count against the budget too
  const std::int64_t staging = static_cast<std::int64_t>(std::max(c.ring_slots, 2)) * largest;
  if (total <= budget) return std::vector<int>(static_cast<std::size_t>(n), 0);
  const std::int64_t fast_budget = budget - staging;
  if (fast_budget < 0) throw std::runtime_error("plan_offload: no feasible plan (staging ring exceeds the budget)");
  // fewest SLOW layers (largest first) that bring the resident granules under budget
  std::vector<int> order(static_cast<std::size_t>(n));
  for (int i = 0; i < n; ++i) order[static_cast<std::size_t>(i)] = i;
  std::stable_sort(order.begin(), order.end(),
                   [&](int a, int b) { return layer_params[static_cast<std::size_t>(a)] > layer_params[static_cast<std::size_t>(b)]; });
  int k = 0;
  for (std::int64_t fast = total; fast > fast_budget && k < n; ++k)
    fast -= 18 * layer_params[static_cast<std::size_t>(order[static_cast<std::size_t>(k)])];
  std::vector<int> pl(static_cast<std::size_t>(n), 0);
  const std::int64_t budget_fast = fast_budget;
  // spread k SLOW layers evenly, half a stride in: every copy gets the most neighbouring
  // compute to hide under, and layer 0 -- whose Fn load would open the step and whose
  // write-back would close it with nothing to overlap -- stays resident when k < n
  for (int j = 0; j < k; ++j) pl[static_cast<std::size_t>((static_cast<long long>(2 * j + 1) * n) / (2 * k))] = 1;
  std::int64_t fast = 0;
  for (int i = 0; i < n; ++i)
    if (!pl[static_cast<std::size_t>(i)]) fast += 18 * layer_params[static_cast<std::size_t>(i)];
  if (fast > budget_fast) {  // non-uniform layers: fall back to the largest-first choice
    std::fill(pl.begin(), pl.end(), 0);
    for (int j = 0; j < k; ++j) pl[static_cast<std::size_t>(order[static_cast<std::size_t>(j)])] = 1;
  }
  (void)c;
  return pl;
}

std::vector<int> plan_offload(const std::vector<std::int64_t>& layer_bytes, std::int64_t budget, double bandwidth,
                              double compute_s, double latency_s) {
  const int n = static_cast<int>(layer_bytes.size());
  std::int64_t total = 0, largest = 0;
  for (auto b : layer_bytes) {
    total += b;
    largest = std::max(largest, b);
  }
  // pre: a SLOW layer must fit the fast tier while it is staged
  if (budget < largest) throw std::runtime_error("plan_offload: no feasible plan (a single layer exceeds the budget)");
  if (n <= 12) {
    std::vector<int> best;
    double best_t = std::numeric_limits<double>::infinity();
    for (std::uint32_t mask = 0; mask < (1u << n); ++mask) {
      std::vector<int> pl(static_cast<std::size_t>(n));
      std::int64_t fast = 0;
      for (int i = 0; i < n; ++i) {
        pl[static_cast<std::size_t>(i)] = (mask >> i) & 1u;
        if (!pl[static_cast<std::size_t>(i)]) fast += layer_bytes[static_cast<std::size_t>(i)];
      }
      if (fast > budget) continue;
      const double t = predict_step_time(layer_bytes, pl, bandwidth, compute_s, latency_s);
      // ties -> offload the lowest-indexed layers (lexicographically larger `pl`)
      if (t < best_t || (t == best_t && pl > best)) {
        best_t = t;
        best = pl;
      }
    }
    if (best.empty()) throw std::runtime_error("plan_offload: no feasible plan");
    return best;
  }
  std::vector<int> pl(static_cast<std::size_t>(n), 0);
  std::int64_t fast = total;
  for (int i = 0; i < n && fast > budget; ++i) {
    pl[static_cast<std::size_t>(i)] = 1;
    fast -= layer_bytes[static_cast<std::size_t>(i)];
  }
  if (fast > budget) throw std::runtime_error("plan_offload: no feasible plan");
  return pl;
}

// ---------------------------------------------------------------- engine side
void Engine::offload_setup(const std::vector<int>& slow, int ring_slots) {
  // A Pseudo model's L graph layers share one granule: reloading it per graph layer
  // would apply L fused AdamW updates from partial gradients
  if (cfg_.n_layers_params != cfg_.n_layers_graph)
    throw std::invalid_argument("offload: granular offload needs an unshared (Real) model");
  if (static_cast<int>(slow.size()) != n_owned_)
    throw std::invalid_argument("offload: placement must give one entry per owned layer");
  if (ring_slots < 2) throw std::invalid_argument("offload: need at least 2 staging slots");
  auto st = std::make_unique<OffloadState>();
  st->ring = ring_slots;
  st->stride = layer_stride_;
  {
    const char* e = std::getenv("P2R_OFFLOAD_FN_SHADOW");
    const char* m = std::getenv("P2R_OFFLOAD_FN_MASTER");
    // default: the bf16-shadow form (H2D 14 B/param = D2H 14 B/param per step with the
    // optimizer); the master form moves 16 in / 12 out
    st->fwd_master = (m != nullptr && m[0] == '1') || (e != nullptr && e[0] == '0');
  }
  st->slot_of.assign(static_cast<std::size_t>(n_owned_), -1);
  st->slot_fwd.assign(static_cast<std::size_t>(n_owned_), -1);
  st->slot_bwd.assign(static_cast<std::size_t>(n_owned_), -1);
  st->host_idx.assign(static_cast<std::size_t>(n_owned_), -1);
  st->hgrad_valid.assign(static_cast<std::size_t>(n_owned_), 0);
  slow_ = slow;
  int nr = 0, ns = 0;
  for (int o = 0; o < n_owned_; ++o) {
    if (slow[static_cast<std::size_t>(o)]) {
      res_idx_[static_cast<std::size_t>(o)] = -1;
      st->host_idx[static_cast<std::size_t>(o)] = ns++;
      st->slow_list.push_back(o);
    } else {
      res_idx_[static_cast<std::size_t>(o)] = nr++;
    }
  }
  n_res_ = nr;
  if (ns == 0) return;  // nothing offloaded
  const std::size_t n = static_cast<std::size_t>(layer_stride_) * ns;
  cuda_check(cudaMallocHost(reinterpret_cast<void**>(&st->hp32), n * 4), "pinned p32");
  cuda_check(cudaMallocHost(reinterpret_cast<void**>(&st->hp16), n * 2), "pinned bf16");
  std::memset(st->hp32, 0, n * 4);
  std::memset(st->hp16, 0, n * 2);
  const std::size_t g = static_cast<std::size_t>(layer_stride_);
  st->slots.resize(static_cast<std::size_t>(ring_slots));
  for (auto& s : st->slots) {
    s.p32 = DevBuf(g * 4);
    s.g32 = DevBuf(g * 4);
    s.m = DevBuf(g * 4);
    s.v = DevBuf(g * 4);
    s.p16 = DevBuf(g * 2);
    cuda_check(cudaEventCreateWithFlags(&s.loaded, cudaEventDisableTiming), "event");
    cuda_check(cudaEventCreateWithFlags(&s.free_ev, cudaEventDisableTiming), "event");
  }
  st->wb_ev.resize(static_cast<std::size_t>(n_owned_));
  st->wb_fn_ev.resize(static_cast<std::size_t>(n_owned_));
  st->wb_recorded.assign(static_cast<std::size_t>(n_owned_), 0);
  for (auto& e : st->wb_ev) cuda_check(cudaEventCreateWithFlags(&e, cudaEventDisableTiming), "event");
  for (auto& e : st->wb_fn_ev) cuda_check(cudaEventCreateWithFlags(&e, cudaEventDisableTiming), "event");
  cuda_check(cudaStreamCreateWithFlags(&st->h2d, cudaStreamNonBlocking), "h2d stream");
  cuda_check(cudaStreamCreateWithFlags(&st->d2h, cudaStreamNonBlocking), "d2h stream");
  off_ = std::move(st);
}

void Engine::offload_alloc_moments() {
  if (!off_ || off_->slow_list.empty() || off_->hm) return;
  const std::size_t n = static_cast<std::size_t>(layer_stride_) * off_->slow_list.size();
  cuda_check(cudaMallocHost(reinterpret_cast<void**>(&off_->hm), n * 4), "pinned m");
  cuda_check(cudaMallocHost(reinterpret_cast<void**>(&off_->hv), n * 4), "pinned v");
  std::memset(off_->hm, 0, n * 4);
  std::memset(off_->hv, 0, n * 4);
}

float* Engine::slow_host_p32(int o) const {
  return off_->hp32 + static_cast<long long>(off_->host_idx[static_cast<std::size_t>(o)]) * layer_stride_;
}
std::uint16_t* Engine::slow_host_p16(int o) const {
  return off_->hp16 + static_cast<long long>(off_->host_idx[static_cast<std::size_t>(o)]) * layer_stride_;
}
float* Engine::slow_host_m(int o, int which) const {
  float* b = which ? off_->hv : off_->hm;
  if (!b) throw std::logic_error("adamw: optimizer not attached");
  return b + static_cast<long long>(off_->host_idx[static_cast<std::size_t>(o)]) * layer_stride_;
}
float* Engine::slow_host_grad(int o) const {
  if (!off_->hg) return nullptr;
  return off_->hg + static_cast<long long>(off_->host_idx[static_cast<std::size_t>(o)]) * layer_stride_;
}

namespace {
void copy_async(OffloadState& st, void* dst, const void* src, std::size_t bytes, cudaStream_t s, bool h2d,
                double* counter) {
  *counter += static_cast<double>(bytes);
  if (st.skip) return;
  cuda_check(cudaMemcpyAsync(dst, src, bytes, h2d ? cudaMemcpyHostToDevice : cudaMemcpyDeviceToHost, s), "offload copy");
}
}  // namespace

void Engine::offload_begin_forward(bool training) {
  OffloadState& st = *off_;
  st.training = training;
  std::fill(st.slot_of.begin(), st.slot_of.end(), -1);
  std::fill(st.slot_fwd.begin(), st.slot_fwd.end(), -1);
  std::fill(st.slot_bwd.begin(), st.slot_bwd.end(), -1);
  for (auto& s : st.slots) s.layer = -1;
  st.sched.clear();
  for (int o : st.slow_list) st.sched.emplace_back(o, false);
  if (training)
    for (auto it = st.slow_list.rbegin(); it != st.slow_list.rend(); ++it) st.sched.emplace_back(*it, true);
  st.next_issue = 0;
  st.in_flight = 0;
  offload_prefetch_next(-1, false);
}

// Issue H2D staging for the next schedule entries while staging slots are
// available: the ring holds `ring` granules in flight, so backward granules
// start loading during the (H2D-light) forward pass. Slots are reused in FIFO
// order; each reuse waits (on the H2D stream) for the slot's previous consumer.
void Engine::offload_prefetch_next(int /*after*/, bool /*backward*/) {
  OffloadState& st = *off_;
  const std::size_t g = static_cast<std::size_t>(layer_stride_);
  while (st.next_issue < st.sched.size() && st.in_flight < st.ring) {
    const int o = st.sched[st.next_issue].first;
    const bool bwd = st.sched[st.next_issue].second;
    ++st.next_issue;
    ++st.in_flight;
    const int si = st.next_slot_rr;
    st.next_slot_rr = (st.next_slot_rr + 1) % st.ring;
    OffloadSlot& sl = st.slots[static_cast<std::size_t>(si)];
    sl.layer = o;
    (bwd ? st.slot_bwd : st.slot_fwd)[static_cast<std::size_t>(o)] = si;
    if (sl.free_recorded) cuda_check(cudaStreamWaitEvent(st.h2d, sl.free_ev, 0), "wait slot free");
    // a reload waits for the previous write-back of what it reads: a shadow-form
    // forward only for the bf16 shadow (written back first), anything else for all
    if (st.wb_recorded[static_cast<std::size_t>(o)]) {
      const bool fn_shadow = !bwd && !st.fwd_master;
      cuda_check(cudaStreamWaitEvent(st.h2d, (fn_shadow ? st.wb_fn_ev : st.wb_ev)[static_cast<std::size_t>(o)], 0),
                 "wait write-back");
    }
    cudaEvent_t a = st.ev(), b = st.ev();
    cuda_check(cudaEventRecord(a, st.h2d), "event");
    // The fp32 master is needed by the backward that runs the fused AdamW; every other
    // use (forward, and backward micro-steps that only accumulate) reads the bf16
    // shadow for the GEMMs and fp32 only for the vectors (LN gains / biases, biases)
    // and the fp32 MoE gate -- unless the master form is selected.
    const bool applies = bwd && has_opt_ && micro_ == accum_n_;
    const bool shadow = !st.fwd_master && !applies;
    double* ctr = bwd ? &st.stats.bn_load : &st.stats.fn_load;
    sl.p16_loaded = shadow;
    if (!shadow) {
      copy_async(st, sl.p32.p, slow_host_p32(o), g * 4, st.h2d, true, ctr);
    } else {
      copy_async(st, sl.p16.p, slow_host_p16(o), g * 2, st.h2d, true, ctr);
      for (const auto& sg : layer_.segs) {
        const bool fp32_use = !sg.decay || (cfg_.moe.enabled() && sg.off == layer_.gate);
        if (!fp32_use) continue;
        copy_async(st, sl.p32.as<float>() + sg.off, slow_host_p32(o) + sg.off, static_cast<std::size_t>(sg.len) * 4,
                   st.h2d, true, ctr);
      }
    }
    if (bwd) {
      // An: the moments only in the micro-step that runs the fused AdamW
      if (applies) {
        copy_async(st, sl.m.p, slow_host_m(o, 0), g * 4, st.h2d, true, &st.stats.opt_load);
        copy_async(st, sl.v.p, slow_host_m(o, 1), g * 4, st.h2d, true, &st.stats.opt_load);
      }
      // accumulation: continue from the partial gradients parked by the previous micro-step
      sl.grads_loaded = st.hgrad_valid[static_cast<std::size_t>(o)] != 0;
      if (sl.grads_loaded) copy_async(st, sl.g32.p, slow_host_grad(o), g * 4, st.h2d, true, &st.stats.grad_load);
    }
    cuda_check(cudaEventRecord(b, st.h2d), "event");
    st.copies.push_back({a, b, true});
    cuda_check(cudaEventRecord(sl.loaded, st.h2d), "event");
  }
}

void Engine::offload_acquire(int o, bool backward) {
  if (res_idx_[static_cast<std::size_t>(o)] >= 0) return;
  OffloadState& st = *off_;
  std::vector<int>& map = backward ? st.slot_bwd : st.slot_fwd;
  if (map[static_cast<std::size_t>(o)] < 0) {
    // used outside the step schedule (e.g. a backward after an inference
    // forward): restart the schedule at this use
    st.sched.assign(1, {o, backward});
    st.next_issue = 0;
    st.in_flight = 0;
    offload_prefetch_next(-1, backward);
  }
  const int si = map[static_cast<std::size_t>(o)];
  st.slot_of[static_cast<std::size_t>(o)] = si;
  OffloadSlot& sl = st.slots[static_cast<std::size_t>(si)];
  cuda_check(cudaStreamWaitEvent(stream_, sl.loaded, 0), "wait loaded");
  if (!sl.p16_loaded)  // the master was staged: derive the bf16 operand on the device
    p2r_check(p2r_cast_bf16(sl.p32.as<float>(), sl.p16.p, layer_stride_, stream_), "offload bf16 operand");
  if (backward && !sl.grads_loaded) cuda_check(cudaMemsetAsync(sl.g32.p, 0, sl.g32.bytes, stream_), "zero slot grads");
}

void Engine::offload_release(int o, bool backward) {
  // resident layers need nothing: SLOW granules are staged ahead by the schedule
  if (res_idx_[static_cast<std::size_t>(o)] >= 0) return;
  OffloadState& st = *off_;
  const int si = st.slot_of[static_cast<std::size_t>(o)];
  OffloadSlot& sl = st.slots[static_cast<std::size_t>(si)];
  const std::size_t g = static_cast<std::size_t>(layer_stride_);
  (backward ? st.slot_bwd : st.slot_fwd)[static_cast<std::size_t>(o)] = -1;
  st.in_flight = std::max(0, st.in_flight - 1);
  if (!backward) {
    cuda_check(cudaEventRecord(sl.free_ev, stream_), "event");
    sl.free_recorded = true;
    offload_prefetch_next(o, false);
    return;
  }
  // An phase. The last micro-step of the accumulation window sums the replicated
  // gradient part over the data-parallel ranks, runs the fused AdamW on the staged
  // granule and writes p, m, v back; earlier micro-steps (and models without an
  // optimizer) park the partial gradients in pinned host memory instead.
  const bool apply = has_opt_ && micro_ == accum_n_;
  cudaEvent_t done = st.ev();
  if (apply) {
    if ((comm_ != nullptr || loop_ != nullptr) && ep_world_ > 1) {
      const long long repl = cfg_.moe.enabled() ? layer_.w1 : layer_.numel;
      allreduce_f32(sl.g32.as<float>(), static_cast<std::size_t>(repl));
    }
    const std::int64_t t = step_count_ + 1;
    const float bc1 = 1.0f - std::pow(b1_, static_cast<float>(t));
    const float bc2 = 1.0f - std::pow(b2_, static_cast<float>(t));
    adamw_granule(sl.p32.as<float>(), sl.g32.as<float>(), sl.m.as<float>(), sl.v.as<float>(), sl.p16.p, offload_lr_,
                  bc1, bc2);
    slow_applied_ = true;
  }
  cuda_check(cudaEventRecord(done, stream_), "event");
  cuda_check(cudaStreamWaitEvent(st.d2h, done, 0), "wait compute");
  cudaEvent_t a = st.ev(), b = st.ev();
  cuda_check(cudaEventRecord(a, st.d2h), "event");
  st.hgrad_valid[static_cast<std::size_t>(o)] = apply ? 0 : 1;
  if (apply) {
    // what a shadow-form forward reloads first (the bf16 shadow and the fp32 vectors /
    // gate): the next step's forward waits only for these, so the fp32 master and the
    // moments drain under that forward instead of stalling it
    if (!st.fwd_master) {
      copy_async(st, slow_host_p16(o), sl.p16.p, g * 2, st.d2h, false, &st.stats.writeback);
      for (const auto& sg : layer_.segs) {
        const bool fp32_use = !sg.decay || (cfg_.moe.enabled() && sg.off == layer_.gate);
        if (fp32_use)
          copy_async(st, slow_host_p32(o) + sg.off, sl.p32.as<float>() + sg.off, static_cast<std::size_t>(sg.len) * 4,
                     st.d2h, false, &st.stats.writeback);
      }
    }
    cuda_check(cudaEventRecord(st.wb_fn_ev[static_cast<std::size_t>(o)], st.d2h), "event");
    copy_async(st, slow_host_p32(o), sl.p32.p, g * 4, st.d2h, false, &st.stats.writeback);
    copy_async(st, slow_host_m(o, 0), sl.m.p, g * 4, st.d2h, false, &st.stats.writeback);
    copy_async(st, slow_host_m(o, 1), sl.v.p, g * 4, st.d2h, false, &st.stats.writeback);
  } else {
    if (!st.hg) {
      const std::size_t n = g * st.slow_list.size();
      cuda_check(cudaMallocHost(reinterpret_cast<void**>(&st.hg), n * 4), "pinned grads");
      std::memset(st.hg, 0, n * 4);
    }
    // (the weights are unchanged: the next micro-step's forward needs no wait)
    cuda_check(cudaEventRecord(st.wb_fn_ev[static_cast<std::size_t>(o)], st.d2h), "event");
    copy_async(st, slow_host_grad(o), sl.g32.p, g * 4, st.d2h, false, &st.stats.grad_offload);
  }
  cuda_check(cudaEventRecord(b, st.d2h), "event");
  st.copies.push_back({a, b, false});
  cuda_check(cudaEventRecord(st.wb_ev[static_cast<std::size_t>(o)], st.d2h), "event");
  st.wb_recorded[static_cast<std::size_t>(o)] = 1;
  cuda_check(cudaEventRecord(sl.free_ev, st.d2h), "event");
  sl.free_recorded = true;
  offload_prefetch_next(o, true);
}

void Engine::offload_finish_step() {}

void offload_sync(const OffloadState& st) {
  if (st.h2d) cuda_check(cudaStreamSynchronize(st.h2d), "sync h2d");
  if (st.d2h) cuda_check(cudaStreamSynchronize(st.d2h), "sync d2h");
}

OffloadStats Engine::offload_stats() {
  OffloadStats out;
  if (!off_) return out;
  OffloadState& st = *off_;
  cuda_check(cudaStreamSynchronize(st.h2d), "sync h2d");
  cuda_check(cudaStreamSynchronize(st.d2h), "sync d2h");
  out = st.stats;
  for (const auto& c : st.copies) {
    float ms = 0;
    cuda_check(cudaEventElapsedTime(&ms, c.a, c.b), "event time");
    (c.h2d ? out.h2d_ms : out.d2h_ms) += ms;
  }
  out.copies = static_cast<std::int64_t>(st.copies.size());
  return out;
}

void Engine::offload_stats_reset() {
  if (!off_) return;
  OffloadState& st = *off_;
  cuda_check(cudaStreamSynchronize(st.h2d), "sync h2d");
  cuda_check(cudaStreamSynchronize(st.d2h), "sync d2h");
  st.stats = OffloadStats{};
  st.copies.clear();
  st.pool_used = 0;
}

void Engine::set_offload_skip_copies(bool skip) {
  if (off_) off_->skip = skip;
}

std::int64_t Engine::device_param_bytes() const {
  std::int64_t b = static_cast<std::int64_t>(emb_p_.bytes + emb_g_.bytes + emb_p16_.bytes + emb_m_.bytes +
                                             emb_v_.bytes + lay_p_.bytes + lay_g_.bytes + lay_p16_.bytes +
                                             lay_m_.bytes + lay_v_.bytes);
  if (off_)
    for (const auto& s : off_->slots)
      b += static_cast<std::int64_t>(s.p32.bytes + s.g32.bytes + s.m.bytes + s.v.bytes + s.p16.bytes);
  return b;
}

}  // namespace p2r
