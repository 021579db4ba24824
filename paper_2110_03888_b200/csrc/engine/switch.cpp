// Switch detector decision logic (SPEC.md:255-259
// [TYPE] SwitchPolicy, :285-293 [OP] detect_switch; §3.2.3).
//
// Every eval_interval_steps the controller snapshots the Pseudo model, delinks
// it, trains the Real model for trial_budget_steps, reverts, trains the Pseudo
// model for the same wall time, and compares the two loss slopes. The slope is
// the least-squares slope of evaluation loss against wall time over the last
// slope_window points (SPEC design decision); the switch fires when the Real
// stage decreases loss faster, i.e. real_slope < pseudo_slope.
#include <stdexcept>
#include <vector>

#include "p2r/engine.hpp"

namespace p2r {

void SwitchPolicy::validate() const {
  if (eval_interval_steps <= 0 || trial_budget_steps <= 0 || slope_window <= 0)
    throw std::invalid_argument("switch policy: all fields must be positive");
  if (trial_budget_steps > eval_interval_steps)
    throw std::invalid_argument("switch policy: trial_budget_steps must not exceed eval_interval_steps");
}

double loss_slope(const std::vector<double>& time_s, const std::vector<double>& loss, int window) {
  if (time_s.size() != loss.size()) throw std::invalid_argument("loss_slope: series lengths differ");
  const std::size_t n = time_s.size();
  if (n < 2) throw std::invalid_argument("loss_slope: need at least two points");
  const std::size_t w = window > 0 && static_cast<std::size_t>(window) < n ? static_cast<std::size_t>(window) : n;
  const std::size_t b = n - w;
  double mt = 0, ml = 0;
  for (std::size_t i = b; i < n; ++i) {
    mt += time_s[i];
    ml += loss[i];
  }
  mt /= static_cast<double>(w);
  ml /= static_cast<double>(w);
  double sxy = 0, sxx = 0;
  for (std::size_t i = b; i < n; ++i) {
    sxy += (time_s[i] - mt) * (loss[i] - ml);
    sxx += (time_s[i] - mt) * (time_s[i] - mt);
  }
  if (sxx == 0) throw std::invalid_argument("loss_slope: time points must differ");
  return sxy / sxx;
}

SwitchDecision switch_criterion(const std::vector<double>& pseudo_t, const std::vector<double>& pseudo_loss,
                                const std::vector<double>& real_t, const std::vector<double>& real_loss,
                                const SwitchPolicy& policy) {
  policy.validate();
  SwitchDecision d;
  d.pseudo_slope = loss_slope(pseudo_t, pseudo_loss, policy.slope_window);
  d.real_slope = loss_slope(real_t, real_loss, policy.slope_window);
  d.fire = d.real_slope < d.pseudo_slope;  // Real decreases loss faster per unit time
  return d;
}

bool switch_evaluation_due(const SwitchPolicy& policy, std::int64_t step) {
  policy.validate();
  return step > 0 && step % policy.eval_interval_steps == 0;
}

}  // namespace p2r
