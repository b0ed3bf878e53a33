// schedule.cu -- dependency-driven generation of the stage programs (see schedule.h).
#include "schedule.h"

namespace xp {

void ScheduleSim::reset(int K, int T, bool gpipe, const std::vector<bool>& record) {
  K_ = K; T_ = T; gpipe_ = gpipe;
  nf_.assign(K, 1);
  nb_.assign(K, 1);
  record_ = record;
  record_.resize(K, true);
  q_.assign(K, {});
  q0_.assign(K, 0);
}

void ScheduleSim::tick() {
  // decisions read the state at the start of the tick: an op finished in this tick is not yet
  // visible to the neighbours (one op per stage per unit of time)
  const std::vector<int64_t> f0 = nf_, b0 = nb_;
  for (int k = 0; k < K_; ++k) {
    const int64_t uf = f0[k], ub = b0[k];
    const bool in_ready = k == 0 || f0[k - 1] > uf;                       // activation of F(uf) arrived
    const bool grad_ready = ub < uf && (k + 1 < K_ ? b0[k + 1] > ub : f0[k] > ub);  // gradient of B(ub)
    bool do_f = false, do_b = false;
    if (!gpipe_) {
      // 1F1B: a runnable backward first; a forward while the stash has room (K-k in flight)
      if (grad_ready) do_b = true;
      else if (in_ready && uf - ub < K_ - k) do_f = true;
    } else {
      const int64_t tf = (uf - 1) / T_, tb = (ub - 1) / T_;               // 0-based mini-batches
      const bool f_ok = in_ready && ub > tf * T_;                           // flushed through t-1
      const bool b_ok = grad_ready && uf > (tb + 1) * T_;                   // all T forwards of t done
      if (f_ok) do_f = true;
      else if (b_ok) do_b = true;
    }
    if (do_f) {
      if (record_[k]) q_[k].emplace_back(0, uf);
      nf_[k] = uf + 1;
    } else if (do_b) {
      if (record_[k]) q_[k].emplace_back(1, ub);
      nb_[k] = ub + 1;
    }
  }
}

void ScheduleSim::op_at(int k, int64_t p, int* op, int64_t* u) {
  while (q0_[k] < p && !q_[k].empty()) { q_[k].pop_front(); ++q0_[k]; }
  // positions skipped without being read (a replayed graph advanced them): generate and drop
  while (q0_[k] + (int64_t)q_[k].size() <= p) {
    tick();
    while (q0_[k] < p && !q_[k].empty()) { q_[k].pop_front(); ++q0_[k]; }
  }
  *op = q_[k][p - q0_[k]].first;
  *u = q_[k][p - q0_[k]].second;
}

}  // namespace xp
