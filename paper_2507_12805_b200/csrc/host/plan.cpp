#include "plan.hpp"

#include <algorithm>
#include <functional>
#include <queue>

namespace pmklc_b200 {

Plan plan_chunks(uint64_t m, uint32_t workers, uint32_t bs, uint32_t t, uint16_t myriad) {
  Plan p;
  p.t = t;
  p.myriad = myriad;
  if (m == 0) {
    p.bs = 1;
    return p;
  }
  const uint64_t per_worker = uint64_t(bs) * (uint64_t(t) + 1);
  const uint64_t w = std::min<uint64_t>(workers, std::max<uint64_t>(1, m / per_worker));
  const uint64_t base = m / w, rem = m % w;
  uint64_t start = 0;
  for (uint64_t i = 0; i < w; ++i) {
    const uint64_t len = base + (i < rem ? 1 : 0);
    p.start.push_back(start);
    p.len.push_back(len);
    start += len;
  }
  p.bs = uint32_t(std::min<uint64_t>(bs, std::max<uint64_t>(1, base / (uint64_t(t) + 1))));
  return p;
}

Schedule make_schedule(const Plan& p, bool smp_on) {
  Schedule s;
  const size_t W = p.len.size();
  s.L.resize(W);
  s.M.resize(W);
  s.offset.resize(W);
  s.src.resize(W);
  s.src_steps.resize(W);
  s.inbound_nonempty.resize(W);
  s.emits.resize(W);
  for (size_t c = 0; c < W; ++c) {
    s.L[c] = p.len[c] / p.bs;
    s.M[c] = s.L[c] > p.t ? s.L[c] - p.t : 0;
  }
  for (size_t c = 0; c < W; ++c) {
    // reference: chunk c emits its snapshot iff SMP is on, it is not the last
    // chunk, and it reaches step snap (steps_done counts warm-up steps)
    const uint64_t snap = smp_on ? p.snapshot_step(c) : 0;
    s.emits[c] = smp_on && c + 1 < W && snap <= s.L[c];
    if (c == 0 || !smp_on) {
      s.src[c] = -1;
      s.src_steps[c] = 0;
      s.offset[c] = 0;
      s.inbound_nonempty[c] = 0;
      continue;
    }
    const uint64_t psnap = p.snapshot_step(c - 1);
    s.inbound_nonempty[c] = s.emits[c - 1] || s.inbound_nonempty[c - 1];
    if (s.emits[c - 1] && psnap > p.t) {
      // snapshot after psnap - t model steps of chunk c-1
      s.src[c] = int64_t(c - 1);
      s.src_steps[c] = psnap - p.t;
      s.offset[c] = s.offset[c - 1] + int64_t(psnap - p.t);
    } else {
      // snapshot taken during warm-up (== c-1's inbound) or never taken
      // (inbound forwarded unchanged): same state as chunk c-1 started from
      s.src[c] = s.src[c - 1];
      s.src_steps[c] = s.src_steps[c - 1];
      s.offset[c] = s.offset[c - 1];
    }
  }
  int64_t ticks = 0;
  for (size_t c = 0; c < W; ++c)
    if (s.M[c]) ticks = std::max<int64_t>(ticks, s.offset[c] + int64_t(s.M[c]));
  s.ticks = ticks;
  // CSR lists
  std::vector<std::vector<uint32_t>> act(static_cast<size_t>(ticks));
  std::vector<std::vector<int32_t>> hand(static_cast<size_t>(ticks));
  for (size_t c = 0; c < W; ++c) {
    if (!s.M[c]) continue;
    for (uint64_t q = 0; q < s.M[c]; ++q) act[size_t(s.offset[c] + int64_t(q))].push_back(uint32_t(c));
    if (s.src[c] >= 0) {
      hand[size_t(s.offset[c])].push_back(int32_t(s.src[c]));
      hand[size_t(s.offset[c])].push_back(int32_t(c));
    }
  }
  s.act_ptr.push_back(0);
  s.hand_ptr.push_back(0);
  for (int64_t t = 0; t < ticks; ++t) {
    s.act.insert(s.act.end(), act[size_t(t)].begin(), act[size_t(t)].end());
    s.act_ptr.push_back(uint32_t(s.act.size()));
    s.hand.insert(s.hand.end(), hand[size_t(t)].begin(), hand[size_t(t)].end());
    s.hand_ptr.push_back(uint32_t(s.hand.size() / 2));
    s.max_active = std::max<uint32_t>(s.max_active, uint32_t(act[size_t(t)].size()));
  }
  return s;
}

RankPlan plan_rank(const Schedule& s, int rank, int world) {
  RankPlan rp;
  rp.rank = rank;
  rp.world = world;
  rp.local = s;
  const size_t W = s.L.size();
  rp.mine.resize(W);
  for (size_t c = 0; c < W; ++c) rp.mine[c] = owner_of(c, world) == rank;
  Schedule& l = rp.local;
  l.act.clear();
  l.hand.clear();
  l.act_ptr.assign(1, 0);
  l.hand_ptr.assign(1, 0);
  l.max_active = 0;
  for (int64_t t = 0; t < s.ticks; ++t) {
    uint32_t n = 0;
    for (uint32_t i = s.act_ptr[size_t(t)]; i < s.act_ptr[size_t(t) + 1]; ++i)
      if (rp.mine[s.act[i]]) {
        l.act.push_back(s.act[i]);
        ++n;
      }
    l.act_ptr.push_back(uint32_t(l.act.size()));
    l.max_active = std::max(l.max_active, n);
    for (uint32_t i = s.hand_ptr[size_t(t)]; i < s.hand_ptr[size_t(t) + 1]; ++i) {
      const int32_t src = s.hand[2 * i], dst = s.hand[2 * i + 1];
      const bool ms = rp.mine[size_t(src)], md = rp.mine[size_t(dst)];
      if (ms && md) {
        l.hand.push_back(src);
        l.hand.push_back(dst);
      } else if (ms) {
        rp.ops.push_back(CommOp{t, src, dst, owner_of(size_t(dst), world), true});
      } else if (md) {
        rp.ops.push_back(CommOp{t, src, dst, owner_of(size_t(src), world), false});
      }
    }
    l.hand_ptr.push_back(uint32_t(l.hand.size() / 2));
  }
  return rp;
}

Slots assign_slots(const Schedule& s, const std::vector<uint8_t>* mine) {
  const size_t W = s.L.size();
  Slots out;
  out.of.assign(W, -1);
  std::vector<int64_t> end(W, -1);
  for (size_t c = 0; c < W; ++c)
    if (s.M[c] && (!mine || (*mine)[c])) end[c] = s.offset[c] + int64_t(s.M[c]) - 1;
  for (size_t c = 0; c < W; ++c) {  // handoff sources stay live until the copy
    const int64_t src = s.src[c];
    if (src >= 0 && s.M[c] && end[size_t(src)] >= 0)
      end[size_t(src)] = std::max(end[size_t(src)], s.offset[c]);
  }
  std::vector<size_t> order;
  for (size_t c = 0; c < W; ++c)
    if (end[c] >= 0) order.push_back(c);
  std::stable_sort(order.begin(), order.end(),
                   [&](size_t a, size_t b) { return s.offset[a] < s.offset[b]; });
  // busy slots keyed by their last tick; a slot is free for an interval
  // starting strictly after it
  using E = std::pair<int64_t, int32_t>;
  std::priority_queue<E, std::vector<E>, std::greater<E>> busy;
  std::vector<int32_t> free_slots;
  for (size_t c : order) {
    while (!busy.empty() && busy.top().first < s.offset[c]) {
      free_slots.push_back(busy.top().second);
      busy.pop();
    }
    int32_t sl;
    if (!free_slots.empty()) {
      std::sort(free_slots.begin(), free_slots.end(), std::greater<int32_t>());
      sl = free_slots.back();  // lowest free slot: deterministic
      free_slots.pop_back();
    } else {
      sl = out.count++;
    }
    out.of[c] = sl;
    busy.push({end[c], sl});
  }
  return out;
}

}  // namespace pmklc_b200
