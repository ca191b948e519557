// Chunk planning (PMKLC-M data-block partitioning) and the tick schedule that
// realises Step-wise Model Passing on the device.
//
// plan_chunks / snapshot_step restate pipeline.cpp:26-52 exactly. The
// schedule turns the reference's thread-per-chunk promise chain
// (run_chunks, pipeline.cpp:253-294) into a deterministic global clock: at
// tick T every chunk whose model phase covers T performs one coded batch step,
// and a chunk's inbound state is copied from its source chunk at the tick its
// source reaches the snapshot step. Warm-up positions (j < t) never touch the
// model, so they are coded for all chunks before tick 0.
#pragma once
#include <cstdint>
#include <vector>

namespace pmklc_b200 {

struct Plan {
  std::vector<uint64_t> start, len;
  uint32_t bs = 1, t = 0;
  uint16_t myriad = 0;
  uint64_t snapshot_step(size_t i) const {
    const uint64_t steps = len[i] / bs;
    const uint64_t s = (uint64_t(myriad) * steps + 9999) / 10000;
    return s ? s : 1;
  }
};

Plan plan_chunks(uint64_t m, uint32_t workers, uint32_t bs, uint32_t t, uint16_t myriad);

struct Schedule {
  std::vector<uint64_t> L, M;         // batch steps, model steps per chunk
  std::vector<int64_t> offset;        // tick of the chunk's first model step
  std::vector<int64_t> src;           // inbound state source chunk, -1 = seeded init
  std::vector<uint64_t> src_steps;    // model steps the source had completed
  std::vector<uint8_t> inbound_nonempty, emits;  // reference stats semantics
  int64_t ticks = 0;
  std::vector<uint32_t> act_ptr, act;        // CSR: chunks stepping at each tick
  std::vector<uint32_t> hand_ptr;            // CSR into hand (pairs src,dst)
  std::vector<int32_t> hand;                 // flattened (src, dst) pairs
  uint32_t max_active = 0;
};

// smp_on: myriad > 0 (the container's smp_per_myriad field)
Schedule make_schedule(const Plan& p, bool smp_on);

// PMKLC-M across ranks (one GPU each): chunk c is owned by rank c % world
// (round robin, so the SMP wavefront of consecutive chunks spreads over all
// GPUs). A rank steps only its own chunks; an SMP handoff between chunks on
// different ranks becomes a point-to-point transfer of the state slot at the
// handoff tick (sender: state after src_steps model steps; receiver: the
// destination slot, before its first model step). Both sides derive the same
// op list from the same schedule, in the same order, so sends and receives
// match without negotiation.
struct CommOp {
  int64_t tick;
  int32_t src, dst, peer;
  bool send;
};
struct RankPlan {
  int rank = 0, world = 1;
  Schedule local;            // act / hand filtered to this rank (hand: local->local only)
  std::vector<CommOp> ops;   // cross-rank handoffs touching this rank, tick order
  std::vector<uint8_t> mine; // per chunk: owned by this rank
};
inline int owner_of(size_t chunk, int world) { return int(chunk % size_t(world)); }
RankPlan plan_rank(const Schedule& s, int rank, int world);

// Device memory by concurrency, not by chunk count: chunk c holds a state /
// tape slot from its first model tick (where its inbound state is copied in)
// through its last model tick, extended to the last tick at which its state
// is the source of a handoff (local or, on the sending rank, remote). Slots
// are assigned greedily by start tick, so their number is the peak number of
// live chunks (max_active plus pending handoff sources). Chunks that never
// step (or are not `mine`) get -1.
struct Slots {
  std::vector<int32_t> of;  // per chunk
  int32_t count = 0;
};
Slots assign_slots(const Schedule& s, const std::vector<uint8_t>* mine = nullptr);

}  // namespace pmklc_b200
