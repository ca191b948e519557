// TEST INFRASTRUCTURE — NOT PRODUCT CODE.
//
// extern "C" access to the seeded synthetic-DNA generators
// (paper_2507_12805_b200/csrc/host/synth.cpp, compiled into the checker
// libraries from that one source file) so that bench.py's reference arm and
// the golden scripts can build the benchmark inputs without loading the
// product library. Input generation only; nothing here touches the coding path.
#include <cstdint>

namespace pmklc_b200 {
void synth_markov3(uint8_t*, uint64_t, uint64_t);
void synth_uniform(uint8_t*, uint64_t, uint64_t);
void synth_genome(uint8_t*, uint64_t, uint64_t, uint32_t);
void synth_species(uint8_t*, uint64_t, uint64_t, uint64_t);
}  // namespace pmklc_b200

#ifndef SYNTH_PREFIX
#error "define SYNTH_PREFIX"
#endif
#define CAT2(a, b) a##b
#define CAT(a, b) CAT2(a, b)

extern "C" {
void CAT(SYNTH_PREFIX, synth_markov3)(uint8_t* o, uint64_t n, uint64_t s) {
  pmklc_b200::synth_markov3(o, n, s);
}
void CAT(SYNTH_PREFIX, synth_uniform)(uint8_t* o, uint64_t n, uint64_t s) {
  pmklc_b200::synth_uniform(o, n, s);
}
void CAT(SYNTH_PREFIX, synth_genome)(uint8_t* o, uint64_t n, uint64_t s, uint32_t seg) {
  pmklc_b200::synth_genome(o, n, s, seg);
}
void CAT(SYNTH_PREFIX, synth_species)(uint8_t* o, uint64_t n, uint64_t s, uint64_t block) {
  pmklc_b200::synth_species(o, n, s, block);
}
}
