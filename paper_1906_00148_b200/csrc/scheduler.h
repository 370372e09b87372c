// scheduler.h — circuit scheduler for SHE's encrypted layers (§3):
// builds the Boolean gate DAG of a layer (shift = rewiring, negation = literal
// flag, constants folded), levelises it ASAP, assigns wire-table slots with
// liveness reuse, and hands each level to an executor (the GPU engine, or the
// clear-bit simulator used by the tests).
#pragma once
#include <stdint.h>

#include <vector>

namespace sched {

// A literal: wire id (bits 0..30) + negation flag (bit 31).  Wire 0 is the
// constant FALSE (a trivial ciphertext (0, -1/8)); !wire0 is TRUE.
struct Lit {
  uint32_t v;
  bool operator==(const Lit& o) const { return v == o.v; }
  bool operator!=(const Lit& o) const { return v != o.v; }
  uint32_t wire() const { return v & 0x7FFFFFFFu; }
  bool neg() const { return (v >> 31) != 0; }
  Lit operator!() const { return Lit{v ^ 0x80000000u}; }
};
constexpr Lit F{0};
constexpr Lit T{0x80000000u};
inline bool is_const(Lit a) { return a.wire() == 0; }

// Only AND, XOR, MUX gates are emitted: OR/NAND/NOR/XNOR/NOT are negation
// flags on literals (free), so every emitted gate is one bootstrapped op.
enum Op : uint8_t { G_AND = 0, G_XOR = 4, G_MUX = 6 };  // she_op codes

struct Gate {
  uint8_t op;
  Lit in[3];
  uint32_t out;  // wire id
};

using Word = std::vector<Lit>;  // LSB first, two's complement

struct Stats {
  uint64_t gates = 0, br_lanes = 0, levels = 0, max_width = 0, min_width = 0;
};

class Circuit {
 public:
  Circuit() : level_(1, 0), input_index_(1, 0xFFFFFFFFu) {}
  // a new circuit input (level 0); inputs are numbered 0, 1, ... in creation order
  Lit new_input() {
    const uint32_t w = (uint32_t)level_.size();
    level_.push_back(0);
    input_index_.push_back(num_inputs_++);
    return Lit{w};
  }
  uint32_t num_inputs() const { return num_inputs_; }
  uint32_t input_index(uint32_t wire) const { return input_index_[wire]; }  // ~0u if not an input
  uint32_t num_wires() const { return (uint32_t)level_.size(); }
  const std::vector<Gate>& gates() const { return gates_; }
  uint32_t level(Lit a) const { return level_[a.wire()]; }

  Lit AND(Lit a, Lit b);
  Lit OR(Lit a, Lit b) { return !AND(!a, !b); }  // De Morgan: negation flags are free
  Lit XOR(Lit a, Lit b);
  Lit MUX(Lit s, Lit a, Lit b);  // s ? a : b

  // words
  static Lit bit(const Word& w, size_t i) { return w.empty() ? F : (i < w.size() ? w[i] : w.back()); }
  Word add(const Word& a, const Word& b, Lit cin, int width);  // ripple carry, FA = XOR, XOR, MUX
  Word neg_bits(const Word& a) const;
  Lit less_than(const Word& x, const Word& y);                // signed x < y (comparator chain)
  Word max(const Word& x, const Word& y);                      // comparator sign + per-bit MUX

 private:
  Lit emit(uint8_t op, Lit a, Lit b, Lit c);
  uint32_t num_inputs_ = 0;
  std::vector<uint32_t> level_;        // per wire
  std::vector<uint32_t> input_index_;  // per wire
  std::vector<Gate> gates_;
};

// Shift-accumulate neuron: sum_k sign_k (x_k >> e_k)
// with a balanced mixed-bitwidth adder tree (width min(max(wa, wb) + 1, cap)),
// negative terms as !(x >> e) with the +1 injected as an adder carry-in.
struct Term {
  Word x;        // input word (unsigned if !is_signed: value bits only)
  bool is_signed;
  int8_t code;   // 0 zero weight, +-(e+1)
};
Word shift_accumulate(Circuit& c, const std::vector<Term>& terms, int cap);
Word relu(Circuit& c, const Word& v);  // unsigned result, width w-1: AND(x_i, !sign)

// Levelised, slot-assigned program of a circuit.
struct Program {
  uint32_t num_slots = 0;     // wire-table slots needed (inputs first, then slot 0 = const)
  std::vector<uint32_t> level_begin;  // gates of level L: [level_begin[L], level_begin[L+1])
  std::vector<uint8_t> ops;
  std::vector<uint32_t> ins;    // 3 per gate: slot | neg << 31
  std::vector<uint32_t> outs;   // slot per gate
  std::vector<uint32_t> out_lits;  // requested outputs: slot | neg << 31
  Stats stats;
};
// Slot layout: slot 0 = constant FALSE trivial ciphertext, slots 1..I = inputs.
Program compile(const Circuit& c, const std::vector<Lit>& outputs);

}  // namespace sched
