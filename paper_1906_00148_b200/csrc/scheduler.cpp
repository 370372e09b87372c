// scheduler.cpp — SHE's encrypted layers as levelised bootstrapped-gate circuits.
//
// PAPER.md §3: ReLU and max-pool units built from TFHE gates (:92, :110, F2);
// log-quantised weights turn products into shifts, which on bit-wise TFHE
// ciphertexts are free rewiring (:118, :142); a mixed-bitwidth adder tree
// whose level-n adders are (b+n) bits (:147, :149).  Readings:
// R11 unsigned pixels zero-extended, R12 term = sign * (x >> e), R13 wrap at
// the accumulator cap, ReLU = AND with !sign, max = subtract
// comparator + per-bit MUX, negation via carry-in
// (SPEC.md:438), full adder FA-B = XOR, XOR, MUX (4 blind rotations).
#include "scheduler.h"

#include <stdint.h>
#include <string.h>

#include <algorithm>
#include <functional>
#include <new>
#include <vector>

#include "common.h"
#include "engine.h"

namespace sched {

// ---------------------------------------------------------------------------
// gates with constant folding
// ---------------------------------------------------------------------------
Lit Circuit::emit(uint8_t op, Lit a, Lit b, Lit c) {
  const uint32_t w = (uint32_t)level_.size();
  uint32_t lv = std::max(level_[a.wire()], level_[b.wire()]);
  if (op == G_MUX) lv = std::max(lv, level_[c.wire()]);
  level_.push_back(lv + 1);
  input_index_.push_back(0xFFFFFFFFu);
  gates_.push_back(Gate{op, {a, b, c}, w});
  return Lit{w};
}

Lit Circuit::AND(Lit a, Lit b) {
  if (a == F || b == F) return F;
  if (a == T) return b;
  if (b == T) return a;
  if (a == b) return a;
  if (a == !b) return F;
  return emit(G_AND, a, b, F);
}

Lit Circuit::XOR(Lit a, Lit b) {
  if (is_const(a)) return a == F ? b : !b;
  if (is_const(b)) return b == F ? a : !a;
  if (a == b) return F;
  if (a == !b) return T;
  // normalise negations onto the output: XOR(!a, b) = !XOR(a, b)
  bool flip = a.neg() != b.neg();
  Lit g = emit(G_XOR, Lit{a.wire()}, Lit{b.wire()}, F);
  return flip ? !g : g;
}

Lit Circuit::MUX(Lit s, Lit a, Lit b) {
  if (s == T) return a;
  if (s == F) return b;
  if (a == b) return a;
  if (a == !b) return XOR(s, b);  // s ? !b : b = s XOR b
  if (a == F) return AND(!s, b);
  if (a == T) return OR(s, b);
  if (b == F) return AND(s, a);
  if (b == T) return OR(!s, a);
  if (s == a) return OR(s, b);   // s ? s : b = s | b
  if (s == !a) return AND(!s, b);
  if (s == b) return AND(s, a);
  if (s == !b) return OR(!s, a);
  if (s.neg()) return emit(G_MUX, !s, b, a);
  return emit(G_MUX, s, a, b);
}

Word Circuit::neg_bits(const Word& a) const {
  Word r(a.size());
  for (size_t i = 0; i < a.size(); ++i) r[i] = !a[i];
  return r;
}

// Ripple-carry adder, result width `width` (bits beyond are dropped: wrap).
// FA-B: t = a ^ b, s = t ^ c, c' = t ? c : a  (2 XOR + 1 MUX = 4 BR).
Word Circuit::add(const Word& a, const Word& b, Lit cin, int width) {
  Word s(width);
  Lit c = cin;
  for (int i = 0; i < width; ++i) {
    const Lit ai = bit(a, i), bi = bit(b, i);
    const Lit t = XOR(ai, bi);
    s[i] = XOR(t, c);
    if (i + 1 < width) {
      if (c == F) c = AND(ai, bi);
      else if (c == T) c = OR(ai, bi);
      else c = MUX(t, c, ai);
    }
  }
  return s;
}

// Signed x < y: the sign of x - y = x + !y + 1 computed on max(w)+1 bits,
// carry chain only (the subtract comparator of the max-pool unit).
Lit Circuit::less_than(const Word& x, const Word& y) {
  const size_t w = std::max(x.size(), y.size());
  Lit c = T;
  for (size_t i = 0; i < w; ++i) {
    const Lit a = bit(x, i), b = !bit(y, i);
    const Lit t = XOR(a, b);
    if (c == F) c = AND(a, b);
    else if (c == T) c = OR(a, b);
    else c = MUX(t, c, a);
  }
  // bit w of the difference: sign-extended operands
  return XOR(XOR(bit(x, w), !bit(y, w)), c);
}

Word Circuit::max(const Word& x, const Word& y) {
  const size_t w = std::max(x.size(), y.size());
  const Lit lt = less_than(x, y);
  Word z(w);
  for (size_t i = 0; i < w; ++i) z[i] = MUX(lt, bit(y, i), bit(x, i));
  return z;
}

// ---------------------------------------------------------------------------
// neurons
// ---------------------------------------------------------------------------
Word shift_accumulate(Circuit& c, const std::vector<Term>& terms, int cap) {
  struct Node {
    Word w;
    int pending;  // +1s not yet added (negated terms)
  };
  std::vector<Node> level;
  for (const Term& t : terms) {
    if (t.code == 0) continue;
    const int e = std::abs(t.code) - 1;
    Word y;
    if (t.is_signed) {  // arithmetic shift: bits [e, w) (sign replicated if e >= w)
      const int w = (int)t.x.size();
      if (e >= w) y.push_back(t.x.back());
      else y.assign(t.x.begin() + e, t.x.end());
    } else {  // unsigned: logical shift, then a constant-0 sign bit
      const int w = (int)t.x.size();
      if (e >= w) continue;  // term is 0
      y.assign(t.x.begin() + e, t.x.end());
      y.push_back(F);
    }
    if ((int)y.size() > cap) y.resize(cap);  // wrap at the cap (R13)
    if (t.code < 0) level.push_back(Node{c.neg_bits(y), 1});  // -y = !y + 1
    else level.push_back(Node{y, 0});
  }
  if (level.empty()) return Word{F};
  while (level.size() > 1) {
    std::vector<Node> next;
    for (size_t k = 0; k + 1 < level.size(); k += 2) {
      const Node& a = level[k];
      const Node& b = level[k + 1];
      const int width = std::min<int>((int)std::max(a.w.size(), b.w.size()) + 1, cap);
      int pend = a.pending + b.pending;
      Lit cin = F;
      if (pend > 0) {
        cin = T;
        pend -= 1;
      }
      next.push_back(Node{c.add(a.w, b.w, cin, width), pend});
    }
    if (level.size() % 2) next.push_back(level.back());
    level.swap(next);
  }
  Node root = level[0];
  if (root.pending > 0) {  // at most 1 (a binary tree absorbs all but one)
    const int width = std::min<int>((int)root.w.size() + 1, cap);
    Word k(width, F);
    k[0] = T;
    for (int i = 1; i < width && (root.pending >> i); ++i) k[i] = ((root.pending >> i) & 1) ? T : F;
    root.w = c.add(root.w, k, F, width);
  }
  return root.w;
}

Word relu(Circuit& c, const Word& v) {
  const Lit sign = v.back();
  Word r(v.size() - 1);
  for (size_t i = 0; i + 1 < v.size(); ++i) r[i] = c.AND(v[i], !sign);
  return r;
}

// ---------------------------------------------------------------------------
// levelise + slot allocation with liveness reuse
// ---------------------------------------------------------------------------
Program compile(const Circuit& c, const std::vector<Lit>& outputs) {
  Program p;
  const auto& gates = c.gates();
  const uint32_t nin = c.num_inputs();
  const uint32_t nw = c.num_wires();
  // liveness: keep only gates reachable from the outputs
  std::vector<uint8_t> live(nw, 0);
  for (Lit o : outputs) live[o.wire()] = 1;
  for (size_t g = gates.size(); g-- > 0;) {
    const Gate& gt = gates[g];
    if (!live[gt.out]) continue;
    live[gt.in[0].wire()] = live[gt.in[1].wire()] = 1;
    if (gt.op == G_MUX) live[gt.in[2].wire()] = 1;
  }
  uint32_t maxlv = 0;
  std::vector<uint32_t> cnt;
  for (const Gate& gt : gates) {
    if (!live[gt.out]) continue;
    const uint32_t lv = c.level(Lit{gt.out});
    if (lv >= cnt.size()) cnt.resize(lv + 1, 0);
    cnt[lv]++;
    maxlv = std::max(maxlv, lv);
  }
  // last use level of each wire (outputs: never freed)
  const uint32_t kNever = 0xFFFFFFFFu;
  std::vector<uint32_t> last(nw, 0);
  for (const Gate& gt : gates) {
    if (!live[gt.out]) continue;
    const uint32_t lv = c.level(Lit{gt.out});
    for (int j = 0; j < (gt.op == G_MUX ? 3 : 2); ++j) {
      uint32_t& l = last[gt.in[j].wire()];
      l = std::max(l, lv);
    }
  }
  for (Lit o : outputs) last[o.wire()] = kNever;
  // bucket gates by level (stable)
  p.level_begin.assign(maxlv + 2, 0);
  for (uint32_t lv = 1; lv <= maxlv; ++lv) p.level_begin[lv + 1] = p.level_begin[lv] + (lv < cnt.size() ? cnt[lv] : 0);
  p.level_begin[0] = 0;
  p.level_begin[1] = 0;
  const uint32_t total = p.level_begin[maxlv + 1];
  std::vector<uint32_t> order(total);
  {
    std::vector<uint32_t> pos(p.level_begin.begin(), p.level_begin.end());
    for (uint32_t g = 0; g < gates.size(); ++g) {
      if (!live[gates[g].out]) continue;
      order[pos[c.level(Lit{gates[g].out})]++] = g;
    }
  }
  // free lists by level
  std::vector<std::vector<uint32_t>> free_at(maxlv + 2);
  std::vector<uint32_t> slot(nw, kNever);
  slot[0] = 0;
  for (uint32_t w = 1; w < nw; ++w)
    if (c.input_index(w) != 0xFFFFFFFFu) slot[w] = 1 + c.input_index(w);
  uint32_t next_slot = 1 + nin;
  std::vector<uint32_t> free_slots;
  p.ops.resize(total);
  p.ins.resize(3 * (size_t)total);
  p.outs.resize(total);
  uint64_t lanes = 0, maxw = 0, minw = ~0ull;
  for (uint32_t lv = 1; lv <= maxlv; ++lv) {
    // wires whose last consumer ran before this level can be reused now
    for (uint32_t w : free_at[lv - 1]) free_slots.push_back(slot[w]);
    free_at[lv - 1].clear();
    const uint32_t b = p.level_begin[lv], e = p.level_begin[lv + 1];
    if (e > b) {
      maxw = std::max<uint64_t>(maxw, e - b);
      minw = std::min<uint64_t>(minw, e - b);
    }
    for (uint32_t q = b; q < e; ++q) {
      const Gate& gt = gates[order[q]];
      p.ops[q] = gt.op;
      lanes += gt.op == G_MUX ? 2 : 1;
      for (int j = 0; j < 3; ++j) {
        const Lit in = (j < 2 || gt.op == G_MUX) ? gt.in[j] : gt.in[0];
        p.ins[3 * (size_t)q + j] = slot[in.wire()] | (in.v & 0x80000000u);
      }
    }
    for (uint32_t q = b; q < e; ++q) {
      const uint32_t w = gates[order[q]].out;
      uint32_t s;
      if (!free_slots.empty()) {
        s = free_slots.back();
        free_slots.pop_back();
      } else {
        s = next_slot++;
      }
      slot[w] = s;
      p.outs[q] = s;
      if (last[w] != kNever) {
        // last[w] == 0 cannot happen for a live non-output wire
        free_at[std::min(last[w], maxlv + 1)].push_back(w);
      }
    }
  }
  p.num_slots = next_slot;
  p.out_lits.resize(outputs.size());
  for (size_t o = 0; o < outputs.size(); ++o)
    p.out_lits[o] = slot[outputs[o].wire()] | (outputs[o].v & 0x80000000u);
  p.stats.gates = total;
  p.stats.br_lanes = lanes;
  p.stats.levels = maxlv;
  p.stats.max_width = maxw;
  p.stats.min_width = total ? minw : 0;
  return p;
}

}  // namespace sched


// ---------------------------------------------------------------------------
// layers: tiles of neurons -> circuit -> program -> executor
// ---------------------------------------------------------------------------
namespace {

using namespace sched;

struct Executor {
  virtual ~Executor() {}
  // Run a compiled tile.  input_bits[k] = layer-input bit (slot) of circuit
  // input k; outputs go to layer-output bit positions [out_first, +n).
  virtual she_status run(const Program& p, const std::vector<uint32_t>& input_bits,
                         size_t out_first) = 0;
};

struct ClearExec : Executor {
  const uint8_t* in = nullptr;
  uint8_t* out = nullptr;
  she_status run(const Program& p, const std::vector<uint32_t>& input_bits,
                 size_t out_first) override {
    std::vector<uint8_t> table(p.num_slots, 0);
    for (size_t k = 0; k < input_bits.size(); ++k) table[1 + k] = in[input_bits[k]] & 1;
    for (size_t lv = 1; lv + 1 < p.level_begin.size(); ++lv) {
      for (uint32_t q = p.level_begin[lv]; q < p.level_begin[lv + 1]; ++q) {
        uint8_t x[3];
        for (int j = 0; j < 3; ++j) {
          const uint32_t v = p.ins[3 * (size_t)q + j];
          x[j] = table[v & 0x7FFFFFFFu] ^ (uint8_t)(v >> 31);
        }
        uint8_t r = 0;
        switch (p.ops[q]) {
          case G_AND: r = x[0] & x[1]; break;
          case G_XOR: r = x[0] ^ x[1]; break;
          case G_MUX: r = x[0] ? x[1] : x[2]; break;
        }
        table[p.outs[q]] = r;
      }
    }
    for (size_t o = 0; o < p.out_lits.size(); ++o) {
      const uint32_t v = p.out_lits[o];
      out[out_first + o] = table[v & 0x7FFFFFFFu] ^ (uint8_t)(v >> 31);
    }
    return SHE_OK;
  }
};

struct GpuExec : Executor {
  she_ctx* ctx = nullptr;
  const uint32_t* in = nullptr;
  uint32_t* out = nullptr;
  void* stream = nullptr;
  she_status run(const Program& p, const std::vector<uint32_t>& input_bits,
                 size_t out_first) override {
    return she::engine_run_program(ctx, p, in, input_bits, out, out_first, stream);
  }
};

void add_stats(she_circuit_stats* st, const Program& p) {
  if (!st) return;
  st->gates += p.stats.gates;
  st->br_lanes += p.stats.br_lanes;
  st->levels += p.stats.levels;
  st->tiles += 1;
  st->max_level_width = std::max<uint64_t>(st->max_level_width, p.stats.max_width);
  if (p.stats.gates)
    st->min_level_width = st->min_level_width
                              ? std::min<uint64_t>(st->min_level_width, p.stats.min_width)
                              : p.stats.min_width;
}

// Maps layer-input bits to circuit inputs, created on first use.
struct InputMap {
  Circuit* c;
  std::vector<uint32_t> bits;                  // circuit input k -> layer bit
  std::vector<std::pair<uint32_t, Lit>> table;  // open addressing
  size_t used = 0;
  explicit InputMap(Circuit* cc) : c(cc), table(1 << 12, {0xFFFFFFFFu, F}) {}
  Lit operator()(uint32_t bit) {
    if (2 * (used + 1) > table.size()) grow();
    size_t h = (bit * 0x9E3779B1u) & (table.size() - 1);
    while (table[h].first != 0xFFFFFFFFu) {
      if (table[h].first == bit) return table[h].second;
      h = (h + 1) & (table.size() - 1);
    }
    Lit l = c->new_input();
    table[h] = {bit, l};
    bits.push_back(bit);
    ++used;
    return l;
  }
  void grow() {
    std::vector<std::pair<uint32_t, Lit>> old;
    old.swap(table);
    table.assign(old.size() * 2, {0xFFFFFFFFu, F});
    for (auto& kv : old) {
      if (kv.first == 0xFFFFFFFFu) continue;
      size_t h = (kv.first * 0x9E3779B1u) & (table.size() - 1);
      while (table[h].first != 0xFFFFFFFFu) h = (h + 1) & (table.size() - 1);
      table[h] = kv;
    }
  }
};

using NeuronFn = std::function<Word(Circuit&, InputMap&, uint64_t)>;

// Gates per tile: bounds the host DAG and the device wire table.
constexpr uint64_t kTileGates = 1ull << 22;

// Evaluate neurons [lo, hi) of the layer (this rank's shard), in tiles.  Each
// neuron's word is sign-extended (or truncated: never needed) to w_out bits.
she_status run_layer(uint64_t neurons, int w_out, bool signed_out, int rank, int world,
                     const NeuronFn& neuron, Executor& ex, she_circuit_stats* st) {
  const uint64_t per = (neurons + world - 1) / world;
  const uint64_t lo = std::min<uint64_t>(neurons, per * (uint64_t)rank);
  const uint64_t hi = std::min<uint64_t>(neurons, lo + per);
  uint64_t q = lo;
  while (q < hi) {
    Circuit c;
    InputMap im(&c);
    std::vector<Lit> outs;
    const uint64_t first = q;
    while (q < hi && (q == first || c.gates().size() < kTileGates)) {
      Word w = neuron(c, im, q);
      for (int i = 0; i < w_out; ++i)  // sign- or zero-extend to the layer width
        outs.push_back(i < (int)w.size() ? w[i] : (signed_out ? w.back() : F));
      ++q;
    }
    Program p = compile(c, outs);
    add_stats(st, p);
    she_status s = ex.run(p, im.bits, (size_t)first * w_out);
    if (s != SHE_OK) return s;
  }
  return SHE_OK;
}

// Weights: SHE log-quantised codes wq (0 or +-(e+1): the term sign * (x >> e)),
// or, for the TCN baseline, plaintext fixed-point
// multipliers wm = c in [-255, 255] standing for c / 2^7: the product is the
// shift-and-add over the set bits of |c| (SPEC.md:238-246 build_pc_mult),
// sign * sum_{b : bit b of |c|} (x >> (7 - b)), i.e. one SHE term of code
// sign * (7 - b + 1) per set bit.  A single-bit c = 2^(7-e) is exactly SHE's
// code e + 1.
constexpr int kTcnFrac = 7;

template <class Fn>
void for_each_code(const int8_t* wq, const int16_t* wm, size_t idx, Fn f) {
  if (!wm) {
    if (wq[idx]) f((int8_t)wq[idx]);
    return;
  }
  const int c = wm[idx];
  const int mag = c < 0 ? -c : c, sgn = c < 0 ? -1 : 1;
  for (int b = kTcnFrac; b >= 0; --b)
    if ((mag >> b) & 1) f((int8_t)(sgn * (kTcnFrac - b + 1)));
}

struct ConvGeom {
  int H, W, C, w_in, in_signed, Co, K, stride, pad, cap, relu;
  const int8_t* wq;
  const int16_t* wm = nullptr;  // TCN multipliers (wq unused when set)
  int Ho() const { return (H + 2 * pad - K) / stride + 1; }
  int Wo() const { return (W + 2 * pad - K) / stride + 1; }
};

Word conv_neuron(const ConvGeom& g, Circuit& c, InputMap& im, uint64_t q) {
  const int co = (int)(q % g.Co);
  const int ow = (int)((q / g.Co) % g.Wo());
  const int oh = (int)(q / ((uint64_t)g.Co * g.Wo()));
  std::vector<Term> terms;
  for (int kh = 0; kh < g.K; ++kh)
    for (int kw = 0; kw < g.K; ++kw) {
      const int ih = oh * g.stride - g.pad + kh, iw = ow * g.stride - g.pad + kw;
      if (ih < 0 || ih >= g.H || iw < 0 || iw >= g.W) continue;  // zero padding
      for (int ci = 0; ci < g.C; ++ci) {
        const size_t widx = (((size_t)co * g.K + kh) * g.K + kw) * g.C + ci;
        const uint32_t base = (uint32_t)((((size_t)ih * g.W + iw) * g.C + ci) * g.w_in);
        for_each_code(g.wq, g.wm, widx, [&](int8_t code) {
          Term t;
          t.is_signed = g.in_signed != 0;
          t.code = code;
          t.x.resize(g.w_in);
          const int e = std::abs(code) - 1;
          for (int b = 0; b < g.w_in; ++b)  // only bits that survive the shift are inputs
            t.x[b] = (b >= e || (t.is_signed && b == g.w_in - 1)) ? im(base + b) : F;
          terms.push_back(std::move(t));
        });
      }
    }
  Word v = shift_accumulate(c, terms, g.cap);
  return g.relu ? relu(c, v.size() > 1 ? v : Word{v[0], v[0]}) : v;
}

struct FcGeom {
  int K, w_in, in_signed, M, cap, relu;
  const int8_t* wq;
  const int16_t* wm = nullptr;  // TCN multipliers (wq unused when set)
};

Word fc_neuron(const FcGeom& g, Circuit& c, InputMap& im, uint64_t m) {
  std::vector<Term> terms;
  for (int k = 0; k < g.K; ++k) {
    for_each_code(g.wq, g.wm, (size_t)m * g.K + k, [&](int8_t code) {
      Term t;
      t.is_signed = g.in_signed != 0;
      t.code = code;
      const int e = std::abs(code) - 1;
      t.x.resize(g.w_in);
      for (int b = 0; b < g.w_in; ++b)
        t.x[b] = (b >= e || (t.is_signed && b == g.w_in - 1)) ? im((uint32_t)(k * g.w_in + b)) : F;
      terms.push_back(std::move(t));
    });
  }
  Word v = shift_accumulate(c, terms, g.cap);
  return g.relu ? relu(c, v.size() > 1 ? v : Word{v[0], v[0]}) : v;
}

// Fast width computation without building gates: mirrors shift_accumulate.
int neuron_width(const std::vector<int>& leaf_widths, int cap, bool relu_) {
  if (leaf_widths.empty()) return 1;
  std::vector<std::pair<int, int>> lv;  // (width, pending)
  for (int w : leaf_widths) lv.push_back({std::abs(w), w < 0 ? 1 : 0});
  while (lv.size() > 1) {
    std::vector<std::pair<int, int>> nx;
    for (size_t k = 0; k + 1 < lv.size(); k += 2) {
      int width = std::min(std::max(lv[k].first, lv[k + 1].first) + 1, cap);
      int pend = lv[k].second + lv[k + 1].second;
      if (pend > 0) pend -= 1;
      nx.push_back({width, pend});
    }
    if (lv.size() % 2) nx.push_back(lv.back());
    lv.swap(nx);
  }
  int w = lv[0].first;
  if (lv[0].second > 0) w = std::min(w + 1, cap);
  return relu_ ? std::max(1, w - 1) : w;
}

int leaf_width(int w_in, bool is_signed, int8_t code, int cap) {
  const int e = std::abs(code) - 1;
  int y;
  if (is_signed) y = e >= w_in ? 1 : w_in - e;
  else {
    if (e >= w_in) return 0;
    y = w_in - e + 1;
  }
  y = std::min(y, cap);
  return code < 0 ? -y : y;
}

int conv_width(const ConvGeom& g) {
  int w = 1;
  const uint64_t neurons = (uint64_t)g.Ho() * g.Wo() * g.Co;
  for (uint64_t q = 0; q < neurons; ++q) {
    const int co = (int)(q % g.Co);
    const int ow = (int)((q / g.Co) % g.Wo());
    const int oh = (int)(q / ((uint64_t)g.Co * g.Wo()));
    std::vector<int> leaves;
    for (int kh = 0; kh < g.K; ++kh)
      for (int kw = 0; kw < g.K; ++kw) {
        const int ih = oh * g.stride - g.pad + kh, iw = ow * g.stride - g.pad + kw;
        if (ih < 0 || ih >= g.H || iw < 0 || iw >= g.W) continue;
        for (int ci = 0; ci < g.C; ++ci)
          for_each_code(g.wq, g.wm, (((size_t)co * g.K + kh) * g.K + kw) * g.C + ci,
                        [&](int8_t code) {
                          int lw = leaf_width(g.w_in, g.in_signed != 0, code, g.cap);
                          if (lw) leaves.push_back(lw);
                        });
      }
    w = std::max(w, neuron_width(leaves, g.cap, g.relu != 0));
  }
  return w;
}

int fc_width(const FcGeom& g) {
  int w = 1;
  for (int m = 0; m < g.M; ++m) {
    std::vector<int> leaves;
    for (int k = 0; k < g.K; ++k)
      for_each_code(g.wq, g.wm, (size_t)m * g.K + k, [&](int8_t code) {
        int lw = leaf_width(g.w_in, g.in_signed != 0, code, g.cap);
        if (lw) leaves.push_back(lw);
      });
    w = std::max(w, neuron_width(leaves, g.cap, g.relu != 0));
  }
  return w;
}

she_status check_codes(const int8_t* wq, const int16_t* wm, size_t n) {
  if (wm) {
    for (size_t i = 0; i < n; ++i)
      if (wm[i] < -255 || wm[i] > 255)
        return she::fail(SHE_ERR_ARG, "TCN multiplier %d out of [-255, 255]", wm[i]);
    return SHE_OK;
  }
  for (size_t i = 0; i < n; ++i)
    if (wq[i] < -8 || wq[i] > 8) return she::fail(SHE_ERR_ARG, "weight code %d out of [-8, 8]", wq[i]);
  return SHE_OK;
}

she_status conv_common(const ConvGeom& g, int* w_out, int rank, int world, Executor* ex,
                       she_circuit_stats* st) {
  if ((!g.wq && !g.wm) || !w_out) return she::fail(SHE_ERR_ARG, "NULL argument");
  if (g.H <= 0 || g.W <= 0 || g.C <= 0 || g.Co <= 0 || g.K <= 0 || g.stride <= 0 || g.pad < 0 ||
      g.w_in <= 0 || g.w_in > 32 || g.cap < 2 || g.cap > 32 || g.Ho() <= 0 || g.Wo() <= 0)
    return she::fail(SHE_ERR_SHAPE, "bad conv shape");
  she_status s = check_codes(g.wq, g.wm, (size_t)g.Co * g.K * g.K * g.C);
  if (s != SHE_OK) return s;
  const int w = conv_width(g);
  if (!ex) {
    *w_out = w;
    return SHE_OK;
  }
  if (*w_out < w) return she::fail(SHE_ERR_SHAPE, "output word capacity %d < width %d", *w_out, w);
  *w_out = w;
  const uint64_t neurons = (uint64_t)g.Ho() * g.Wo() * g.Co;
  return run_layer(neurons, w, g.relu == 0, rank, world,
                   [&](Circuit& c, InputMap& im, uint64_t q) { return conv_neuron(g, c, im, q); },
                   *ex, st);
}

she_status fc_common(const FcGeom& g, int* w_out, int rank, int world, Executor* ex,
                     she_circuit_stats* st) {
  if ((!g.wq && !g.wm) || !w_out) return she::fail(SHE_ERR_ARG, "NULL argument");
  if (g.K <= 0 || g.M <= 0 || g.w_in <= 0 || g.w_in > 32 || g.cap < 2 || g.cap > 32)
    return she::fail(SHE_ERR_SHAPE, "bad fc shape");
  she_status s = check_codes(g.wq, g.wm, (size_t)g.M * g.K);
  if (s != SHE_OK) return s;
  const int w = fc_width(g);
  if (!ex) {
    *w_out = w;
    return SHE_OK;
  }
  if (*w_out < w) return she::fail(SHE_ERR_SHAPE, "output word capacity %d < width %d", *w_out, w);
  *w_out = w;
  return run_layer((uint64_t)g.M, w, g.relu == 0, rank, world,
                   [&](Circuit& c, InputMap& im, uint64_t m) { return fc_neuron(g, c, im, m); },
                   *ex, st);
}

she_status relu_common(size_t words, int width, int rank, int world, Executor& ex,
                       she_circuit_stats* st) {
  if (width < 2) return she::fail(SHE_ERR_SHAPE, "ReLU needs width >= 2");
  return run_layer(words, width - 1, false, rank, world,
                   [&](Circuit& c, InputMap& im, uint64_t q) {
                     Word v(width);
                     for (int b = 0; b < width; ++b) v[b] = im((uint32_t)(q * width + b));
                     return relu(c, v);
                   },
                   ex, st);
}

// Batch normalisation lowered to a power-of-two scale and a constant
// (SURVEY.md §8(f) NEXT-3; the B layers of PAPER.md T3, :202-203):
//   y = wrap_cap(sign * scale(x, s) + bias),  scale(x, s) = x 2^s (s >= 0) or
//   floor(x / 2^-s) (s < 0)
// The scale is rewiring, the sign NOT flags plus a carry-in, the bias an adder
// against constant bits (constant folding leaves ~2 gates per bit).
struct BnGeom {
  size_t words;
  int C, w_in, in_signed, cap, relu;
  const int8_t* shift;   // [C], in [-8, 8]
  const uint8_t* neg;    // [C], 0 / 1 (may be NULL: all positive)
  const int32_t* bias;   // [C]
};

int bits_signed(int64_t v) {  // two's-complement width of a constant
  int w = 1;
  while (w < 40 && (v < -(int64_t(1) << (w - 1)) || v >= (int64_t(1) << (w - 1)))) ++w;
  return w;
}

int bn_scaled_width(const BnGeom& g, int ch) {
  const int s = g.shift[ch];
  const int base = g.in_signed ? g.w_in : g.w_in + 1;  // with the (constant-0) sign bit
  return std::max(1, base + s);
}

int bn_width(const BnGeom& g, int ch) {
  const int w = std::max(bn_scaled_width(g, ch), bits_signed(g.bias[ch])) + 1;
  const int y = std::min(w, g.cap);
  return g.relu ? std::max(1, y - 1) : y;
}

Word bn_word(const BnGeom& g, Circuit& c, const Word& x, int ch) {
  const int s = g.shift[ch];
  Word v = x;  // LSB first
  if (!g.in_signed) v.push_back(F);
  if (s > 0) v.insert(v.begin(), (size_t)s, F);
  if (s < 0) {
    const size_t drop = (size_t)(-s);
    if (drop >= v.size()) v = Word{v.back()};
    else v.erase(v.begin(), v.begin() + (long)drop);
  }
  if ((int)v.size() > g.cap) v.resize(g.cap);
  const bool ng = g.neg && g.neg[ch];
  const int width = std::min(std::max((int)v.size(), bits_signed(g.bias[ch])) + 1, g.cap);
  Word k(width);
  for (int i = 0; i < width; ++i) k[i] = ((int64_t)g.bias[ch] >> std::min(i, 39)) & 1 ? T : F;
  Word y = c.add(ng ? c.neg_bits(v) : v, k, ng ? T : F, width);  // -v = !v + 1
  return g.relu ? relu(c, y.size() > 1 ? y : Word{y[0], y[0]}) : y;
}

she_status bn_common(const BnGeom& g, int* w_out, int rank, int world, Executor* ex,
                     she_circuit_stats* st) {
  if (!g.shift || !g.bias || !w_out) return she::fail(SHE_ERR_ARG, "NULL argument");
  if (g.C <= 0 || g.w_in <= 0 || g.w_in > 32 || g.cap < 2 || g.cap > 32 || g.words % g.C)
    return she::fail(SHE_ERR_SHAPE, "bad batch-norm shape");
  int w = 1;
  for (int ch = 0; ch < g.C; ++ch) {
    if (g.shift[ch] < -8 || g.shift[ch] > 8)
      return she::fail(SHE_ERR_ARG, "BN shift %d out of [-8, 8]", g.shift[ch]);
    if (g.bias[ch] < -(1 << 20) || g.bias[ch] > (1 << 20))
      return she::fail(SHE_ERR_ARG, "BN bias %d out of [-2^20, 2^20]", g.bias[ch]);
    w = std::max(w, bn_width(g, ch));
  }
  if (!ex) {
    *w_out = w;
    return SHE_OK;
  }
  if (*w_out < w) return she::fail(SHE_ERR_SHAPE, "output word capacity %d < width %d", *w_out, w);
  *w_out = w;
  return run_layer(g.words, w, g.relu == 0, rank, world,
                   [&](Circuit& c, InputMap& im, uint64_t q) {
                     Word x(g.w_in);
                     for (int b = 0; b < g.w_in; ++b) x[b] = im((uint32_t)(q * g.w_in + b));
                     return bn_word(g, c, x, (int)(q % g.C));
                   },
                   *ex, st);
}

she_status maxpool_common(int H, int W, int C, int w, int in_signed, int rank, int world,
                          Executor& ex, she_circuit_stats* st) {
  if (H < 2 || W < 2 || C <= 0 || w <= 0) return she::fail(SHE_ERR_SHAPE, "bad maxpool shape");
  const int Ho = H / 2, Wo = W / 2;
  return run_layer((uint64_t)Ho * Wo * C, w, in_signed != 0, rank, world,
                   [&](Circuit& c, InputMap& im, uint64_t q) {
                     const int ch = (int)(q % C);
                     const int ow = (int)((q / C) % Wo);
                     const int oh = (int)(q / ((uint64_t)C * Wo));
                     Word v[4];
                     for (int d = 0; d < 4; ++d) {
                       const int ih = 2 * oh + d / 2, iw = 2 * ow + d % 2;
                       const uint32_t base = (uint32_t)((((size_t)ih * W + iw) * C + ch) * w);
                       for (int b = 0; b < w; ++b) v[d].push_back(im(base + b));
                       if (!in_signed) v[d].push_back(F);  // unsigned: constant-0 sign
                     }
                     Word m = c.max(c.max(v[0], v[1]), c.max(v[2], v[3]));
                     m.resize(w);  // drop the constant sign bit again for unsigned words
                     return m;
                   },
                   ex, st);
}

}  // namespace

// ---------------------------------------------------------------------------
// C-ABI
// ---------------------------------------------------------------------------
extern "C" {

she_status she_conv_shift_acc(she_ctx* ctx, const uint32_t* in, int H, int W, int C, int w_in,
                              int in_signed, const int8_t* wq, int Co, int K, int stride, int pad,
                              int acc_cap, int relu_, uint32_t* out, int* w_out, void* stream) {
  ConvGeom g{H, W, C, w_in, in_signed, Co, K, stride, pad, acc_cap, relu_, wq};
  if (!out) return conv_common(g, w_out, 0, 1, nullptr, nullptr);
  if (!ctx || !in) return she::fail(SHE_ERR_ARG, "NULL argument");
  GpuExec ex;
  ex.ctx = ctx;
  ex.in = in;
  ex.out = out;
  ex.stream = stream;
  she_circuit_stats* st = she::engine_stats(ctx, true);
  return conv_common(g, w_out, she::engine_rank(ctx), she::engine_world(ctx), &ex, st);
}

she_status she_fc_shift_acc(she_ctx* ctx, const uint32_t* in, int K, int w_in, int in_signed,
                            const int8_t* wq, int M, int acc_cap, int relu_, uint32_t* out,
                            int* w_out, void* stream) {
  FcGeom g{K, w_in, in_signed, M, acc_cap, relu_, wq};
  if (!out) return fc_common(g, w_out, 0, 1, nullptr, nullptr);
  if (!ctx || !in) return she::fail(SHE_ERR_ARG, "NULL argument");
  GpuExec ex;
  ex.ctx = ctx;
  ex.in = in;
  ex.out = out;
  ex.stream = stream;
  she_circuit_stats* st = she::engine_stats(ctx, true);
  return fc_common(g, w_out, she::engine_rank(ctx), she::engine_world(ctx), &ex, st);
}

she_status she_conv_mul_acc(she_ctx* ctx, const uint32_t* in, int H, int W, int C, int w_in,
                            int in_signed, const int16_t* wm, int Co, int K, int stride, int pad,
                            int acc_cap, int relu_, uint32_t* out, int* w_out, void* stream) {
  ConvGeom g{H, W, C, w_in, in_signed, Co, K, stride, pad, acc_cap, relu_, nullptr, wm};
  if (!out) return conv_common(g, w_out, 0, 1, nullptr, nullptr);
  if (!ctx || !in) return she::fail(SHE_ERR_ARG, "NULL argument");
  GpuExec ex;
  ex.ctx = ctx;
  ex.in = in;
  ex.out = out;
  ex.stream = stream;
  she_circuit_stats* st = she::engine_stats(ctx, true);
  return conv_common(g, w_out, she::engine_rank(ctx), she::engine_world(ctx), &ex, st);
}

she_status she_fc_mul_acc(she_ctx* ctx, const uint32_t* in, int K, int w_in, int in_signed,
                          const int16_t* wm, int M, int acc_cap, int relu_, uint32_t* out,
                          int* w_out, void* stream) {
  FcGeom g{K, w_in, in_signed, M, acc_cap, relu_, nullptr, wm};
  if (!out) return fc_common(g, w_out, 0, 1, nullptr, nullptr);
  if (!ctx || !in) return she::fail(SHE_ERR_ARG, "NULL argument");
  GpuExec ex;
  ex.ctx = ctx;
  ex.in = in;
  ex.out = out;
  ex.stream = stream;
  she_circuit_stats* st = she::engine_stats(ctx, true);
  return fc_common(g, w_out, she::engine_rank(ctx), she::engine_world(ctx), &ex, st);
}

she_status she_relu(she_ctx* ctx, const uint32_t* in, size_t words, int width, uint32_t* out,
                    void* stream) {
  if (words == 0) return SHE_OK;
  if (!ctx || !in || !out) return she::fail(SHE_ERR_ARG, "NULL argument");
  GpuExec ex;
  ex.ctx = ctx;
  ex.in = in;
  ex.out = out;
  ex.stream = stream;
  return relu_common(words, width, she::engine_rank(ctx), she::engine_world(ctx), ex,
                     she::engine_stats(ctx, true));
}

she_status she_bn_shift_add(she_ctx* ctx, const uint32_t* in, size_t words, int C, int w_in,
                            int in_signed, const int8_t* shift, const uint8_t* neg,
                            const int32_t* bias, int acc_cap, int relu_, uint32_t* out,
                            int* w_out, void* stream) {
  BnGeom g{words, C, w_in, in_signed, acc_cap, relu_, shift, neg, bias};
  if (!out) return bn_common(g, w_out, 0, 1, nullptr, nullptr);
  if (words == 0) return SHE_OK;
  if (!ctx || !in) return she::fail(SHE_ERR_ARG, "NULL argument");
  GpuExec ex;
  ex.ctx = ctx;
  ex.in = in;
  ex.out = out;
  ex.stream = stream;
  she_circuit_stats* st = she::engine_stats(ctx, true);
  return bn_common(g, w_out, she::engine_rank(ctx), she::engine_world(ctx), &ex, st);
}

she_status she_maxpool2x2(she_ctx* ctx, const uint32_t* in, int H, int W, int C, int w,
                          int in_signed, uint32_t* out, void* stream) {
  if (!ctx || !in || !out) return she::fail(SHE_ERR_ARG, "NULL argument");
  GpuExec ex;
  ex.ctx = ctx;
  ex.in = in;
  ex.out = out;
  ex.stream = stream;
  return maxpool_common(H, W, C, w, in_signed, she::engine_rank(ctx), she::engine_world(ctx), ex,
                        she::engine_stats(ctx, true));
}

she_status she_ctx_layer_stats(she_ctx* ctx, she_circuit_stats* st) {
  if (!ctx || !st) return she::fail(SHE_ERR_ARG, "NULL argument");
  *st = *she::engine_stats(ctx, false);
  return SHE_OK;
}

// ---- clear-bit backend (SPEC.md:88-143 idea): the same circuits on plaintext
// bits, host only; used to test the scheduler and to count gates/levels.
she_status she_clear_conv_shift_acc(const uint8_t* in, int H, int W, int C, int w_in,
                                    int in_signed, const int8_t* wq, int Co, int K, int stride,
                                    int pad, int acc_cap, int relu_, uint8_t* out, int* w_out,
                                    int rank, int world, she_circuit_stats* st) {
  ConvGeom g{H, W, C, w_in, in_signed, Co, K, stride, pad, acc_cap, relu_, wq};
  if (st) *st = she_circuit_stats{};
  if (!out) return conv_common(g, w_out, 0, 1, nullptr, nullptr);
  if (!in) return she::fail(SHE_ERR_ARG, "NULL argument");
  if (world < 1 || rank < 0 || rank >= world) return she::fail(SHE_ERR_ARG, "bad rank/world");
  ClearExec ex;
  ex.in = in;
  ex.out = out;
  return conv_common(g, w_out, rank, world, &ex, st);
}

she_status she_clear_fc_shift_acc(const uint8_t* in, int K, int w_in, int in_signed,
                                  const int8_t* wq, int M, int acc_cap, int relu_, uint8_t* out,
                                  int* w_out, int rank, int world, she_circuit_stats* st) {
  FcGeom g{K, w_in, in_signed, M, acc_cap, relu_, wq};
  if (st) *st = she_circuit_stats{};
  if (!out) return fc_common(g, w_out, 0, 1, nullptr, nullptr);
  if (!in) return she::fail(SHE_ERR_ARG, "NULL argument");
  if (world < 1 || rank < 0 || rank >= world) return she::fail(SHE_ERR_ARG, "bad rank/world");
  ClearExec ex;
  ex.in = in;
  ex.out = out;
  return fc_common(g, w_out, rank, world, &ex, st);
}

she_status she_clear_conv_mul_acc(const uint8_t* in, int H, int W, int C, int w_in,
                                  int in_signed, const int16_t* wm, int Co, int K, int stride,
                                  int pad, int acc_cap, int relu_, uint8_t* out, int* w_out,
                                  int rank, int world, she_circuit_stats* st) {
  ConvGeom g{H, W, C, w_in, in_signed, Co, K, stride, pad, acc_cap, relu_, nullptr, wm};
  if (st) *st = she_circuit_stats{};
  if (!out) return conv_common(g, w_out, 0, 1, nullptr, nullptr);
  if (!in) return she::fail(SHE_ERR_ARG, "NULL argument");
  if (world < 1 || rank < 0 || rank >= world) return she::fail(SHE_ERR_ARG, "bad rank/world");
  ClearExec ex;
  ex.in = in;
  ex.out = out;
  return conv_common(g, w_out, rank, world, &ex, st);
}

she_status she_clear_fc_mul_acc(const uint8_t* in, int K, int w_in, int in_signed,
                                const int16_t* wm, int M, int acc_cap, int relu_, uint8_t* out,
                                int* w_out, int rank, int world, she_circuit_stats* st) {
  FcGeom g{K, w_in, in_signed, M, acc_cap, relu_, nullptr, wm};
  if (st) *st = she_circuit_stats{};
  if (!out) return fc_common(g, w_out, 0, 1, nullptr, nullptr);
  if (!in) return she::fail(SHE_ERR_ARG, "NULL argument");
  if (world < 1 || rank < 0 || rank >= world) return she::fail(SHE_ERR_ARG, "bad rank/world");
  ClearExec ex;
  ex.in = in;
  ex.out = out;
  return fc_common(g, w_out, rank, world, &ex, st);
}

she_status she_clear_relu(const uint8_t* in, size_t words, int width, uint8_t* out, int rank,
                          int world, she_circuit_stats* st) {
  if (st) *st = she_circuit_stats{};
  if (words == 0) return SHE_OK;
  if (!in || !out) return she::fail(SHE_ERR_ARG, "NULL argument");
  if (world < 1 || rank < 0 || rank >= world) return she::fail(SHE_ERR_ARG, "bad rank/world");
  ClearExec ex;
  ex.in = in;
  ex.out = out;
  return relu_common(words, width, rank, world, ex, st);
}

she_status she_clear_bn_shift_add(const uint8_t* in, size_t words, int C, int w_in,
                                  int in_signed, const int8_t* shift, const uint8_t* neg,
                                  const int32_t* bias, int acc_cap, int relu_, uint8_t* out,
                                  int* w_out, int rank, int world, she_circuit_stats* st) {
  BnGeom g{words, C, w_in, in_signed, acc_cap, relu_, shift, neg, bias};
  if (st) *st = she_circuit_stats{};
  if (!out) return bn_common(g, w_out, 0, 1, nullptr, nullptr);
  if (words == 0) return SHE_OK;
  if (!in) return she::fail(SHE_ERR_ARG, "NULL argument");
  if (world < 1 || rank < 0 || rank >= world) return she::fail(SHE_ERR_ARG, "bad rank/world");
  ClearExec ex;
  ex.in = in;
  ex.out = out;
  return bn_common(g, w_out, rank, world, &ex, st);
}

she_status she_clear_maxpool2x2(const uint8_t* in, int H, int W, int C, int w, int in_signed,
                                uint8_t* out, int rank, int world, she_circuit_stats* st) {
  if (st) *st = she_circuit_stats{};
  if (!in || !out) return she::fail(SHE_ERR_ARG, "NULL argument");
  if (world < 1 || rank < 0 || rank >= world) return she::fail(SHE_ERR_ARG, "bad rank/world");
  ClearExec ex;
  ex.in = in;
  ex.out = out;
  return maxpool_common(H, W, C, w, in_signed, rank, world, ex, st);
}

}  // extern "C"
