// Host-side lowering of an instrumented program to the device program and the
// HBM tile-pass plan (see devprog.hpp).
#include "devprog.hpp"

#include <algorithm>
#include <bit>
#include <cstdio>
#include <stdexcept>
#include <string>

#include "exact.cuh"

namespace ssb {

uint64_t classify_matrix(const double* m, unsigned k, bool scaled) {
  const unsigned entries = 1u << (2 * k);
  uint64_t cls = 0;
  for (unsigned i = 0; i < entries; ++i) {
    const double re = m[2 * i], im = m[2 * i + 1];
    uint64_t c;
    if (re == 0.0 && im == 0.0) c = E_ZERO;
    else if (im == 0.0) c = (!scaled && re == 1.0) ? E_ONE : (!scaled && re == -1.0) ? E_NEG_ONE : E_REAL;
    else if (re == 0.0) c = E_IMAG;
    else c = E_GEN;
    cls |= c << (3 * i);
  }
  return cls;
}

namespace {

bool is_identity_cls(uint64_t cls, unsigned k) {
  const unsigned d = 1u << k;
  for (unsigned r = 0; r < d; ++r)
    for (unsigned c = 0; c < d; ++c)
      if (entry_class(cls, r * d + c) != (r == c ? E_ONE : E_ZERO)) return false;
  return true;
}

// Picks the arithmetic template for a gate matrix (see MicroKind). Every
// template performs exactly the reference's nonzero-term products and sums.
uint8_t micro_kind(uint64_t cls, unsigned k, uint8_t* src) {
  *src = 0;
  if (k == 1) {
    const uint32_t c0 = entry_class(cls, 0), c1 = entry_class(cls, 1), c2 = entry_class(cls, 2),
                   c3 = entry_class(cls, 3);
    if (c0 == E_REAL && c1 == E_GEN && c2 == E_GEN && c3 == E_GEN) return MK_1Q_U;
    if (c0 == E_REAL && c1 == E_REAL && c2 == E_REAL && c3 == E_REAL) return MK_1Q_REAL;
    return MK_1Q_GEN;
  }
  uint8_t s = 0;
  for (unsigned r = 0; r < 4; ++r) {
    int col = -1, nz = 0;
    for (unsigned c = 0; c < 4; ++c)
      if (entry_class(cls, r * 4 + c) != E_ZERO) {
        ++nz;
        col = static_cast<int>(c);
      }
    if (nz != 1) return MK_2Q_GEN;
    s |= static_cast<uint8_t>(col << (2 * r));
  }
  *src = s;
  return MK_2Q_MONO;
}

}  // namespace

HostDevProgram build_device_program(const shotsim::NoisyCircuit& p) {
  using shotsim::ProgramOp;
  if (p.num_qubits < 1 || p.num_qubits > 30) throw std::invalid_argument("qubit count must be in [1, 30]");
  HostDevProgram d;
  d.n = p.num_qubits;
  d.num_clbits = p.num_clbits;
  d.num_events = p.num_events;
  d.eligible = p.sampling_eligible;
  d.has_measure = p.has_measure;
  d.end = static_cast<uint32_t>(p.sampling_eligible ? p.terminal_measure_begin : p.ops.size());

  auto push_matrix = [&d](const shotsim::GateMatrix& m) {
    const uint32_t slot = static_cast<uint32_t>(d.mats.size() / 32);
    d.mats.resize(d.mats.size() + 32, 0.0);
    for (size_t i = 0; i < m.entries.size(); ++i) {
      d.mats[slot * 32 + 2 * i] = m.entries[i].real();
      d.mats[slot * 32 + 2 * i + 1] = m.entries[i].imag();
    }
    d.scaled_cls.push_back(classify_matrix(&d.mats[slot * 32], m.num_qubits, true));
    return slot;
  };

  for (const shotsim::KrausError& k : p.kraus_channels) {
    if (k.arity < 1 || k.arity > 2) throw std::invalid_argument("kraus arity must be 1 or 2");
    DevChannel ch{k.arity, static_cast<uint32_t>(k.matrices.size()), 0, 0};
    for (size_t i = 0; i < k.matrices.size(); ++i) {
      const uint32_t s = push_matrix(k.matrices[i]);
      if (i == 0) ch.mat_begin = s;
    }
    if (ch.nmat == 0) throw std::invalid_argument("kraus channel without matrices");
    d.channels.push_back(ch);
    d.max_kraus = std::max(d.max_kraus, ch.nmat);
  }

  for (const ProgramOp& op : p.ops) {
    DevOp o{};
    o.kind = static_cast<uint8_t>(op.kind);
    if (op.qubits.size() > 4) throw std::invalid_argument("op has more than 4 qubits");
    o.nq = static_cast<uint8_t>(op.qubits.size());
    for (size_t i = 0; i < op.qubits.size(); ++i) {
      if (op.qubits[i] >= p.num_qubits) throw std::invalid_argument("target qubit out of range");
      o.q[i] = static_cast<uint8_t>(op.qubits[i]);
    }
    for (size_t i = 0; i < op.clbits.size() && i < 4; ++i) {
      if (op.clbits[i] >= 64) throw std::invalid_argument("clbit out of range");
      o.c[i] = static_cast<uint8_t>(op.clbits[i]);
    }
    o.has_cond = op.condition.has_value();
    if (op.condition) {
      o.cond_mask = op.condition->clbit_mask;
      o.cond_value = op.condition->value;
    }
    o.event = op.event;
    switch (op.kind) {
      case ProgramOp::Kind::Gate: {
        if (op.matrix.num_qubits != op.qubits.size() || op.qubits.size() < 1 || op.qubits.size() > 2)
          throw std::invalid_argument("matrix dimension does not match target count");
        if (op.qubits.size() == 2 && op.qubits[0] == op.qubits[1])
          throw std::invalid_argument("duplicate target qubit");
        o.aux = push_matrix(op.matrix);
        o.cls = classify_matrix(&d.mats[o.aux * 32], op.matrix.num_qubits, false);
        o.skip = is_identity_cls(o.cls, op.matrix.num_qubits);
        o.mk = micro_kind(o.cls, op.matrix.num_qubits, &o.src);
        break;
      }
      case ProgramOp::Kind::PauliSite: {
        o.aux = static_cast<uint32_t>(d.terms.size());
        o.count = static_cast<uint32_t>(op.term_cum.size());
        o.site = d.num_pauli_sites++;
        if (o.count == 0 || o.count > 255) throw std::invalid_argument("pauli site term count");
        for (size_t t = 0; t < op.term_cum.size(); ++t) {
          const shotsim::PauliMasks& m = op.term_masks[t];
          if ((m.x_mask >> p.num_qubits) || (m.z_mask >> p.num_qubits))
            throw std::invalid_argument("pauli mask out of range for state");
          d.terms.push_back({op.term_cum[t], static_cast<uint32_t>(m.x_mask), static_cast<uint32_t>(m.z_mask),
                             m.num_y, op.term_identity[t]});
        }
        break;
      }
      case ProgramOp::Kind::KrausSite: {
        if (op.channel >= d.channels.size()) throw std::invalid_argument("kraus channel out of range");
        o.aux = op.channel;
        o.count = d.channels[op.channel].nmat;
        if (d.channels[op.channel].arity != op.qubits.size())
          throw std::invalid_argument("matrix dimension does not match target count");
        d.has_kraus = true;
        break;
      }
      case ProgramOp::Kind::Measure:
      case ProgramOp::Kind::Reset:
        if (op.qubits.empty()) throw std::invalid_argument("measure/reset needs qubits");
        if (op.kind == ProgramOp::Kind::Measure && op.clbits.size() != op.qubits.size())
          throw std::invalid_argument("measure needs one clbit per qubit");
        d.has_measure_ops = true;
        break;
      case ProgramOp::Kind::Barrier: break;
    }
    d.ops.push_back(o);
  }
  for (unsigned q : p.sample_qubits) d.sample_qubits.push_back(static_cast<uint8_t>(q));
  for (const auto& [c, b] : p.sample_writes) {
    d.write_clbit.push_back(static_cast<uint8_t>(c));
    d.write_pos.push_back(static_cast<uint8_t>(b));
  }
  d.sample_identity = d.sample_qubits.size() == d.n;
  for (size_t i = 0; i < d.sample_qubits.size() && d.sample_identity; ++i)
    d.sample_identity = d.sample_qubits[i] == i;
  return d;
}

namespace {

// Shared-memory budget of one pass's staged micro-op stream: 2 x 16 B per op
// (uop + compacted copy) + its matrix entries (2q dense: 16 x 16 B, else 4).
constexpr size_t kMaxPassStageBytes = 28 * 1024;
size_t stage_bytes(const DevOp& o) {
  if (o.kind == K_PAULI) return 32;
  if (o.kind == K_KRAUS) return 32 + 16 * 16;
  return 32 + 16 * ((o.nq == 2 && o.mk != MK_2Q_MONO) ? 16 : 4);
}

// Splits pass ops [first, ops.size()) into register segments: maximal runs of
// consecutive ops whose qubits stay inside one 2-qubit set. pos: qubit ->
// local position. A single-qubit segment is paired with another local qubit.
void segment_ops(HostDevProgram& d, const std::vector<uint32_t>& ops, const uint8_t* pos, unsigned k) {
  size_t i = 0;
  while (i < ops.size()) {
    uint32_t set = 0;  // local positions
    size_t j = i;
    for (; j < ops.size(); ++j) {
      uint32_t m = 0;
      for (unsigned b = 0; b < d.ops[ops[j]].nq; ++b) m |= 1u << pos[d.ops[ops[j]].q[b]];
      if (std::popcount(set | m) > 2) break;
      set |= m;
    }
    Item it{};
    it.kind = IT_SEGMENT;
    it.shape = kNoShape;
    unsigned la = static_cast<unsigned>(std::countr_zero(set));
    unsigned lb = std::popcount(set) == 2 ? 31u - static_cast<unsigned>(std::countl_zero(set)) : (la == 0 ? 1u : 0u);
    if (k < 2) lb = la;  // degenerate 1-qubit state: per-op fallback in the kernel
    if (la > lb) std::swap(la, lb);
    it.la = static_cast<uint8_t>(la);
    it.lb = static_cast<uint8_t>(lb);
    it.begin = static_cast<uint32_t>(d.pass_ops.size());
    for (size_t t = i; t < j; ++t) {
      PassOp po{ops[t], {}};
      for (unsigned b = 0; b < d.ops[ops[t]].nq; ++b) po.qb[b] = pos[d.ops[ops[t]].q[b]] == la ? 0 : 1;
      if (k < 2)
        for (unsigned b = 0; b < d.ops[ops[t]].nq; ++b) po.qb[b] = pos[d.ops[ops[t]].q[b]];
      d.pass_ops.push_back(po);
    }
    it.end = static_cast<uint32_t>(d.pass_ops.size());
    d.items.push_back(it);
    i = j;
  }
}

bool fused_kind(const DevOp& o) { return o.kind == K_GATE || o.kind == K_PAULI; }

// Shape key of a lowered segment: every field of its non-Pauli micro-ops that
// the straight-line executor bakes in (code, register operands, classes,
// matrix offsets relative to the segment's first matrix), plus the final
// register map. Items with equal keys share one generated executor.
void assign_shape(HostDevProgram& d, Item& it, uint32_t uop_base) {
  std::string key;
  uint32_t nfast = 0, mat0 = it.end > it.begin ? d.uops[uop_base + it.begin].mat : 0;
  char buf[96];
  for (uint32_t i = it.begin; i < it.end; ++i) {
    const Uop& u = d.uops[uop_base + i];
    if (u.code == UC_PAULI) {
      // Position and register map only: the draw is per shot (noisy variant).
      std::snprintf(buf, sizeof buf, "P.%u.%u;", u.sigma, i - it.begin);
      key += buf;
      continue;
    }
    const uint64_t cls = (u.code == UC_GEN1 || u.code == UC_GEN2) ? d.ops[u.ref].cls : 0;
    std::snprintf(buf, sizeof buf, "%u.%u.%u.%u.%u.%llx.%u;", u.code, u.qb, u.src, u.mcls, u.sigma,
                  static_cast<unsigned long long>(cls), static_cast<unsigned>(u.mat - mat0));
    key += buf;
    ++nfast;
  }
  std::snprintf(buf, sizeof buf, "|%u", it.sigma);
  key += buf;
  if (nfast > 0xFFFF) throw std::length_error("segment too long");
  it.nfast = static_cast<uint16_t>(nfast);
  auto pos = std::find(d.shapes.begin(), d.shapes.end(), key);
  if (pos == d.shapes.end()) {
    if (d.shapes.size() >= kNoShape) {
      it.shape = kNoShape;
      return;
    }
    d.shapes.push_back(key);
    pos = d.shapes.end() - 1;
  }
  it.shape = static_cast<uint16_t>(pos - d.shapes.begin());
}

// Lowers the pass ops [po_begin, ...) of pass `pd` to micro-ops + a compact
// matrix table, segment by segment, folding unconditional 2q permutations
// into the register relabeling sigma; items are re-based to uop indices
// relative to the pass.
void build_uops(HostDevProgram& d, PassDesc& pd, uint32_t po_begin) {
  pd.uop_begin = static_cast<uint32_t>(d.uops.size());
  pd.po_begin = po_begin;
  pd.mat_begin = static_cast<uint32_t>(d.uop_mats.size() / 2);
  uint32_t mat = 0;
  auto push = [&](const double* e) {
    d.uop_mats.push_back(e[0]);
    d.uop_mats.push_back(e[1]);
    ++mat;
  };
  auto pack = [](const int* sg) {
    return static_cast<uint8_t>(sg[0] | (sg[1] << 2) | (sg[2] << 4) | (sg[3] << 6));
  };
  for (uint32_t it_i = pd.item_begin; it_i < pd.item_end; ++it_i) {
    Item& it = d.items[it_i];
    if (it.kind != IT_SEGMENT) continue;  // resident plans interleave special ops
    int sg[4] = {0, 1, 2, 3};  // logical element -> register
    const uint32_t ubegin = static_cast<uint32_t>(d.uops.size()) - pd.uop_begin;
    for (uint32_t i = it.begin; i < it.end; ++i) {
      const PassOp& po = d.pass_ops[i];
      const DevOp& o = d.ops[po.op];
      Uop u{};
      u.ref = po.op;
      u.flags = o.has_cond ? 1 : 0;
      u.mat = static_cast<uint16_t>(mat);
      u.sigma = pack(sg);
      const double* m = &d.mats[static_cast<size_t>(o.aux) * 32];
      if (o.kind == K_PAULI) {
        u.code = UC_PAULI;
        u.qb = static_cast<uint8_t>((po.qb[0] & 1) | (o.nq > 1 ? (po.qb[1] & 1) << 1 : 0));
      } else if (o.kind == K_KRAUS) {
        // Per-shot matrix: staged by the tile kernel into the pass's Kraus slot.
        u.code = o.nq == 1 ? UC_KRAUS1 : UC_KRAUS2;
        u.src = po.qb[0];
        if (o.nq == 1) {  // physical register pairs, as for 1q gates
          const int bit = 1 << po.qb[0];
          const int l0 = 0, l1 = bit, l2 = bit == 1 ? 2 : 1, l3 = l2 | bit;
          u.qb = static_cast<uint8_t>(sg[l0] | (sg[l1] << 2) | (sg[l2] << 4) | (sg[l3] << 6));
        } else {
          u.qb = po.qb[0];
        }
        u.mat = static_cast<uint16_t>(0xFFFF);  // patched to pd.kraus_mat below
      } else if (o.nq == 1) {
        u.code = o.mk == MK_1Q_U ? UC_U : o.mk == MK_1Q_REAL ? UC_REAL : UC_GEN1;
        const int bit = 1 << po.qb[0];
        const int l0 = 0, l1 = bit, l2 = bit == 1 ? 2 : 1, l3 = l2 | bit;  // logical pairs (l0,l1), (l2,l3)
        u.qb = static_cast<uint8_t>(sg[l0] | (sg[l1] << 2) | (sg[l2] << 4) | (sg[l3] << 6));
        u.src = po.qb[0];  // logical quad bit (generic path)
        for (int e = 0; e < 4; ++e) push(m + 2 * e);
      } else {
        // Quad element of matrix index r (index bits: q0, q1).
        auto el = [swapped = po.qb[0] != 0](int r) { return swapped ? ((r & 1) << 1) | (r >> 1) : r; };
        int perm[4] = {0, 1, 2, 3}, cls_r[4] = {0, 0, 0, 0}, n_nonone = 0, moved = 0;
        if (o.mk == MK_2Q_MONO) {
          for (int r = 0; r < 4; ++r) {
            const int c = (o.src >> (2 * r)) & 3;
            perm[el(r)] = el(c);  // new logical element el(r) takes old element el(c)
            cls_r[r] = static_cast<int>(entry_class(o.cls, r * 4 + c));
            n_nonone += cls_r[r] != E_ONE;
            moved += el(c) != el(r);
          }
        }
        if (o.mk == MK_2Q_MONO && n_nonone == 0 && !o.has_cond) {
          // Exact pure permutation (every moved entry is 1): relabel registers.
          int ns[4];
          for (int e = 0; e < 4; ++e) ns[e] = sg[perm[e]];
          for (int e = 0; e < 4; ++e) sg[e] = ns[e];
          continue;  // no micro-op
        }
        if (o.mk == MK_2Q_MONO && n_nonone == 0 && moved == 2) {
          u.code = UC_SWAP;  // conditional transposition: physical registers
          int a = -1, b = -1;
          for (int e = 0; e < 4; ++e)
            if (perm[e] != e) (a < 0 ? a : b) = e;
          u.qb = static_cast<uint8_t>(std::min(sg[a], sg[b]) | (std::max(sg[a], sg[b]) << 2));  // physical, ascending
        } else if (o.mk == MK_2Q_MONO && n_nonone == 1 && moved == 0) {
          u.code = UC_PHASE;
          for (int r = 0; r < 4; ++r)
            if (cls_r[r] != E_ONE) {
              u.qb = static_cast<uint8_t>(sg[el(r)]);
              u.mcls = static_cast<uint16_t>(cls_r[r]);
              push(m + 2 * (r * 4 + r));
            }
        } else if (o.mk == MK_2Q_MONO) {
          u.code = UC_MONO;
          u.qb = po.qb[0];
          u.src = o.src;
          for (int r = 0; r < 4; ++r) {
            const int c = (o.src >> (2 * r)) & 3;
            push(m + 2 * (r * 4 + c));
            u.mcls |= static_cast<uint16_t>(entry_class(o.cls, r * 4 + c) << (3 * r));
          }
        } else {
          u.code = UC_GEN2;
          u.qb = po.qb[0];
          for (int e = 0; e < 16; ++e) push(m + 2 * e);
        }
      }
      if (mat > 0xFFFF) throw std::length_error("pass matrix table too large");
      d.uops.push_back(u);
    }
    it.begin = ubegin;
    it.end = static_cast<uint32_t>(d.uops.size()) - pd.uop_begin;
    it.sigma = pack(sg);
  }
  pd.uop_end = static_cast<uint32_t>(d.uops.size());
  // Per-shot Kraus matrix slot (16 entries) after the static matrices.
  pd.kraus_mat = mat;
  bool has_kraus = false;
  for (uint32_t i = pd.uop_begin; i < pd.uop_end; ++i)
    if (d.uops[i].code == UC_KRAUS1 || d.uops[i].code == UC_KRAUS2) {
      d.uops[i].mat = static_cast<uint16_t>(mat);
      has_kraus = true;
    }
  if (has_kraus) {
    for (int e = 0; e < 16; ++e) {
      d.uop_mats.push_back(0.0);
      d.uop_mats.push_back(0.0);
    }
    mat += 16;
  }
  if (mat > 0xFFFF) throw std::length_error("pass matrix table too large");
  pd.mat_count = mat;
  for (uint32_t it_i = pd.item_begin; it_i < pd.item_end; ++it_i)
    if (d.items[it_i].kind == IT_SEGMENT) assign_shape(d, d.items[it_i], pd.uop_begin);
}

}  // namespace

// Greedy in-order pass formation: consecutive gates / Pauli sites whose union
// of qubits (plus the always-local low qubits, for coalesced tile rows) fits k
// local qubits share one HBM read+write of the state. Ops are never reordered
// (gates on disjoint qubits do not commute bitwise in floating point); Kraus /
// measure / reset sites end a pass. Inside a pass, ops are grouped into
// register segments (segment_ops).
void plan_passes(HostDevProgram& d, unsigned tile_k, bool fuse_kraus) {
  d.shapes.clear();
  d.passes.clear();
  d.items.clear();
  d.pass_ops.clear();
  d.uops.clear();
  d.uop_mats.clear();
  d.steps.clear();
  const unsigned n = d.n;
  const unsigned k = std::min(tile_k, n);
  d.tile_k = k;
  // Always-local low qubits (coalesced 2^low-amplitude rows), leaving room for
  // any 2-qubit op so a fresh pass can always take the next op.
  const unsigned low_bits = k >= 2 ? std::min(3u, k - 2) : 0;
  const uint32_t low = (1u << low_bits) - 1;
  uint32_t cur = low;
  std::vector<uint32_t> cur_ops;
  bool need_init = true;
  size_t staged = 0;

  // epi_site: the Kraus site whose decide step follows this pass; when the
  // pass can hold its reduction's index structure (the target(s) plus the
  // lowest 9 (1q) / 3 (2q) other qubits), the pass computes that site's
  // matrix-0 partial sums in an epilogue (PassDesc::epi_*).
  auto close = [&](bool force, int64_t epi_site = -1) {
    staged = 0;
    if (cur_ops.empty() && !(force && need_init)) {
      cur = low;
      return;
    }
    uint32_t mask = cur;
    uint32_t epi_req = 0, epi_tq[2] = {0, 0}, epi_arity = 0;
    uint32_t epi_lowq[9];
    unsigned epi_nlow = 0;
    if (epi_site >= 0 && k >= 10) {
      const DevOp& ko = d.ops[static_cast<size_t>(epi_site)];
      const DevChannel& ch = d.channels[ko.aux];
      epi_arity = ch.arity;
      const unsigned want = ch.arity == 1 ? 9u : 3u;
      // 1q: pairs = 2^(n-1) >= 512 (blocks of exactly 512); 2q: groups >= 8
      // (and at most 128 partials per tile: EpiTables in tile_pass.cuh)
      const bool sized = (ch.arity == 1 ? n >= 10 : n >= 5) && k - ch.arity - want <= 7;
      if (sized && (ch.arity == 1 || ch.arity == 2)) {
        uint32_t tm = 0;
        for (unsigned b = 0; b < ch.arity; ++b) {
          epi_tq[b] = ko.q[b];
          tm |= 1u << ko.q[b];
        }
        epi_req = tm;
        for (unsigned q = 0; q < n && epi_nlow < want; ++q)
          if (!(tm >> q & 1)) {
            epi_lowq[epi_nlow++] = q;
            epi_req |= 1u << q;
          }
        if (static_cast<unsigned>(std::popcount(mask | epi_req)) <= k) mask |= epi_req;
        else epi_req = 0;
      }
    }
    for (unsigned q = 0; q < n && static_cast<unsigned>(std::popcount(mask)) < k; ++q) mask |= 1u << q;
    PassDesc pd{};
    pd.lmask = mask;
    pd.k = static_cast<uint8_t>(k);
    pd.first = need_init;
    need_init = false;
    uint8_t pos[32] = {};
    for (unsigned q = 0, j = 0; q < n; ++q)
      if (mask >> q & 1) {
        pd.lq[j] = static_cast<uint8_t>(q);
        pos[q] = static_cast<uint8_t>(j++);
      }
    if (epi_req) {
      pd.epi_kind = static_cast<uint8_t>(epi_arity);
      pd.epi_op = static_cast<uint32_t>(epi_site);
      for (unsigned b = 0; b < epi_arity; ++b) pd.epi_t[b] = pos[epi_tq[b]];
      pd.epi_nlow = static_cast<uint8_t>(epi_nlow);
      for (unsigned i = 0; i < epi_nlow; ++i) pd.epi_low[i] = pos[epi_lowq[i]];
      uint8_t nhi = 0;
      for (unsigned q = 0; q < n; ++q)
        if ((mask >> q & 1) && !(epi_req >> q & 1)) pd.epi_hi[nhi++] = pos[q];
      pd.epi_nhi = nhi;
    }
    pd.item_begin = static_cast<uint32_t>(d.items.size());
    const uint32_t po_begin = static_cast<uint32_t>(d.pass_ops.size());
    segment_ops(d, cur_ops, pos, k);
    pd.item_end = static_cast<uint32_t>(d.items.size());
    build_uops(d, pd, po_begin);
    d.steps.push_back({S_PASS, static_cast<uint32_t>(d.passes.size())});
    d.passes.push_back(pd);
    cur = low;
    cur_ops.clear();
  };

  auto add = [&](uint32_t i) {
    const DevOp& o = d.ops[i];
    uint32_t qm = 0;
    for (unsigned b = 0; b < o.nq; ++b) qm |= 1u << o.q[b];
    if (static_cast<unsigned>(std::popcount(cur | qm)) > k || staged + stage_bytes(o) > kMaxPassStageBytes) {
      close(false);
      staged = 0;
    }
    cur |= qm;
    cur_ops.push_back(i);
    staged += stage_bytes(o);
  };
  for (uint32_t i = 0; i < d.end; ++i) {
    const DevOp& o = d.ops[i];
    if (o.kind == K_BARRIER || (o.kind == K_GATE && o.skip)) continue;
    if (fused_kind(o)) {
      add(i);
    } else if (o.kind == K_KRAUS && fuse_kraus && k >= 2) {
      // Probabilities and per-shot choice between passes; the apply becomes
      // the first micro-op of the next pass (no separate HBM sweep), and the
      // pass before computes the probabilities' matrix-0 partials.
      close(true, i);
      d.steps.push_back({S_KRAUS_DECIDE, i});
      add(i);
    } else {
      close(true);
      d.steps.push_back({S_SPECIAL, i});
    }
  }
  close(true);
  if (d.eligible) d.steps.push_back({S_SAMPLE, 0});
}

void plan_resident(HostDevProgram& d) {
  d.passes.clear();
  d.items.clear();
  d.pass_ops.clear();
  d.steps.clear();
  const unsigned n = d.n;
  d.tile_k = n;
  PassDesc pd{};
  pd.lmask = n >= 32 ? ~0u : (1u << n) - 1;
  pd.k = static_cast<uint8_t>(n);
  pd.first = 1;
  uint8_t pos[32] = {};
  for (unsigned q = 0; q < n; ++q) pos[q] = pd.lq[q] = static_cast<uint8_t>(q);
  pd.item_begin = 0;
  std::vector<uint32_t> run;
  for (uint32_t i = 0; i < d.end; ++i) {
    const DevOp& o = d.ops[i];
    if (o.kind == K_BARRIER || (o.kind == K_GATE && o.skip)) continue;
    if (fused_kind(o)) {
      run.push_back(i);
      continue;
    }
    segment_ops(d, run, pos, n);
    run.clear();
    Item sp{};
    sp.kind = IT_SPECIAL;
    sp.shape = kNoShape;
    sp.begin = i;
    d.items.push_back(sp);
  }
  segment_ops(d, run, pos, n);
  pd.item_end = static_cast<uint32_t>(d.items.size());
  // Micro-op lowering (CX / SWAP relabeling, specialised U layouts) for the
  // resident kernel's staged segments, for states of up to 10 qubits (the
  // one-warp-CTA build: C1 14.1M -> 18.7M shots/s). Larger resident states
  // keep the direct per-op segments: the staged tables' shared memory would
  // cost a CTA per SM (C3 batch 533k -> 431k shots/s).
  d.uops.clear();
  d.uop_mats.clear();
  d.shapes.clear();
  if (n >= 2 && n <= 10) build_uops(d, pd, 0);
  d.passes.push_back(pd);
}

namespace {

// Parses one micro-op of a shape key back (see assign_shape).
struct ShapeOp {
  unsigned code, qb, src, mcls, sigma, off;
  unsigned long long cls;
  unsigned pos;  // UC_PAULI: index within the item (per-shot draw table)
};

std::vector<ShapeOp> parse_shape(const std::string& key, unsigned* final_sigma) {
  std::vector<ShapeOp> ops;
  size_t i = 0;
  while (i < key.size() && key[i] != '|') {
    ShapeOp o{};
    if (key[i] == 'P') {
      o.code = UC_PAULI;
      if (std::sscanf(key.c_str() + i, "P.%u.%u;", &o.sigma, &o.pos) != 2) throw std::logic_error("bad shape key");
      ops.push_back(o);
      i = key.find(';', i) + 1;
      continue;
    }
    if (std::sscanf(key.c_str() + i, "%u.%u.%u.%u.%u.%llx.%u;", &o.code, &o.qb, &o.src, &o.mcls, &o.sigma, &o.cls,
                    &o.off) != 7)
      throw std::logic_error("bad shape key");
    ops.push_back(o);
    i = key.find(';', i) + 1;
  }
  *final_sigma = static_cast<unsigned>(std::stoul(key.substr(i + 1)));
  return ops;
}

}  // namespace

// One straight-line executor per shape: the segment's micro-ops with every
// operand a compile-time constant (register pairs, relabelings, entry classes,
// matrix offsets), so the quads stay in registers with no per-op dispatch.
// Each executor performs exactly the interpreter's arithmetic
// (run_segment_staged), op for op.
std::string shape_source(const HostDevProgram& d) {
  std::string src = "namespace ssb {\n";
  char buf[512];
  // Drawn Paulis inline (fastest) while the shape set is small; out of line
  // (one shared body) when many Pauli positions would make the run-time
  // compile slow (random circuits: ~60 s -> ~15 s).
  size_t pauli_positions = 0;
  for (const std::string& key : d.shapes)
    for (size_t p = key.find("P."); p != std::string::npos; p = key.find("P.", p + 2)) ++pauli_positions;
  const char* pauli_macro = pauli_positions <= 100 ? "SSB_SHAPE_PAULI_INLINE" : "SSB_SHAPE_PAULI";
  for (size_t id = 0; id < d.shapes.size(); ++id) {
    unsigned fs = 0;
    const std::vector<ShapeOp> ops = parse_shape(d.shapes[id], &fs);
    // NOISY = 0: every Pauli draw of the shot identity (skipped); NOISY = 1:
    // some drew a Pauli — applied where pinfo[pos] != 0xFF (uniform branch).
    std::snprintf(buf, sizeof buf,
                  "template <int NOISY>\nstatic __device__ __forceinline__ void ssb_shape_%zu(double2* st, unsigned k, "
                  "unsigned la, unsigned lb, const double2* m, uint64_t kcls, const uint8_t* pinfo) {\n"
                  "  SSB_SHAPE_BEGIN\n",
                  id);
    src += buf;
    for (const ShapeOp& o : ops) {
      const unsigned a0 = o.qb & 3, a1 = (o.qb >> 2) & 3, b0 = (o.qb >> 4) & 3, b1 = (o.qb >> 6) & 3;
      switch (o.code) {
        case UC_PAULI:
          std::snprintf(buf, sizeof buf, "  if (NOISY) { %s(%u, pinfo[%u]) }\n", pauli_macro, o.sigma, o.pos);
          break;
        case UC_U:
        case UC_REAL:
        case UC_GEN1:
          std::snprintf(buf, sizeof buf,
                        "  { const double2 mm[4] = {m[%u], m[%u], m[%u], m[%u]}; "
                        "quad_apply1p<%u, %u, %u, %u, %s, true>(v, mm, 0x%llxull, QPT); }\n",
                        o.off, o.off + 1, o.off + 2, o.off + 3, a0, a1, b0, b1,
                        o.code == UC_U ? "MK_1Q_U" : o.code == UC_REAL ? "MK_1Q_REAL" : "MK_1Q_GEN", o.cls);
          break;
        case UC_KRAUS1:  // the shot's chosen M/sqrt(p): runtime entry classes
          std::snprintf(buf, sizeof buf,
                        "  { const double2 mm[4] = {m[%u], m[%u], m[%u], m[%u]}; "
                        "quad_apply1p<%u, %u, %u, %u, MK_1Q_GEN, true>(v, mm, kcls, QPT); }\n",
                        o.off, o.off + 1, o.off + 2, o.off + 3, a0, a1, b0, b1);
          break;
        case UC_SWAP:
          std::snprintf(buf, sizeof buf, "  quad_swap<%u, %u>(v, QPT);\n", std::min(a0, a1), std::max(a0, a1));
          break;
        case UC_PHASE:
          std::snprintf(buf, sizeof buf, "  quad_phase<%u>(v, m[%u], %uu, QPT);\n", o.qb & 3, o.off, o.mcls);
          break;
        default:  // UC_MONO / UC_GEN2 / UC_KRAUS2 through the logical view (constant relabeling)
          std::snprintf(buf, sizeof buf,
                        "  { Uop u{}; u.code = %u; u.qb = %u; u.src = %u; u.mcls = %u; u.sigma = %u;\n"
                        "    SSB_SHAPE_LOGICAL(u, m + %u, %s) }\n",
                        o.code, o.qb, o.src, o.mcls, o.sigma, o.off,
                        o.code == UC_KRAUS2 ? "kcls" : (std::to_string(o.cls) + "ull").c_str());
          break;
      }
      src += buf;
    }
    std::snprintf(buf, sizeof buf, "  SSB_SHAPE_END(%u)\n}\n", fs);
    src += buf;
  }
  src += "static __device__ __forceinline__ bool ssb_run_shape(unsigned id, bool noisy, double2* st, unsigned k, "
         "unsigned la, unsigned lb, const double2* m, uint64_t kcls, const uint8_t* pinfo) {\n  switch (id) {\n";
  for (size_t id = 0; id < d.shapes.size(); ++id) {
    std::snprintf(buf, sizeof buf,
                  "    case %zu: if (noisy) ssb_shape_%zu<1>(st, k, la, lb, m, kcls, pinfo); "
                  "else ssb_shape_%zu<0>(st, k, la, lb, m, kcls, pinfo); return true;\n",
                  id, id, id);
    src += buf;
  }
  src += "    default: return false;\n  }\n}\n}  // namespace ssb\n";
  return src;
}

}  // namespace ssb
