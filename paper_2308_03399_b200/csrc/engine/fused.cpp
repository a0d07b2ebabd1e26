// Fused-matrix planner (fused.hpp): blocks, their products and folded Pauli
// factors, the HBM tile-pass schedule over the block DAG and the rounding
// bound behind the sampler's guard band.
#include "fused.hpp"

#include <algorithm>
#include <array>
#include <bit>
#include <cmath>
#include <complex>
#include <cstdlib>
#include <limits>
#include <map>
#include <mutex>
#include <string>

namespace ssb {

namespace {

using cld = std::complex<long double>;
using M4 = std::array<cld, 16>;  // row-major: (r, c) at r * 4 + c

M4 eye4() {
  M4 m{};
  for (int i = 0; i < 4; ++i) m[i * 5] = 1.0L;
  return m;
}

M4 mul(const M4& a, const M4& b) {
  M4 c{};
  for (int r = 0; r < 4; ++r)
    for (int col = 0; col < 4; ++col) {
      cld s = 0.0L;
      for (int k = 0; k < 4; ++k) s += a[r * 4 + k] * b[k * 4 + col];
      c[r * 4 + col] = s;
    }
  return c;
}

M4 dagger(const M4& a) {
  M4 c{};
  for (int r = 0; r < 4; ++r)
    for (int col = 0; col < 4; ++col) c[r * 4 + col] = std::conj(a[col * 4 + r]);
  return c;
}

struct Elem {
  bool pauli;
  uint32_t op;
};

struct Blk {
  unsigned q0, q1;  // matrix bit 0 / bit 1 qubits (q0 < q1)
  std::vector<Elem> elems;
};

// Block-basis bit of qubit q.
unsigned bit_of(const Blk& b, unsigned q) { return q == b.q0 ? 0u : 1u; }

// Gate op embedded in the block basis (program.hpp: qubits[0] = low matrix axis).
M4 embed_gate(const HostDevProgram& h, const DevOp& o, const Blk& b) {
  const double* g = &h.mats[size_t{o.aux} * 32];
  const unsigned d = 1u << o.nq;
  auto G = [&](unsigned r, unsigned c) { return cld(g[2 * (r * d + c)], g[2 * (r * d + c) + 1]); };
  auto gidx = [&](unsigned r) {
    unsigned x = 0;
    for (unsigned j = 0; j < o.nq; ++j) x |= ((r >> bit_of(b, o.q[j])) & 1u) << j;
    return x;
  };
  // Block bits not touched by the gate must match between row and column.
  unsigned touched = 0;
  for (unsigned j = 0; j < o.nq; ++j) touched |= 1u << bit_of(b, o.q[j]);
  M4 m{};
  for (unsigned r = 0; r < 4; ++r)
    for (unsigned c = 0; c < 4; ++c)
      if (((r ^ c) & ~touched & 3u) == 0) m[r * 4 + c] = G(gidx(r), gidx(c));
  return m;
}

// Pauli term (destination-sign form, kernels_scalar.cpp:58-81):
// new[i] = (-i)^num_y (-1)^popcount(i & z) old[i ^ x], restricted to the block.
M4 embed_pauli(const DevTerm& t, const Blk& b) {
  unsigned xb = 0, zb = 0;
  for (unsigned q : {b.q0, b.q1}) {
    xb |= ((t.x >> q) & 1u) << bit_of(b, q);
    zb |= ((t.z >> q) & 1u) << bit_of(b, q);
  }
  static const cld phase[4] = {cld(1, 0), cld(0, -1), cld(-1, 0), cld(0, 1)};
  const cld ph = phase[t.num_y & 3u];
  M4 m{};
  for (unsigned r = 0; r < 4; ++r) m[r * 4 + (r ^ xb)] = (std::popcount(r & zb) & 1) ? -ph : ph;
  return m;
}

uint32_t push(FusedPlan& f, const M4& m) {
  const uint32_t idx = static_cast<uint32_t>(f.mats.size() / 32);
  for (const cld& e : m) {
    f.mats.push_back(static_cast<double>(e.real()));
    f.mats.push_back(static_cast<double>(e.imag()));
  }
  return idx;
}

}  // namespace

FusedPlan plan_fused(const HostDevProgram& h, unsigned tile_k, unsigned gq) {
  FusedPlan f;
  const unsigned n = h.n;
  if (n < 3) {
    f.why = "fewer than 3 qubits";
    return f;
  }
  if (h.eligible && h.sample_qubits.size() != n) {
    f.why = "terminal sampling over a subset of the qubits";
    return f;
  }
  for (uint32_t i = 0; i < h.end; ++i) {
    const DevOp& o = h.ops[i];
    const bool ok = o.kind == K_BARRIER || ((o.kind == K_GATE || o.kind == K_PAULI) && !o.has_cond && o.nq <= 2);
    if (!ok) {
      f.why = "op " + std::to_string(i) + " is not an unconditioned gate / Pauli site on <= 2 qubits";
      return f;
    }
  }

  // ---- blocks (greedy: an op joins the last block on its qubits when that
  // block is the last one touching each of them; 1q ops wait for the next 2q
  // block on their qubit) ----
  std::vector<Blk> blks;
  std::vector<int> frontier(n, -1);
  std::vector<std::vector<Elem>> pending(n);
  uint64_t exact_gates = 0;
  for (uint32_t i = 0; i < h.end; ++i) {
    const DevOp& o = h.ops[i];
    if (o.kind == K_BARRIER) continue;
    if (o.kind == K_GATE) {
      if (o.skip) continue;  // exact identity: no factor
      ++exact_gates;
    }
    const Elem e{o.kind == K_PAULI, i};
    if (o.nq == 1) {
      const unsigned q = o.q[0];
      if (frontier[q] >= 0) blks[frontier[q]].elems.push_back(e);
      else pending[q].push_back(e);
      continue;
    }
    const unsigned a = o.q[0], c = o.q[1];
    if (frontier[a] >= 0 && frontier[a] == frontier[c]) {
      blks[frontier[a]].elems.push_back(e);
      continue;
    }
    Blk b{std::min(a, c), std::max(a, c), {}};
    for (unsigned q : {a, c}) {
      b.elems.insert(b.elems.end(), pending[q].begin(), pending[q].end());
      pending[q].clear();
    }
    b.elems.push_back(e);
    frontier[a] = frontier[c] = static_cast<int>(blks.size());
    blks.push_back(std::move(b));
  }
  for (unsigned q = 0; q < n; ++q)
    if (!pending[q].empty()) {  // a qubit no 2q op ever touches: I (x) G on a partner
      const unsigned partner = q == 0 ? 1 : 0;
      Blk b{std::min(q, partner), std::max(q, partner), std::move(pending[q])};
      blks.push_back(std::move(b));
    }

  // ---- products, folded Pauli factors ----
  std::vector<uint32_t> base(blks.size());
  std::vector<std::pair<uint32_t, uint32_t>> site_range(blks.size());
  double work = 16.0 * static_cast<double>(exact_gates);  // reference's own rounding
  for (size_t bi = 0; bi < blks.size(); ++bi) {
    const Blk& b = blks[bi];
    // suffix[j] = product of the gates after element j (V_j), built backwards.
    std::vector<M4> after(b.elems.size());
    M4 acc = eye4();
    for (size_t j = b.elems.size(); j-- > 0;) {
      after[j] = acc;
      const Elem& e = b.elems[j];
      if (!e.pauli) acc = mul(acc, embed_gate(h, h.ops[e.op], b));
    }
    base[bi] = push(f, acc);  // acc = G_k ... G_1
    site_range[bi].first = static_cast<uint32_t>(f.sites.size());
    for (size_t j = 0; j < b.elems.size(); ++j) {
      const Elem& e = b.elems[j];
      if (!e.pauli) continue;
      const DevOp& o = h.ops[e.op];
      FSite s{o.site, static_cast<uint32_t>(f.qidx.size())};
      const M4 vd = dagger(after[j]);
      for (uint32_t t = 0; t < o.count; ++t) {
        const DevTerm& term = h.terms[o.aux + t];
        f.qidx.push_back(term.identity ? kNoQ : push(f, mul(mul(after[j], embed_pauli(term, b)), vd)));
      }
      f.sites.push_back(s);
    }
    site_range[bi].second = static_cast<uint32_t>(f.sites.size());
    // fused rounding: the product's representation + the apply, and per
    // drawn site one more factor (product or extra apply)
    work += 16.0 + 16.0 * (site_range[bi].second - site_range[bi].first);
  }
  // Margin x4 over the per-operation constants (complex 2x2 / 4x4 products
  // with and without FMA stay below 16 unit roundoffs of the state norm).
  f.err_bound = 4.0 * work * std::ldexp(1.0, -53);

  // ---- HBM tile passes over the block DAG ----
  const unsigned k = std::min(tile_k, n);
  f.k = k;
  const uint32_t low = (1u << std::min(3u, k - 2)) - 1;
  const uint32_t all = n >= 32 ? ~0u : (1u << n) - 1;
  // Blocks per pass (shared-memory staging): kFusedMaxPassBlocks, or the
  // SHOTSIM_B200_FUSED_CAP tuning override (8..64).
  uint32_t cap = kFusedMaxPassBlocks;
  if (const char* v = std::getenv("SHOTSIM_B200_FUSED_CAP"); v && *v)
    cap = std::max<uint32_t>(8, std::min<uint32_t>(64, static_cast<uint32_t>(std::strtoul(v, nullptr, 10))));
  std::vector<uint32_t> remaining(blks.size());
  for (uint32_t i = 0; i < remaining.size(); ++i) remaining[i] = i;
  bool first = true;
  // Blocks a pass with the fixed local set L takes from `rem` (in order; a
  // block is blocked once an earlier untaken block shares a qubit).
  auto take_from = [&](const std::vector<uint32_t>& rem, uint32_t L, std::vector<uint32_t>* taken,
                       std::vector<uint32_t>* rest) {
    uint32_t blocked = 0;
    size_t cnt = 0;
    for (size_t r = 0; r < rem.size(); ++r) {
      const uint32_t b = rem[r];
      const uint32_t qm = (1u << blks[b].q0) | (1u << blks[b].q1);
      if (!(qm & blocked) && (qm & ~L) == 0 && cnt < cap) {
        ++cnt;
        if (taken) taken->push_back(b);
      } else {
        blocked |= qm;
        if (rest) rest->push_back(b);
      }
      if (blocked == all && !rest) break;
    }
    return cnt;
  };
  // One-pass lookahead in the exhaustive local-set search (default on;
  // SHOTSIM_B200_FUSED_LOOKAHEAD=0 disables): C2 9 -> 8 passes, +0.6%.
  const char* lv = std::getenv("SHOTSIM_B200_FUSED_LOOKAHEAD");
  const bool lookahead = !(lv && *lv == '0');
  const char* pv = std::getenv("SHOTSIM_B200_FUSED_GREEDY_PASSES");
  const bool greedy_passes = pv && *pv && *pv != '0';
  // The local set of the next pass over `rem`: first-fit, then hill-climbing
  // one-qubit swaps, then (small registers) every subset with one pass of
  // lookahead. `top` (optional) receives the best-scoring sets, best first.
  auto choose_local = [&](const std::vector<uint32_t>& rem, std::vector<uint32_t>* top) {
    uint32_t L = low, blocked = 0;
    size_t nt = 0;
    for (size_t r = 0; r < rem.size(); ++r) {
      const uint32_t b = rem[r];
      const uint32_t qm = (1u << blks[b].q0) | (1u << blks[b].q1);
      if (!(qm & blocked) && static_cast<unsigned>(std::popcount(L | qm)) <= k && nt < cap) {
        L |= qm;
        ++nt;
      } else {
        blocked |= qm;
      }
      if (blocked == all) break;
    }
    for (unsigned q = 0; q < n && static_cast<unsigned>(std::popcount(L)) < k; ++q) L |= 1u << q;
    if (greedy_passes || k >= n) return L;
    size_t best = take_from(rem, L, nullptr, nullptr);
    for (bool improved = true; improved;) {
      improved = false;
      for (unsigned qi = 0; qi < n && !improved; ++qi) {
        if (!(L >> qi & 1) || (low >> qi & 1)) continue;
        for (unsigned qo = 0; qo < n && !improved; ++qo) {
          if (L >> qo & 1) continue;
          const uint32_t L2 = (L & ~(1u << qi)) | (1u << qo);
          const size_t got = take_from(rem, L2, nullptr, nullptr);
          if (got > best) best = got, L = L2, improved = true;
        }
      }
    }
    const unsigned free_q = n - static_cast<unsigned>(std::popcount(low));
    const unsigned pick = k - static_cast<unsigned>(std::popcount(low));
    double combos = 1.0;
    for (unsigned i = 0; i < pick; ++i) combos = combos * (free_q - i) / (i + 1);
    const double scan = combos * static_cast<double>(rem.size());  // bounded work
    if (combos <= 20000.0 && scan <= 3e7 && std::getenv("SHOTSIM_B200_FUSED_NO_EXHAUSTIVE") == nullptr) {
      std::vector<unsigned> fq;
      for (unsigned q = 0; q < n; ++q)
        if (!(low >> q & 1)) fq.push_back(q);
      std::vector<unsigned> idx(pick);
      for (unsigned i = 0; i < pick; ++i) idx[i] = i;
      std::vector<uint32_t> sets;
      while (true) {
        uint32_t L2 = low;
        for (unsigned i : idx) L2 |= 1u << fq[i];
        sets.push_back(L2);
        int i = static_cast<int>(pick) - 1;  // next combination
        while (i >= 0 && idx[i] == fq.size() - pick + i) --i;
        if (i < 0) break;
        ++idx[i];
        for (unsigned j = i + 1; j < pick; ++j) idx[j] = idx[j - 1] + 1;
      }
      std::vector<std::pair<size_t, uint32_t>> scored;
      for (uint32_t L2 : sets) scored.emplace_back(take_from(rem, L2, nullptr, nullptr), L2);
      std::stable_sort(scored.begin(), scored.end(), [](const auto& a, const auto& b) { return a.first > b.first; });
      if (!scored.empty() && scored[0].first > best) best = scored[0].first, L = scored[0].second;
      if (lookahead && rem.size() > best && 24.0 * scan <= 3e8) {
        size_t best2 = 0;
        const size_t ntop = std::min<size_t>(scored.size(), 24);
        for (size_t c = 0; c < ntop; ++c) {
          std::vector<uint32_t> r1;
          take_from(rem, scored[c].second, nullptr, &r1);
          size_t next = 0;
          for (uint32_t L3 : sets) next = std::max(next, take_from(r1, L3, nullptr, nullptr));
          if (scored[c].first + next > best2) best2 = scored[c].first + next, L = scored[c].second;
        }
      }
      if (top) {
        top->push_back(L);
        for (size_t c = 0; c < scored.size() && top->size() < 8; ++c)
          if (scored[c].second != L && scored[c].first + 2 >= scored[0].first) top->push_back(scored[c].second);
      }
    }
    return L;
  };
  // Register groups a pass over these blocks needs (greedy largest closure):
  // the cost model of the plan rollouts below.
  auto count_groups = [&](const std::vector<uint32_t>& bl) {
    std::vector<uint32_t> qm(bl.size());
    for (size_t t = 0; t < bl.size(); ++t) qm[t] = (1u << blks[bl[t]].q0) | (1u << blks[bl[t]].q1);
    std::vector<char> pl(bl.size(), 0);
    auto closure = [&](uint32_t gm, bool commit) {
      std::vector<char> q = pl;
      size_t cnt = 0;
      for (bool grew = true; grew;) {
        grew = false;
        uint32_t pending = 0;
        for (size_t t = 0; t < bl.size(); ++t) {
          if (q[t]) continue;
          if (!(qm[t] & pending) && std::popcount(gm | qm[t]) <= static_cast<int>(gq)) {
            gm |= qm[t], q[t] = 1, ++cnt, grew = true;
          } else {
            pending |= qm[t];
          }
        }
      }
      if (commit) pl = q;
      return cnt;
    };
    size_t groups = 0;
    for (size_t left = bl.size(); left > 0; ++groups) {
      std::vector<size_t> ready;
      uint32_t pq = 0;
      for (size_t t = 0; t < bl.size(); ++t) {
        if (pl[t]) continue;
        if (!(qm[t] & pq)) ready.push_back(t);
        pq |= qm[t];
      }
      uint32_t bq = 0;
      size_t bc = 0;
      for (size_t a : ready)
        for (size_t c = 0; c < bl.size(); ++c) {
          if (pl[c]) continue;
          const uint32_t q = qm[a] | qm[c];
          if (std::popcount(q) > static_cast<int>(gq)) continue;
          const size_t got = closure(q, false);
          if (got > bc) bc = got, bq = q;
        }
      if (bc == 0) break;
      closure(bq, true);
      left -= bc;
    }
    return groups;
  };
  // Cost of finishing the plan greedily from `rem` (a pass's tile IO costs
  // about four register groups: profiles/r02/fused_variants.log).
  constexpr double kPassCost = 4.0;
  auto rollout_cost = [&](std::vector<uint32_t> rem) {
    double cost = 0.0;
    while (!rem.empty()) {
      const uint32_t L = choose_local(rem, nullptr);
      std::vector<uint32_t> t, r;
      take_from(rem, L, &t, &r);
      if (t.empty()) return 1e300;
      cost += kPassCost + static_cast<double>(count_groups(t));
      rem.swap(r);
    }
    return cost;
  };
  const char* rv = std::getenv("SHOTSIM_B200_FUSED_ROLLOUT");
  const bool plan_rollout = !(rv && *rv == '0');
  while (first || !remaining.empty()) {
    std::vector<uint32_t> taken, rest, top;
    uint32_t L = choose_local(remaining, &top);
    // Plan rollouts (small plans): among the best-scoring local sets, the
    // one whose pass + greedy completion costs the fewest passes and groups.
    if (plan_rollout && top.size() > 1 && remaining.size() <= 400) {
      double best_cost = 1e300;
      for (uint32_t L2 : top) {
        std::vector<uint32_t> t, r;
        take_from(remaining, L2, &t, &r);
        if (t.empty()) continue;
        const double c = kPassCost + static_cast<double>(count_groups(t)) + rollout_cost(r);
        if (c < best_cost - 1e-9) best_cost = c, L = L2;
      }
    }
    take_from(remaining, L, &taken, &rest);
    remaining.swap(rest);
    FPass pd{};
    pd.lmask = L;
    pd.k = static_cast<uint8_t>(k);
    pd.first = first;
    first = false;
    uint8_t pos[32] = {};
    for (unsigned q = 0, j = 0; q < n; ++q)
      if (L >> q & 1) {
        pd.lq[j] = static_cast<uint8_t>(q);
        pos[q] = static_cast<uint8_t>(j++);
      }
    // Register groups: repeatedly open a group with the first block whose
    // predecessors in the pass are applied, then add every ready block whose
    // qubits keep the group within four local positions (blocks sharing a
    // qubit keep their order; disjoint ones commute).
    const char* gv = std::getenv("SHOTSIM_B200_FUSED_GREEDY");
    const bool greedy_groups = gv && *gv && *gv != '0';
    pd.grp_begin = static_cast<uint32_t>(f.groups.size());
    pd.blk_begin = static_cast<uint32_t>(f.blocks.size());
    std::vector<char> placed(taken.size(), 0);
    size_t nplaced = 0;
    uint32_t sites_in_pass = 0;
    auto qmask = [&](size_t t) { return (1u << blks[taken[t]].q0) | (1u << blks[taken[t]].q1); };
    // The blocks one group starting from qubit set gm0 would take (in order):
    // every block whose earlier unplaced blocks share none of its qubits and
    // whose qubits keep the group within gq, rescanned until nothing grows.
    auto closure = [&](uint32_t gm0, std::vector<char> pl, std::vector<size_t>* order) {
      uint32_t gm = gm0;
      size_t cnt = 0;
      for (bool grew = true; grew;) {
        grew = false;
        uint32_t pending_q = 0;
        for (size_t t = 0; t < taken.size(); ++t) {
          if (pl[t]) continue;
          const uint32_t qm = qmask(t);
          if (!(qm & pending_q) && std::popcount(gm | qm) <= static_cast<int>(gq)) {
            gm |= qm;
            pl[t] = 1;
            ++cnt;
            grew = true;
            if (order) order->push_back(t);
          } else {
            pending_q |= qm;
          }
        }
      }
      return cnt;
    };
    // Candidate seeds: qubit sets spanned by one or two ready blocks.
    auto seeds = [&](const std::vector<char>& pl) {
      std::vector<size_t> ready;
      uint32_t pq = 0;
      for (size_t t = 0; t < taken.size(); ++t) {
        if (pl[t]) continue;
        if (!(qmask(t) & pq)) ready.push_back(t);
        pq |= qmask(t);
      }
      // (the second block may be any unplaced one: it can become ready
      // inside the group once its predecessors there are applied)
      std::vector<uint32_t> out;
      for (size_t a = 0; a < ready.size(); ++a)
        for (size_t c = 0; c < taken.size(); ++c) {
          if (pl[c]) continue;
          const uint32_t q = qmask(ready[a]) | qmask(c);
          if (std::popcount(q) <= static_cast<int>(gq) && std::find(out.begin(), out.end(), q) == out.end())
            out.push_back(q);
        }
      return out;
    };
    // Groups a greedy largest-closure seeding needs to place the rest.
    auto rollout = [&](std::vector<char> pl) {
      size_t groups = 0;
      for (size_t left = std::count(pl.begin(), pl.end(), 0); left > 0; ++groups) {
        uint32_t bq = 0;
        size_t bc = 0;
        for (uint32_t q : seeds(pl)) {
          const size_t got = closure(q, pl, nullptr);
          if (got > bc) bc = got, bq = q;
        }
        std::vector<size_t> ord;
        closure(bq, pl, &ord);
        for (size_t t : ord) pl[t] = 1;
        left -= ord.size();
        if (ord.empty()) break;  // cannot happen: a ready block always fits
      }
      return groups;
    };
    while (nplaced < taken.size()) {
      // Seed: the qubit set (the union of one or two ready blocks) after
      // which a greedy largest-closure rollout needs the fewest groups for
      // the rest of the pass — a first-fit seed often closes the group after
      // two blocks (SHOTSIM_B200_FUSED_GREEDY=1 keeps first-fit).
      uint32_t seed_q = 0;
      if (!greedy_groups) {
        size_t best_total = ~size_t{0}, best_now = 0;
        for (uint32_t q : seeds(placed)) {
          std::vector<size_t> ord;
          const size_t got = closure(q, placed, &ord);
          std::vector<char> pl = placed;
          for (size_t t : ord) pl[t] = 1;
          const size_t total = 1 + rollout(pl);
          if (total < best_total || (total == best_total && got > best_now))
            best_total = total, best_now = got, seed_q = q;
        }
      }
      std::vector<size_t> order;
      closure(seed_q, placed, &order);
      uint32_t gm = 0;  // group qubit mask
      FGroup g{};
      g.blk_begin = static_cast<uint32_t>(f.blocks.size());
      {
        for (size_t t : order) {
          const uint32_t b = taken[t];
          const uint32_t qm = qmask(t);
          {
            gm |= qm;
            placed[t] = 1;
            ++nplaced;
            FBlock fb{};
            fb.p0 = pos[blks[b].q0];
            fb.p1 = pos[blks[b].q1];
            fb.mat = base[b];
            fb.site_begin = site_range[b].first;
            fb.site_end = site_range[b].second;
            sites_in_pass += fb.site_end - fb.site_begin;
            f.blocks.push_back(fb);
          }
        }
      }
      // (group bits assigned below; then the lane / register bit schedule)
      uint32_t lm = 0;
      for (unsigned q = 0; q < n; ++q)
        if (gm >> q & 1) lm |= 1u << pos[q];
      for (unsigned j = 0; j < k && std::popcount(lm) < static_cast<int>(gq); ++j) lm |= 1u << j;
      for (unsigned j = 0, i = 0; j < k; ++j)
        if (lm >> j & 1) g.g[i++] = static_cast<uint8_t>(j);
      if (gq == 3) g.g[3] = static_cast<uint8_t>(k);  // unused slot (3-qubit groups)
      g.blk_end = static_cast<uint32_t>(f.blocks.size());
      for (uint32_t b = g.blk_begin; b < g.blk_end; ++b)
        for (uint8_t i = 0; i < 4; ++i) {
          if (g.g[i] == f.blocks[b].p0) f.blocks[b].gb0 = i;
          if (g.g[i] == f.blocks[b].p1) f.blocks[b].gb1 = i;
        }
      // Lane / register bit schedule for the tensor-core kernel: the lanes
      // start on the first block's bits; before each block, a lane bit the
      // block does not use is exchanged with the register bit it does use.
      {
        uint8_t lane[2] = {f.blocks[g.blk_begin].gb0, f.blocks[g.blk_begin].gb1};
        uint8_t reg[2], nr = 0;
        for (uint8_t i = 0; i < 4; ++i)
          if (i != lane[0] && i != lane[1]) reg[nr++] = i;
        g.init[0] = lane[0], g.init[1] = lane[1], g.init[2] = reg[0], g.init[3] = reg[1];
        for (uint32_t b = g.blk_begin; b < g.blk_end; ++b) {
          FBlock& fb = f.blocks[b];
          const auto want = [&](uint8_t x) { return x == fb.gb0 || x == fb.gb1; };
          uint8_t xch = 0, nx = 0;
          for (uint8_t pbit = 0; pbit < 2; ++pbit) {
            if (want(lane[pbit])) continue;
            const uint8_t qbit = want(reg[0]) && reg[0] != lane[pbit ^ 1] ? 0 : 1;
            std::swap(lane[pbit], reg[qbit]);
            xch |= static_cast<uint8_t>((8 | pbit << 1 | qbit) << (4 * nx++));
          }
          fb.xch = xch;
          fb.perm = lane[0] != fb.gb0;
        }
        g.fin[0] = lane[0], g.fin[1] = lane[1], g.fin[2] = reg[0], g.fin[3] = reg[1];
      }
      f.groups.push_back(g);
    }
    pd.grp_end = static_cast<uint32_t>(f.groups.size());
    pd.blk_end = static_cast<uint32_t>(f.blocks.size());
    f.max_pass_blocks = std::max<uint32_t>(f.max_pass_blocks, pd.blk_end - pd.blk_begin);
    f.max_pass_sites = std::max<uint32_t>(f.max_pass_sites, sites_in_pass);
    f.passes.push_back(pd);
  }
  f.num_blocks = static_cast<uint32_t>(blks.size());
  f.gq = gq;
  f.ok = true;
  return f;
}

// Plans are pure functions of the program's ops / terms / channels /
// matrices, the tile size, the group size and the planner knobs; a caller
// that lowers the same circuit again (the drop-in plugin flattens the
// program on every run) gets the cached plan instead of re-running the
// products and the local-set search (C2: ~50 ms).
FusedPlan plan_fused_cached(const HostDevProgram& h, unsigned tile_k, unsigned gq) {
  uint64_t h1 = 1469598103934665603ull, h2 = 0x9E3779B97F4A7C15ull;
  auto mix = [&](const void* p, size_t n) {
    const auto* b = static_cast<const unsigned char*>(p);
    for (size_t i = 0; i < n; ++i) {
      h1 = (h1 ^ b[i]) * 1099511628211ull;
      h2 = (h2 ^ b[i]) * 0x100000001B3ull + 0x632BE59BD9B4E019ull;
    }
  };
  const uint32_t scal[4] = {h.n, h.end, tile_k, gq};
  mix(scal, sizeof scal);
  mix(h.ops.data(), h.ops.size() * sizeof(DevOp));
  mix(h.terms.data(), h.terms.size() * sizeof(DevTerm));
  mix(h.channels.data(), h.channels.size() * sizeof(DevChannel));
  mix(h.mats.data(), h.mats.size() * sizeof(double));
  for (const char* k : {"SHOTSIM_B200_FUSED_CAP", "SHOTSIM_B200_FUSED_GREEDY", "SHOTSIM_B200_FUSED_GREEDY_PASSES",
                        "SHOTSIM_B200_FUSED_LOOKAHEAD", "SHOTSIM_B200_FUSED_NO_EXHAUSTIVE"}) {
    const char* v = std::getenv(k);
    const std::string kv = std::string(k) + "=" + (v ? v : "");
    mix(kv.data(), kv.size() + 1);
  }
  static std::mutex mu;
  static std::map<std::pair<uint64_t, uint64_t>, FusedPlan> cache;
  const auto key = std::make_pair(h1, h2);
  {
    std::lock_guard<std::mutex> lk(mu);
    if (auto it = cache.find(key); it != cache.end()) return it->second;
  }
  FusedPlan f = plan_fused(h, tile_k, gq);
  std::lock_guard<std::mutex> lk(mu);
  if (cache.size() >= 32) cache.erase(cache.begin());  // bounded (plans of up to ~MBs each)
  cache.emplace(key, f);
  return f;
}

}  // namespace ssb
