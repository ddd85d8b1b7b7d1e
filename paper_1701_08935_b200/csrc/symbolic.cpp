// Host symbolic analysis for the block-sparse factor path (north star:
// "ordering and symbolic analysis remain host-side setup").
//
//   nd_order        nested dissection by recursive BFS-level bisection: the
//                   median BFS level of each connected piece is its separator;
//                   pieces below `leaf` rows are ordered by reverse
//                   Cuthill-McKee inside. Nodes come out in post-order
//                   (children before their separator).
//   block_symbolic  nodes padded to whole 32-row tiles (identity padding
//                   rows), the block graph of the pattern, and its symbolic
//                   elimination (fill) through the block elimination tree:
//                   struct(k) = adj+(k) U (U_children struct(c) \ {k}).
//
// The reference orders by RCM and factors a band (rcm.hpp, band_factor.hpp);
// nested dissection is SURVEY.md §8(f) rank 2 ("host symbolic analysis: ND
// ordering, supernodes, etree"), here at 32x32-tile granularity.
#include <algorithm>
#include <atomic>
#include <cstdlib>
#include <exception>
#include <memory>
#include <cstdint>
#include <numeric>
#include <stdexcept>
#include <thread>
#include <vector>

#include "host.hpp"

namespace zolo {

namespace {

struct Graph {
  int64_t n;
  const int64_t* rp;
  const int64_t* ci;
};

// BFS over the vertices with mark[v] == tag; returns the visit order and fills level.
using Marks = std::unique_ptr<std::atomic<int>[]>;
inline int mk_get(const Marks& m, int64_t v) { return m[v].load(std::memory_order_relaxed); }
inline void mk_set(Marks& m, int64_t v, int t) { m[v].store(t, std::memory_order_relaxed); }

void bfs(const Graph& g, const Marks& mark, int tag, int64_t root, std::vector<int64_t>& level,
         std::vector<int64_t>& order) {
  order.clear();
  order.push_back(root);
  level[root] = 0;
  for (size_t h = 0; h < order.size(); ++h) {
    const int64_t u = order[h];
    for (int64_t k = g.rp[u]; k < g.rp[u + 1]; ++k) {
      const int64_t v = g.ci[k];
      if (mk_get(mark, v) == tag && level[v] < 0) {
        level[v] = level[u] + 1;
        order.push_back(v);
      }
    }
  }
}

// The two sides of a separator are independent subproblems: down to PAR_DEPTH the first side runs
// on its own host thread. Pieces are disjoint vertex sets, so `level` entries are touched by one
// thread only; `mark` entries of neighbours in other pieces are read concurrently (they never
// equal this piece's tag: tags are unique), hence the relaxed atomics. Every piece's result
// depends on the graph and the piece alone, so the ordering does not depend on the threading.
struct NdOut {
  std::vector<std::vector<int64_t>> nodes;  // elimination order of tree nodes
  std::vector<int> is_sep;
  void append(NdOut&& o) {
    for (auto& nd : o.nodes) nodes.push_back(std::move(nd));
    is_sep.insert(is_sep.end(), o.is_sep.begin(), o.is_sep.end());
  }
};
struct NdState {
  static constexpr int PAR_DEPTH = 3;
  const Graph& g;
  int64_t leaf;
  Marks mark;
  std::atomic<int> next_tag{1};
  std::vector<int64_t> level;
  explicit NdState(const Graph& gr, int64_t lf) : g(gr), leaf(lf), mark(new std::atomic<int>[gr.n]), level(gr.n, -1) {
    for (int64_t v = 0; v < gr.n; ++v) mk_set(mark, v, 0);
  }

  void emit_leaf(std::vector<int64_t>& idx, NdOut& out, std::vector<int64_t>& order) {
    // reverse Cuthill-McKee inside the leaf (degree tie-breaks within the piece)
    const int tag = next_tag++;
    for (int64_t v : idx) mk_set(mark, v, tag);
    std::vector<int64_t> seq;
    seq.reserve(idx.size());
    std::vector<char> seen_local;
    auto deg = [&](int64_t v) {
      int64_t d = 0;
      for (int64_t k = g.rp[v]; k < g.rp[v + 1]; ++k) d += mk_get(mark, g.ci[k]) == tag;
      return d;
    };
    std::vector<int64_t> q, nb;
    size_t done = 0;
    while (done < idx.size()) {
      int64_t root = -1, best = INT64_MAX;
      for (int64_t v : idx)
        if (mk_get(mark, v) == tag) {
          const int64_t d = deg(v);
          if (d < best) best = d, root = v;
        }
      // pseudo-peripheral refinement
      for (int it = 0; it < 2; ++it) {
        for (int64_t v : idx)
          if (mk_get(mark, v) == tag) level[v] = -1;
        bfs(g, mark, tag, root, level, order);
        root = order.back();
      }
      q.clear();
      q.push_back(root);
      mk_set(mark, root, -tag);
      for (size_t h = 0; h < q.size(); ++h) {
        const int64_t u = q[h];
        seq.push_back(u);
        nb.clear();
        for (int64_t k = g.rp[u]; k < g.rp[u + 1]; ++k) {
          const int64_t v = g.ci[k];
          if (mk_get(mark, v) == tag) {
            mk_set(mark, v, -tag);
            nb.push_back(v);
          }
        }
        std::sort(nb.begin(), nb.end(), [&](int64_t x, int64_t y) {
          const int64_t dx = g.rp[x + 1] - g.rp[x], dy = g.rp[y + 1] - g.rp[y];
          return dx < dy || (dx == dy && x < y);
        });
        for (int64_t v : nb) q.push_back(v);
      }
      done = seq.size();
    }
    std::reverse(seq.begin(), seq.end());
    for (int64_t v : idx) level[v] = -1;
    out.nodes.push_back(std::move(seq));
    out.is_sep.push_back(0);
  }

  void rec(std::vector<int64_t> idx, int depth, NdOut& out, std::vector<int64_t>& order) {
    if (static_cast<int64_t>(idx.size()) <= leaf) {
      emit_leaf(idx, out, order);
      return;
    }
    const int tag = next_tag++;
    for (int64_t v : idx) mk_set(mark, v, tag);
    int64_t root = idx[0];
    for (int it = 0; it < 2; ++it) {
      for (int64_t v : idx) level[v] = -1;
      bfs(g, mark, tag, root, level, order);
      root = order.back();
    }
    for (int64_t v : idx) level[v] = -1;
    bfs(g, mark, tag, root, level, order);
    if (order.size() < idx.size()) {  // disconnected: the reached component, then the rest
      std::vector<int64_t> a(order.begin(), order.end()), b;
      for (int64_t v : idx)
        if (level[v] < 0) b.push_back(v);
      for (int64_t v : idx) level[v] = -1;
      rec(std::move(a), depth, out, order);
      rec(std::move(b), depth, out, order);
      return;
    }
    // median level by vertex count
    std::vector<int64_t> lv;
    lv.reserve(idx.size());
    for (int64_t v : idx) lv.push_back(level[v]);
    std::vector<int64_t> srt = lv;
    std::nth_element(srt.begin(), srt.begin() + srt.size() / 2, srt.end());
    int64_t med = srt[srt.size() / 2];
    static const double win = [] {
      const char* v = std::getenv("ZOLO_ND_WINDOW");
      return v ? std::atof(v) : 0.0;
    }();
    if (win > 0.0) {
      // smallest level set whose two sides both hold at least (0.5 - win) of the piece
      std::vector<int64_t> cnt;
      for (int64_t l : lv) {
        if (l >= static_cast<int64_t>(cnt.size())) cnt.resize(l + 1, 0);
        ++cnt[l];
      }
      const double tot = static_cast<double>(idx.size());
      int64_t below = 0, best = -1;
      for (int64_t l = 0; l < static_cast<int64_t>(cnt.size()); ++l) {
        const double fa = below / tot, fb = (tot - below - cnt[l]) / tot;
        if (fa >= 0.5 - win && fb >= 0.5 - win && (best < 0 || cnt[l] < cnt[best])) best = l;
        below += cnt[l];
      }
      if (best >= 0) med = best;
    }
    std::vector<int64_t> a, b, s;
    for (size_t q = 0; q < idx.size(); ++q) {
      if (lv[q] < med)
        a.push_back(idx[q]);
      else if (lv[q] > med)
        b.push_back(idx[q]);
      else
        s.push_back(idx[q]);
    }
    for (int64_t v : idx) level[v] = -1;
    if (a.empty() || b.empty()) {  // no progress (path-like piece): stop dissecting
      emit_leaf(idx, out, order);
      return;
    }
    if (depth < PAR_DEPTH && static_cast<int64_t>(a.size()) > 4 * leaf) {
      NdOut oa;
      std::exception_ptr err;
      std::thread ta([&] {
        try {
          std::vector<int64_t> scratch;
          rec(std::move(a), depth + 1, oa, scratch);
        } catch (...) {
          err = std::current_exception();
        }
      });
      NdOut ob;
      try {
        rec(std::move(b), depth + 1, ob, order);
      } catch (...) {
        ta.join();
        throw;
      }
      ta.join();
      if (err) std::rethrow_exception(err);
      out.append(std::move(oa));
      out.append(std::move(ob));
    } else {
      rec(std::move(a), depth + 1, out, order);
      rec(std::move(b), depth + 1, out, order);
    }
    out.nodes.push_back(std::move(s));
    out.is_sep.push_back(1);
  }
};

// Separator rows ordered by the descendants they couple to. A separator's
// factor rows below a descendant subtree D are the separator vertices adjacent
// to D, so sorting them by the (already final) position of their earliest
// descendant neighbour makes each subtree's coupling rows contiguous: fewer,
// denser 32x32 tiles in L(separator, D) and U(D, separator). Nodes are in
// post-order, so every earlier neighbour of a separator vertex is a descendant.
// mode 1: earliest neighbour; 2: latest; 3: mean.
void order_separators(const Graph& g, const std::vector<int>& is_sep, std::vector<std::vector<int64_t>>& nodes,
                      int mode) {
  std::vector<int64_t> ord(g.n, -1);
  int64_t next = 0;
  std::vector<std::pair<double, int64_t>> keyed;
  for (size_t t = 0; t < nodes.size(); ++t) {
    auto& nd = nodes[t];
    if (is_sep[t] && nd.size() > 1) {
      keyed.clear();
      for (size_t q = 0; q < nd.size(); ++q) {
        const int64_t v = nd[q];
        double key = 0.0;
        int64_t cnt = 0, lo = INT64_MAX, hi = -1;
        for (int64_t k = g.rp[v]; k < g.rp[v + 1]; ++k) {
          const int64_t o = ord[g.ci[k]];
          if (o < 0) continue;
          lo = std::min(lo, o);
          hi = std::max(hi, o);
          key += static_cast<double>(o);
          ++cnt;
        }
        if (!cnt)
          key = 1e300;
        else if (mode == 1)
          key = static_cast<double>(lo);
        else if (mode == 2)
          key = static_cast<double>(hi);
        else
          key /= static_cast<double>(cnt);
        keyed.emplace_back(key, static_cast<int64_t>(q));
      }
      std::stable_sort(keyed.begin(), keyed.end(),
                       [](const auto& x, const auto& y) { return x.first < y.first; });
      std::vector<int64_t> out(nd.size());
      for (size_t q = 0; q < nd.size(); ++q) out[q] = nd[keyed[q].second];
      nd.swap(out);
    }
    for (int64_t v : nd) ord[v] = next++;
  }
}

}  // namespace

void nd_order(int64_t n, const int64_t* rp, const int64_t* ci, int64_t leaf, std::vector<std::vector<int64_t>>& nodes) {
  Graph g{n, rp, ci};
  NdState st(g, leaf);
  std::vector<int64_t> all(n);
  std::iota(all.begin(), all.end(), 0);
  NdOut res;
  {
    std::vector<int64_t> scratch;
    st.rec(std::move(all), 0, res, scratch);
  }
  nodes = std::move(res.nodes);
  static const int sep_mode = [] {
    const char* v = std::getenv("ZOLO_SEP_ORDER");
    return v ? std::atoi(v) : 1;
  }();
  if (sep_mode) order_separators(g, res.is_sep, nodes, sep_mode);
  // The node just before a separator (in post-order) is the root of its last child subtree,
  // whose factor structure lies inside separator + struct(separator): the two can share a
  // tile without adding fill, so only nodes followed by a non-separator start a new tile.
  static const bool merge = [] {
    const char* v = std::getenv("ZOLO_ND_MERGE");
    return v ? std::atoi(v) != 0 : true;
  }();
  if (merge && nodes.size() > 1) {
    std::vector<std::vector<int64_t>> out;
    std::vector<int64_t> cur;
    for (size_t t = 0; t < nodes.size(); ++t) {
      cur.insert(cur.end(), nodes[t].begin(), nodes[t].end());
      if (t + 1 == nodes.size() || !res.is_sep[t + 1]) {
        out.push_back(std::move(cur));
        cur.clear();
      }
    }
    nodes.swap(out);
  }
}

void block_symbolic(int64_t n, const int64_t* rp, const int64_t* ci, const std::vector<std::vector<int64_t>>& nodes,
                    int tile, BlockStructure& bs) {
  // padded positions: each node occupies a whole number of tiles
  bs.pos.assign(n, -1);
  std::vector<int64_t> inv;
  for (const auto& nd : nodes) {
    for (int64_t v : nd) {
      bs.pos[v] = static_cast<int64_t>(inv.size());
      inv.push_back(v);
    }
    while (inv.size() % tile) inv.push_back(-1);
  }
  bs.npad = static_cast<int64_t>(inv.size());
  bs.inv = std::move(inv);
  const int64_t nb = bs.npad / tile;
  bs.nb = nb;
  // block graph (upper part: neighbours with a larger block index)
  // (block rows are independent: host threads over ranges of blocks, each with its own stamp array,
  // so a dense-block pencil's millions of entries collapse to the few distinct neighbours at once)
  std::vector<std::vector<int64_t>> up(nb);
  {
    const int nt = static_cast<int>(std::min<int64_t>(std::min(16u, std::max(1u, std::thread::hardware_concurrency())),
                                                      std::max<int64_t>(1, nb / 64)));
    auto blocks = [&](int64_t lo, int64_t hi) {
      std::vector<int64_t> stamp(nb, -1);
      for (int64_t bv = lo; bv < hi; ++bv) {
        for (int t = 0; t < tile; ++t) {
          const int64_t v = bs.inv[bv * tile + t];
          if (v < 0) continue;
          for (int64_t k = rp[v]; k < rp[v + 1]; ++k) {
            const int64_t bw = bs.pos[ci[k]] / tile;
            if (bw > bv && stamp[bw] != bv) {
              stamp[bw] = bv;
              up[bv].push_back(bw);
            }
          }
        }
        std::sort(up[bv].begin(), up[bv].end());
      }
    };
    if (nt < 2) {
      blocks(0, nb);
    } else {
      std::vector<std::thread> pool;
      for (int q = 0; q < nt; ++q) pool.emplace_back(blocks, nb * q / nt, nb * (q + 1) / nt);
      for (auto& th : pool) th.join();
    }
  }
  // symbolic elimination through the elimination tree
  std::vector<int64_t> parent(nb, -1);
  std::vector<std::vector<int64_t>> children(nb);
  std::vector<std::vector<int64_t>> st(nb);
  std::vector<int64_t> merged;
  for (int64_t k = 0; k < nb; ++k) {
    merged = up[k];
    for (int64_t c : children[k]) {
      for (int64_t x : st[c])
        if (x != k) merged.push_back(x);
      std::vector<int64_t>().swap(st[c]);  // child structure no longer needed
    }
    std::sort(merged.begin(), merged.end());
    merged.erase(std::unique(merged.begin(), merged.end()), merged.end());
    st[k] = merged;
    if (!merged.empty()) {
      parent[k] = merged.front();
      children[merged.front()].push_back(k);
    }
    bs.col_ptr.push_back(static_cast<int64_t>(bs.col_idx.size()));
    for (int64_t i : merged) bs.col_idx.push_back(i);
  }
  bs.col_ptr.push_back(static_cast<int64_t>(bs.col_idx.size()));
  bs.parent = parent;
  // tile ids: one per off-diagonal structural pair (i > k), numbered row-major
  // (by i, then k) so a forward sweep reads a block row's L tiles contiguously
  std::vector<int64_t> cnt(nb + 1, 0);
  for (int64_t e = 0; e < static_cast<int64_t>(bs.col_idx.size()); ++e) ++cnt[bs.col_idx[e] + 1];
  bs.row_ptr.assign(nb + 1, 0);
  for (int64_t i = 0; i < nb; ++i) bs.row_ptr[i + 1] = bs.row_ptr[i] + cnt[i + 1];
  bs.row_idx.assign(bs.col_idx.size(), 0);
  bs.col_tile.assign(bs.col_idx.size(), 0);
  std::vector<int64_t> fill(bs.row_ptr.begin(), bs.row_ptr.end() - 1);
  for (int64_t k = 0; k < nb; ++k)
    for (int64_t e = bs.col_ptr[k]; e < bs.col_ptr[k + 1]; ++e) {
      const int64_t i = bs.col_idx[e];
      const int64_t slot = fill[i]++;
      bs.row_idx[slot] = k;   // rows' entries come out sorted by k (k ascending)
      bs.col_tile[e] = slot;  // the tile id is the row-major slot
    }
  bs.ntiles = static_cast<int64_t>(bs.col_idx.size());
  // critical path of the dependency DAG (forward sweep)
  std::vector<int64_t> depth(nb, 0);
  int64_t cp = 0;
  for (int64_t i = 0; i < nb; ++i) {
    int64_t d = 0;
    for (int64_t e = bs.row_ptr[i]; e < bs.row_ptr[i + 1]; ++e) d = std::max(d, depth[bs.row_idx[e]]);
    depth[i] = d + 1;
    cp = std::max(cp, depth[i]);
  }
  bs.critical_path = cp;
}

// Left-looking plan: block column y (and block row y of U) is completed at the level of y. The
// contributions of tile (x, y), x > y, are the k in row(x) ∩ row(y) (both sorted by k: one merge,
// no searches), those of D(y) the k in row(y); every such k is a descendant of y in the block
// elimination tree, so its panels are final at a lower level. A target collects ALL its
// contributions in ascending k (the fixed summation order) and is written once. Block columns are
// independent: all host threads count (pass 1), a prefix sum in level / column order fixes every
// column's place (the plan does not depend on the thread count), pass 2 writes the packed arrays.
void factor_plan(const BlockStructure& bs, FactorPlan& plan) {
  const int64_t nb = bs.nb;
  if (bs.ntiles >= (int64_t(1) << 30)) throw std::runtime_error("factor_plan: too many tiles");
  // level = height in the block elimination tree (parent = first structural row below)
  std::vector<int> level(nb, 0);
  int nlev = 0;
  for (int64_t k = 0; k < nb; ++k) {
    const int64_t p = bs.col_ptr[k + 1] > bs.col_ptr[k] ? bs.col_idx[bs.col_ptr[k]] : -1;
    if (p >= 0) level[p] = std::max(level[p], level[k] + 1);
    nlev = std::max(nlev, level[k] + 1);
  }
  plan = FactorPlan();
  // columns and panel tiles by level
  std::vector<std::vector<int>> by(nlev);
  for (int64_t k = 0; k < nb; ++k) by[level[k]].push_back(static_cast<int>(k));
  plan.cols.reserve(nb);
  plan.pan.reserve(4 * bs.ntiles);
  plan.lvl_ptr.push_back(0);
  plan.pan_ptr.push_back(0);
  for (int l = 0; l < nlev; ++l) {
    for (int k : by[l]) {
      plan.cols.push_back(k);
      for (int64_t e = bs.col_ptr[k]; e < bs.col_ptr[k + 1]; ++e) {
        const int id = static_cast<int>(bs.col_tile[e]);
        plan.pan.insert(plan.pan.end(), {k, 2 * id, k, 2 * id + 1});
      }
    }
    plan.lvl_ptr.push_back(static_cast<int>(plan.cols.size()));
    plan.pan_ptr.push_back(static_cast<int>(plan.pan.size() / 2));
  }
  // targets of block column y: emit(kind, tile id, m) with the m contributions (L tile id, U tile
  // id) in buf[0, m); the U target of a tile has the same k with the ids swapped
  struct Con {
    int la, ub;
  };
  auto column_targets = [&](int64_t y, std::vector<Con>& buf, auto&& emit) {
    const int64_t y0 = bs.row_ptr[y], y1 = bs.row_ptr[y + 1];
    const int ny = static_cast<int>(y1 - y0);
    buf.resize(std::max<size_t>(buf.size(), ny));
    if (ny) {  // D(y) -= L(y, k) U(k, y)
      for (int q = 0; q < ny; ++q) buf[q] = {static_cast<int>(y0 + q), static_cast<int>(y0 + q)};
      emit(0, static_cast<int>(y), ny);
    }
    if (!ny) return;
    for (int64_t e = bs.col_ptr[y]; e < bs.col_ptr[y + 1]; ++e) {
      const int64_t x = bs.col_idx[e];
      // k in row(x) ∩ row(y): L(x, y) -= L(x, k) U(k, y), U(y, x) -= L(y, k) U(k, x)
      int64_t a = bs.row_ptr[x], b = y0;
      const int64_t a1 = bs.row_ptr[x + 1];
      int m = 0;
      while (a < a1 && b < y1) {
        const int64_t ka = bs.row_idx[a], kb = bs.row_idx[b];
        if (ka == kb)
          buf[m++] = {static_cast<int>(a), static_cast<int>(b)}, ++a, ++b;
        else if (ka < kb)
          ++a;
        else
          ++b;
      }
      if (m) emit(1, static_cast<int>(bs.col_tile[e]), m);
    }
  };
  // Long lists are split: a target with more than SPLIT_MIN contributions becomes up to MAXP part
  // records (kind 3) that each write their partial product into a scratch slot of the level, and
  // one combine entry subtracts the parts from the tile in part order (fixed summation order). The
  // top of the tree has few targets with lists of hundreds of products: splitting fills the GPU
  // there and shortens each level's critical path.
  auto part_size = [](int m) {
    constexpr int SPLIT_MIN = 48, PART = 32, MAXP = 16;
    return m <= SPLIT_MIN ? std::max(m, 1) : std::max(PART, (m + MAXP - 1) / MAXP);
  };
  struct Cnt {
    int64_t nt = 0, nc = 0, ns = 0, nm = 0;  // records, contributions, scratch slots, combine entries
  };
  std::vector<Cnt> cnt(nb);
  const int nthr = static_cast<int>(std::max(1u, std::min(16u, std::thread::hardware_concurrency())));
  auto run = [&](auto&& body) {
    std::atomic<int64_t> next{0};
    auto worker = [&] {
      std::vector<Con> buf;
      // heavy columns (the separators at the end) first
      for (int64_t i = next++; i < nb; i = next++) body(nb - 1 - i, buf);
    };
    std::vector<std::thread> pool;
    for (int q = 1; q < nthr; ++q) pool.emplace_back(worker);
    worker();
    for (auto& t : pool) t.join();
  };
  run([&](int64_t y, std::vector<Con>& buf) {
    Cnt c;
    column_targets(y, buf, [&](int kind, int, int m) {
      const int both = kind ? 2 : 1;
      const int sz = part_size(m);
      const int np = (m + sz - 1) / sz;
      c.nt += both * np;
      c.nc += both * m;
      if (np > 1) c.ns += both * np, c.nm += both;
    });
    cnt[y] = c;
  });
  // offsets in level order, columns in plan.cols order; scratch slots restart at every level
  plan.tgt_ptr.assign(1, 0);
  plan.cmb_ptr.assign(1, 0);
  int64_t ntgt = 0, ncon = 0, ncmb = 0;
  plan.scratch_slots = 0;
  for (int l = 0; l < nlev; ++l) {
    int64_t slots = 0;
    for (int y : by[l]) {
      const Cnt c = cnt[y];
      cnt[y] = {ntgt, ncon, slots, ncmb};
      ntgt += c.nt;
      ncon += c.nc;
      slots += c.ns;
      ncmb += c.nm;
    }
    plan.scratch_slots = std::max(plan.scratch_slots, slots);
    plan.tgt_ptr.push_back(static_cast<int>(ntgt));
    plan.cmb_ptr.push_back(static_cast<int>(ncmb));
  }
  if (ncon >= (int64_t(1) << 31)) throw std::runtime_error("factor_plan: too many updates");
  if (plan.scratch_slots >= (int64_t(1) << 30)) throw std::runtime_error("factor_plan: too many partial products");
  plan.tgt.resize(2 * ntgt + 2);
  plan.con.resize(2 * ncon);
  plan.cmb.resize(3 * ncmb);
  plan.tgt[2 * ntgt] = 0;
  plan.tgt[2 * ntgt + 1] = static_cast<int>(ncon);  // sentinel: the last target's end
  run([&](int64_t y, std::vector<Con>& buf) {
    int64_t t = cnt[y].nt, c = cnt[y].nc, sl = cnt[y].ns, cm = cnt[y].nm;
    // one target (kind, tile id) with the m contributions of buf, ids swapped for the U target
    auto write = [&](int kind, int id, int m, bool swap) {
      const int sz = part_size(m);
      const int np = (m + sz - 1) / sz;
      if (np > 1) {
        plan.cmb[3 * cm] = static_cast<int>(static_cast<unsigned>(kind) << 30 | static_cast<unsigned>(id));
        plan.cmb[3 * cm + 1] = static_cast<int>(sl);
        plan.cmb[3 * cm + 2] = np;
        ++cm;
      }
      for (int p = 0; p < np; ++p) {
        plan.tgt[2 * t] = np > 1 ? static_cast<int>(3u << 30 | static_cast<unsigned>(sl++))
                                 : static_cast<int>(static_cast<unsigned>(kind) << 30 | static_cast<unsigned>(id));
        plan.tgt[2 * t + 1] = static_cast<int>(c);
        ++t;
        for (int i = p * sz; i < std::min(m, (p + 1) * sz); ++i, ++c) {
          plan.con[2 * c] = swap ? buf[i].ub : buf[i].la;
          plan.con[2 * c + 1] = swap ? buf[i].la : buf[i].ub;
        }
      }
    };
    column_targets(y, buf, [&](int kind, int id, int m) {
      write(kind, id, m, false);
      if (kind) write(2, id, m, true);  // the U target: same k, ids swapped
    });
  });
  plan.contributions = ncon;
}

int trailing_dense_start(const BlockStructure& bs, int kmax) {
  const int64_t nb = bs.nb;
  auto has = [&](int64_t i, int64_t k) {
    return std::binary_search(bs.row_idx.begin() + bs.row_ptr[i], bs.row_idx.begin() + bs.row_ptr[i + 1], k);
  };
  // grow S = [s, nb) while every row of S holds every earlier row of S
  int64_t s = nb;
  while (s > 0 && nb - (s - 1) <= kmax) {
    bool dense = true;
    for (int64_t i = s; i < nb && dense; ++i) dense = has(i, s - 1);
    if (!dense) break;
    --s;
  }
  return static_cast<int>(s);
}

// Partial slots along the claim order (see DagTask). Chunk tasks arrive with distinct slots
// `out`, consecutive per row in chunk order. A row's chunks are chained into the K_i slots of a
// unit taken at its first chunk -- a K_i-slot unit freed REUSE_GAP records after the row task that
// last read it, else a new one -- so the partial sums need one unit per row in flight
// instead of one 32-row block per chunk task for the whole sweep (config 3: ~1900 slots instead
// of ~11600), while up to DAG_PCHAINS chunks of a row still run in parallel. Returns the slot
// count.
int accumulate_slots(std::vector<DagTask>& tasks, int64_t nb) {
  constexpr int64_t REUSE_GAP = 64;  // records between a row task and the reuse of its unit
  constexpr int K = DAG_PCHAINS;
  struct Free {
    int base;
    int64_t free_at;  // claim position from which the unit may be taken
    int wait;         // the row task that last read it
    int use;          // uses so far
  };
  // freed units by size (a row with K_i chains takes a K_i-slot unit), oldest first
  std::vector<std::vector<Free>> pool(K + 1);
  std::vector<size_t> head(K + 1, 0);
  auto chains = [&](int nchunk) { return std::max(std::min(K, nchunk), (nchunk + 62) / 63); };
  std::vector<int> base_of(nb, -1), use_of(nb, 0), wait_of(nb, -1), first_out(nb, -1), seen(nb, 0), nch(nb, 0);
  std::vector<std::vector<int>> next_step(nb);  // per row, per chain
  for (const DagTask& t : tasks) {
    if (t.out >= 0 && (first_out[t.i] < 0 || t.out < first_out[t.i])) first_out[t.i] = t.out;
    if (t.out < 0) nch[t.i] = t.pc;
  }
  int nslots = 0;
  for (int64_t p = 0; p < static_cast<int64_t>(tasks.size()); ++p) {
    DagTask& t = tasks[p];
    if (t.out >= 0) {  // chunk c of row t.i
      const int c = t.out - first_out[t.i];
      const int ki = chains(nch[t.i]);
      if (static_cast<int>(pool.size()) <= ki) {
        pool.resize(ki + 1);
        head.resize(ki + 1, 0);
      }
      std::vector<int>& ns = next_step[t.i];
      if (ns.empty()) ns.assign(ki, 0);
      if (c / ki != ns[c % ki]++)
        throw std::logic_error("dag_schedule: chunks of a partial chain out of order");
      ++seen[t.i];
      if (base_of[t.i] < 0) {  // the row's first chunk in claim order takes a unit
        std::vector<Free>& pl = pool[ki];
        size_t& hd = head[ki];
        if (hd < pl.size() && pl[hd].free_at <= p) {
          base_of[t.i] = pl[hd].base;
          wait_of[t.i] = pl[hd].wait;
          use_of[t.i] = pl[hd].use + 1;
          ++hd;
        } else {
          base_of[t.i] = nslots;
          nslots += ki;
          wait_of[t.i] = -1;
          use_of[t.i] = 0;
        }
      }
      const int step = c / ki;
      if (step >= 64) throw std::runtime_error("dag_schedule: too many chunks per partial chain");
      t.out = base_of[t.i] + c % ki;
      t.pa = t.out;
      t.pc = step > 0 ? 1 : 0;  // the chain's partial so far (step - 1)
      t.wait = step > 0 ? -1 : wait_of[t.i];
      t.gen = use_of[t.i];
      t.aux = c | (ki << 16);
    } else if (t.pc > 0) {  // row task: adds its K_i partials, then frees the unit
      if (base_of[t.i] < 0 || seen[t.i] != t.pc) throw std::logic_error("dag_schedule: row task before its chunks");
      t.aux = t.pc;
      t.pa = base_of[t.i];
      t.pc = chains(t.pc);
      t.gen = use_of[t.i];
      if (use_of[t.i] + 1 < DAG_GENS / 64) pool[t.pc].push_back(Free{base_of[t.i], p + REUSE_GAP, t.i, use_of[t.i]});
    }
  }
  return std::max(nslots, 1);
}

int dag_schedule(int64_t nb, const std::vector<int64_t>& ptr, const std::vector<int64_t>& idx, bool fwd, int chunk,
                 int near, int order, std::vector<DagTask>& tasks) {
  if (chunk < 1 || near < 0) throw std::invalid_argument("dag_schedule: chunk >= 1, near >= 0");
  // processing position of block row j in the sweep (forward: j, backward: nb-1-j)
  auto position = [&](int64_t j) { return fwd ? j : nb - 1 - j; };
  std::vector<std::vector<DagTask>> after(nb);  // chunks claimed right after row task at a position
  std::vector<DagTask> rows(nb);
  int slots = 0;
  for (int64_t s = 0; s < nb; ++s) {
    const int64_t i = fwd ? s : nb - 1 - s;
    const int64_t e0 = ptr[i];
    const int nd = static_cast<int>(ptr[i + 1] - e0);
    // dependency at processing index q (ascending completion order)
    auto dep = [&](int q) { return fwd ? idx[e0 + q] : idx[e0 + nd - 1 - q]; };
    DagTask row{static_cast<int>(i), 0, nd, slots, 0, -1};
    if (nd > near + chunk) {
      const int far = nd - near;
      const int nchunk = (far + chunk - 1) / chunk;
      for (int c = 0, q0 = 0; c < nchunk; ++c) {
        const int q1 = static_cast<int>((static_cast<int64_t>(far) * (c + 1)) / nchunk);  // balanced cut
        const int64_t last = position(dep(q1 - 1));
        after[last].push_back(DagTask{static_cast<int>(i), q0, q1, 0, 0, slots++});
        q0 = q1;
      }
      row.qa = far;
      row.pc = nchunk;
    }
    rows[s] = row;
  }
  std::vector<DagTask> seq;  // positional topological order
  for (int64_t s = 0; s < nb; ++s) {
    seq.push_back(rows[s]);
    for (const DagTask& t : after[s]) seq.push_back(t);
  }
  tasks.clear();
  if (order == 0) {
    tasks = std::move(seq);
    return accumulate_slots(tasks, nb);
  }
  // list-scheduling priority over the task graph, with cost = tile products
  // (+1 for the diagonal pre-transform and the store/flag latency)
  const int64_t nt = static_cast<int64_t>(seq.size());
  std::vector<int64_t> row_task(nb, -1), slot_task(slots, -1);
  for (int64_t t = 0; t < nt; ++t) (seq[t].out >= 0 ? slot_task[seq[t].out] : row_task[seq[t].i]) = t;
  std::vector<double> cost(nt);
  std::vector<std::vector<int64_t>> deps(nt);
  for (int64_t t = 0; t < nt; ++t) {
    const DagTask& k = seq[t];
    const int64_t e0 = ptr[k.i];
    const int nd = static_cast<int>(ptr[k.i + 1] - e0);
    for (int q = k.qa; q < k.qb; ++q) deps[t].push_back(row_task[fwd ? idx[e0 + q] : idx[e0 + nd - 1 - q]]);
    for (int p = k.pa; p < k.pa + k.pc; ++p) deps[t].push_back(slot_task[p]);
    // a row's chunks accumulate in DAG_PCHAINS chains (accumulate_slots): chunk c waits on c - K_i
    bool later_chunk = false;
    if (k.out >= 0) {
      const DagTask& row = seq[row_task[k.i]];
      const int ki = std::max(std::min(DAG_PCHAINS, row.pc), (row.pc + 62) / 63);  // accumulate_slots chains()
      if (k.out - row.pa >= ki) {
        deps[t].push_back(slot_task[k.out - ki]);
        later_chunk = true;
      }
    }
    cost[t] = (k.qb - k.qa) + 0.25 * k.pc + (later_chunk ? 0.25 : 0.0) + 2.0;
  }
  std::vector<double> key(nt, 0.0);
  // earliest start time (EST) and longest path to the end (bottom level, BL); key = EST - lambda * BL
  // is topological for every lambda >= 0: lambda = 0 pure EST (order 1), order 2 pure BL,
  // order >= 3 a blend with lambda = (order - 2) / 8
  std::vector<double> est(nt, 0.0), bl(cost);
  for (int64_t t = 0; t < nt; ++t)
    for (int64_t d : deps[t]) est[t] = std::max(est[t], est[d] + cost[d]);
  for (int64_t t = nt - 1; t >= 0; --t)
    for (int64_t d : deps[t]) bl[d] = std::max(bl[d], cost[d] + bl[t]);
  const double lambda = order >= 3 ? (order - 2) / 8.0 : 0.0;
  for (int64_t t = 0; t < nt; ++t) key[t] = order == 2 ? -bl[t] : est[t] - lambda * bl[t];
  std::vector<int64_t> perm(nt);
  for (int64_t t = 0; t < nt; ++t) perm[t] = t;
  std::stable_sort(perm.begin(), perm.end(), [&](int64_t a, int64_t b) { return key[a] < key[b]; });
  for (int64_t t : perm) tasks.push_back(seq[t]);
  return accumulate_slots(tasks, nb);
}

}  // namespace zolo
