// Exact depth-first 0-1 branch-and-bound over the scheduling ILP (host code).
//
// Search semantics follow the reference solver (pkg/src/remsched/solver.py):
// incremental row-activity propagation (54-195), the admissible bound =
// per-group cheapest surviving implementation (197-208, 323-343) plus the
// capacity surrogate (211-320), the static branch order (346-376) or the
// most-tight rule (379-393), bound-probing dives (546-572), node / time /
// gap limits checked where the reference checks them (537-545, 598-609),
// and the same statuses.  Identical search => identical decisions, so the
// schedules it returns are bit-exact against the reference's; it just runs
// natively (the reference spends its time in these loops).
//
// Costs arrive scaled to integers (x lcm of the objective denominators),
// so every bound / objective comparison is exact integer arithmetic.
// Boundary: monet_bnb_* in include/monet_b200.h; no exception crosses it.
#include <algorithm>
#include <chrono>
#include <cstdint>
#include <cstring>
#include <new>
#include <vector>

#include "monet_b200.h"

namespace {

using i64 = long long;
using i128 = __int128;

struct Group {
  std::vector<int> var;
  std::vector<i128> cost;
};

struct Stage {
  i64 grad;
  std::vector<int> db;
  std::vector<i64> ws;
  std::vector<std::vector<int>> deps;  // storable indices, sorted by storable id
};

struct Event {
  int kind;  // 0 root 1 warm-start 2 incumbent 3 tick 4 final
  i64 nodes;
  i64 elapsed_ms;
  int has_inc, has_bound, has_gap;
  i128 inc, bound, gap_num, gap_den;
};

struct Problem {
  int n = 0, m = 0;
  std::vector<int> row_ptr, row_var;
  std::vector<i64> row_coef, row_ub, row_lb;
  std::vector<char> row_has_ub, row_has_lb;
  std::vector<i64> row_maxabs;
  std::vector<std::vector<std::pair<int, i64>>> watch;
  std::vector<int> fix_var, fix_val;
  std::vector<int> obj_var;
  std::vector<i128> obj_cost;
  std::vector<Group> fwd, bwd, re;
  std::vector<int> re_rvar;
  // surrogate
  int has_surr = 0;
  i64 cap_base = 0;
  std::vector<Stage> stages;
  std::vector<i64> st_size, st_recost;
  std::vector<std::vector<int>> st_rcol;  // per storable (sorted by id): R var of stage 1..T
  // state
  std::vector<signed char> val;
  std::vector<int> trail;
  std::vector<i64> minact, maxact;
  std::vector<char> queued;
  std::vector<Event> events;
  // result
  std::vector<signed char> best_assign;
};

struct Prop {
  Problem& P;
  explicit Prop(Problem& p) : P(p) {}

  void reset() {
    P.val.assign(P.n, -1);
    P.trail.clear();
    P.minact.assign(P.m, 0);
    P.maxact.assign(P.m, 0);
    P.queued.assign(P.m, 0);
    for (int r = 0; r < P.m; ++r)
      for (int e = P.row_ptr[r]; e < P.row_ptr[r + 1]; ++e) {
        const i64 c = P.row_coef[e];
        if (c < 0)
          P.minact[r] += c;
        else
          P.maxact[r] += c;
      }
  }

  bool fix(int v, int b, std::vector<int>& queue) {
    const int cur = P.val[v];
    if (cur >= 0) return cur == b;
    P.val[v] = (signed char)b;
    P.trail.push_back(v);
    bool ok = true;  // keep updating every row on conflict: undo reverses the whole list
    for (const auto& w : P.watch[v]) {
      const int r = w.first;
      const i64 c = w.second;
      if (b) {
        if (c > 0)
          P.minact[r] += c;
        else
          P.maxact[r] += c;
      } else {
        if (c < 0)
          P.minact[r] -= c;
        else
          P.maxact[r] -= c;
      }
      if (P.row_has_ub[r] && P.minact[r] > P.row_ub[r]) ok = false;
      if (P.row_has_lb[r] && P.maxact[r] < P.row_lb[r]) ok = false;
      if (ok && !P.queued[r]) {
        P.queued[r] = 1;
        queue.push_back(r);
      }
    }
    return ok;
  }

  bool propagate(std::vector<int>& queue) {
    for (size_t head = 0; head < queue.size(); ++head) {
      const int r = queue[head];
      P.queued[r] = 0;
      const i64 mab = P.row_maxabs[r];
      bool use_ub = P.row_has_ub[r] && !(P.row_ub[r] - P.minact[r] >= mab);
      bool use_lb = P.row_has_lb[r] && !(P.maxact[r] - P.row_lb[r] >= mab);
      if (!use_ub && !use_lb) continue;
      const i64 ub = P.row_ub[r], lb = P.row_lb[r];
      for (int e = P.row_ptr[r]; e < P.row_ptr[r + 1]; ++e) {
        const int v = P.row_var[e];
        if (P.val[v] != -1) continue;
        const i64 c = P.row_coef[e];
        int forced = -1;
        if (use_ub) {
          if (c > 0 && P.minact[r] + c > ub)
            forced = 0;
          else if (c < 0 && P.minact[r] - c > ub)
            forced = 1;
        }
        if (forced == -1 && use_lb) {
          if (c > 0 && P.maxact[r] - c < lb)
            forced = 1;
          else if (c < 0 && P.maxact[r] + c < lb)
            forced = 0;
        }
        if (forced != -1 && !fix(v, forced, queue)) {
          for (int q : queue) P.queued[q] = 0;
          queue.clear();
          return false;
        }
      }
    }
    queue.clear();
    return true;
  }

  bool assign(int v, int b) {
    std::vector<int> queue;
    if (!fix(v, b, queue)) {
      for (int q : queue) P.queued[q] = 0;
      return false;
    }
    return propagate(queue);
  }

  void undo_to(size_t mark) {
    while (P.trail.size() > mark) {
      const int v = P.trail.back();
      P.trail.pop_back();
      const int b = P.val[v];
      P.val[v] = -1;
      for (const auto& w : P.watch[v]) {
        const int r = w.first;
        const i64 c = w.second;
        if (b) {
          if (c > 0)
            P.minact[r] -= c;
          else
            P.maxact[r] -= c;
        } else {
          if (c < 0)
            P.minact[r] += c;
          else
            P.maxact[r] += c;
        }
      }
    }
  }
};

i128 group_min(const Problem& P, const Group& g) {
  bool have = false;
  i128 best = 0;
  for (size_t i = 0; i < g.var.size(); ++i) {
    const int b = P.val[g.var[i]];
    if (b == 1) return g.cost[i];
    if (b == 0) continue;
    if (!have || g.cost[i] < best) {
      best = g.cost[i];
      have = true;
    }
  }
  return have ? best : 0;
}

// capacity surrogate (solver.py:251-320); returns false when infeasible
bool surrogate(const Problem& P, i64& extra) {
  extra = 0;
  const int T = (int)P.stages.size();
  if (T == 0) return true;
  const int NS = (int)P.st_size.size();
  std::vector<int> need_last(NS, 0);
  std::vector<char> has_alive(T + 1, 0);
  std::vector<std::vector<int>> alive(T + 1);  // variant indices alive per stage
  std::vector<char> inter;
  for (int ti = 0; ti < T; ++ti) {
    const Stage& S = P.stages[ti];
    std::vector<int>& al = alive[ti + 1];
    for (size_t l = 0; l < S.db.size(); ++l)
      if (P.val[S.db[l]] != 0) al.push_back((int)l);
    if (al.empty()) continue;
    has_alive[ti + 1] = 1;
    // intersection of the alive variants' deps
    inter.assign(NS, 0);
    for (int u : S.deps[al[0]]) inter[u] = 1;
    for (size_t a = 1; a < al.size(); ++a) {
      std::vector<char> mine(NS, 0);
      for (int u : S.deps[al[a]]) mine[u] = 1;
      for (int u = 0; u < NS; ++u) inter[u] = inter[u] && mine[u];
    }
    for (int u = 0; u < NS; ++u)
      if (inter[u] && need_last[u] < ti + 1) need_last[u] = ti + 1;
  }
  struct Item {
    int u;
    i64 sz, c;
    int tu;
  };
  std::vector<Item> mandatory, open;
  for (int u = 0; u < NS; ++u) {  // storables are indexed in id order == sorted(need_last)
    const int tu = need_last[u];
    if (!tu) continue;
    bool fixed_on = false, all_off = true;
    for (int t = 0; t < tu; ++t) {
      const int b = P.val[P.st_rcol[u][t]];
      if (b == 1) {
        fixed_on = true;
        break;
      }
      if (b != 0) all_off = false;
    }
    if (fixed_on) continue;
    if (all_off)
      mandatory.push_back({u, P.st_size[u], 0, tu});
    else if (P.st_size[u] > 0)
      open.push_back({u, P.st_size[u], P.st_recost[u], tu});
  }
  std::vector<char> charged(NS, 0);
  for (int t = 1; t <= T; ++t) {
    if (!has_alive[t]) continue;
    std::fill(charged.begin(), charged.end(), 0);
    for (const Item& it : mandatory)
      if (it.tu >= t) charged[it.u] = 1;
    for (const Item& it : open)
      if (it.tu >= t) charged[it.u] = 1;
    const Stage& S = P.stages[t - 1];
    bool first = true;
    i64 mn = 0;
    for (int l : alive[t]) {
      i64 v = S.ws[l];
      for (int u : S.deps[l])
        if (!charged[u]) v += P.st_size[u];
      if (first || v < mn) {
        mn = v;
        first = false;
      }
    }
    const i64 cap = P.cap_base - S.grad - mn;
    i64 avail = cap;
    for (const Item& it : mandatory)
      if (it.tu >= t) avail -= it.sz;
    i64 total = 0;
    int nitems = 0;
    i64 bc = 0, bsz = 1;
    for (const Item& it : open) {
      if (it.tu < t) continue;
      total += it.sz;
      if (nitems == 0) {
        bc = it.c;
        bsz = it.sz;
      } else if ((i128)it.c * bsz < (i128)bc * it.sz) {
        bc = it.c;
        bsz = it.sz;
      }
      ++nitems;
    }
    if (avail < 0) return false;
    if (total <= avail || nitems == 0) continue;
    const i128 num = (i128)(total - avail) * bc;
    const i64 cand = (i64)((num + bsz - 1) / bsz);  // non-negative: ceiling division
    if (cand > extra) extra = cand;
  }
  return true;
}

struct Bound {
  bool ok;
  i128 v;
};

Bound bound(const Problem& P, i128 scale) {
  i128 total = 0;
  for (const Group& g : P.fwd) total += group_min(P, g);
  for (const Group& g : P.bwd) total += group_min(P, g);
  for (size_t i = 0; i < P.re.size(); ++i)
    if (P.val[P.re_rvar[i]] == 1 && !P.re[i].var.empty()) total += group_min(P, P.re[i]);
  if (P.has_surr) {
    i64 extra;
    if (!surrogate(P, extra)) return {false, 0};
    total += (i128)extra * scale;
  }
  return {true, total};
}

int pick_most_tight(const Problem& P) {
  int best_v = -1, best_score = -1;
  for (int v = 0; v < P.n; ++v) {
    if (P.val[v] != -1) continue;
    int score = 0;
    for (const auto& w : P.watch[v])
      if (P.row_has_ub[w.first] && P.minact[w.first] == P.row_ub[w.first]) ++score;
    if (score > best_score) {
      best_score = score;
      best_v = v;
    }
  }
  return best_v;
}

i128 rd128(const int64_t* hi_lo, int i) { return ((i128)hi_lo[2 * i] << 64) | (i128)(uint64_t)hi_lo[2 * i + 1]; }
void wr128(int64_t* out, int i, i128 v) {
  out[2 * i] = (int64_t)(v >> 64);
  out[2 * i + 1] = (int64_t)(uint64_t)v;
}

}  // namespace

extern "C" {

// Build a problem.  128-bit costs are passed as (hi, lo) int64 pairs.
void* monet_bnb_create(int n_vars, int n_rows, const int* row_ptr, const int* row_var, const int64_t* row_coef,
                       const int64_t* row_rhs, const int* row_is_eq, int n_fix, const int* fix_var, const int* fix_val,
                       int n_obj, const int* obj_var, const int64_t* obj_cost128, int n_fwd, int n_bwd, int n_re,
                       const int* grp_ptr, const int* grp_var, const int64_t* grp_cost128, const int* re_rvar) {
  Problem* P = new (std::nothrow) Problem();
  if (!P) return nullptr;
  P->n = n_vars;
  P->m = n_rows;
  P->row_ptr.assign(row_ptr, row_ptr + n_rows + 1);
  const int nnz = row_ptr[n_rows];
  P->row_var.assign(row_var, row_var + nnz);
  P->row_coef.assign(row_coef, row_coef + nnz);
  P->row_ub.assign(row_rhs, row_rhs + n_rows);
  P->row_lb.assign(row_rhs, row_rhs + n_rows);
  P->row_has_ub.assign(n_rows, 1);
  P->row_has_lb.resize(n_rows);
  P->row_maxabs.assign(n_rows, 0);
  P->watch.assign(n_vars, {});
  for (int r = 0; r < n_rows; ++r) {
    P->row_has_lb[r] = row_is_eq[r] ? 1 : 0;
    for (int e = row_ptr[r]; e < row_ptr[r + 1]; ++e) {
      P->watch[row_var[e]].push_back({r, row_coef[e]});
      const i64 a = row_coef[e] < 0 ? -row_coef[e] : row_coef[e];
      P->row_maxabs[r] = std::max(P->row_maxabs[r], a);
    }
  }
  P->fix_var.assign(fix_var, fix_var + n_fix);
  P->fix_val.assign(fix_val, fix_val + n_fix);
  P->obj_var.assign(obj_var, obj_var + n_obj);
  for (int i = 0; i < n_obj; ++i) P->obj_cost.push_back(rd128(obj_cost128, i));
  auto read_group = [&](int g) {
    Group G;
    for (int e = grp_ptr[g]; e < grp_ptr[g + 1]; ++e) {
      G.var.push_back(grp_var[e]);
      G.cost.push_back(rd128(grp_cost128, e));
    }
    return G;
  };
  int g = 0;
  for (int i = 0; i < n_fwd; ++i) P->fwd.push_back(read_group(g++));
  for (int i = 0; i < n_bwd; ++i) P->bwd.push_back(read_group(g++));
  for (int i = 0; i < n_re; ++i) {
    P->re.push_back(read_group(g++));
    P->re_rvar.push_back(re_rvar[i]);
  }
  return P;
}

// Capacity surrogate data: per stage its grad-live bytes and backward variants
// (DeltaBwd var, workspace, dep storable indices); per storable (id order) its
// size, truncated cheapest forward cost, and R variable of stages 1..T.
int monet_bnb_set_surrogate(void* h, int64_t cap_base, int n_stages, const int64_t* grad, const int* var_ptr,
                            const int* var_db, const int64_t* var_ws, const int* dep_ptr, const int* dep_idx,
                            int n_storables, const int64_t* size, const int64_t* recost, const int* rcol) {
  Problem* P = static_cast<Problem*>(h);
  P->has_surr = 1;
  P->cap_base = cap_base;
  P->stages.clear();
  for (int t = 0; t < n_stages; ++t) {
    Stage S;
    S.grad = grad[t];
    for (int l = var_ptr[t]; l < var_ptr[t + 1]; ++l) {
      S.db.push_back(var_db[l]);
      S.ws.push_back(var_ws[l]);
      S.deps.emplace_back(dep_idx + dep_ptr[l], dep_idx + dep_ptr[l + 1]);
    }
    P->stages.push_back(std::move(S));
  }
  P->st_size.assign(size, size + n_storables);
  P->st_recost.assign(recost, recost + n_storables);
  P->st_rcol.assign(n_storables, {});
  for (int u = 0; u < n_storables; ++u) P->st_rcol[u].assign(rcol + (size_t)u * n_stages, rcol + (size_t)(u + 1) * n_stages);
  return 0;
}

void monet_bnb_destroy(void* h) { delete static_cast<Problem*>(h); }

// Fixpoint propagation from the model fixings plus a partial assignment.
// Writes every variable's value (-1 = free) to `out`; returns 1 if consistent.
int monet_bnb_propagate(void* h, int n_partial, const int* pvar, const int* pval, signed char* out) {
  Problem& P = *static_cast<Problem*>(h);
  Prop pr(P);
  pr.reset();
  std::vector<int> queue;
  for (size_t i = 0; i < P.fix_var.size(); ++i)
    if (!pr.fix(P.fix_var[i], P.fix_val[i], queue)) return 0;
  for (int i = 0; i < n_partial; ++i)
    if (!pr.fix(pvar[i], pval[i], queue)) return 0;
  if (!pr.propagate(queue)) return 0;
  std::memcpy(out, P.val.data(), P.n);
  return 1;
}

// Admissible bound under a partial assignment (scaled units, (hi, lo) pair);
// returns 0 when inconsistent.
int monet_bnb_lower_bound(void* h, int n_partial, const int* pvar, const int* pval, int64_t scale, int64_t* out128) {
  Problem& P = *static_cast<Problem*>(h);
  std::vector<signed char> tmp(P.n);
  if (!monet_bnb_propagate(h, n_partial, pvar, pval, tmp.data())) return 0;
  const Bound b = bound(P, scale);
  if (!b.ok) return 0;
  wr128(out128, 0, b.v);
  return 1;
}

// The search.  opts: [0] node_limit (-1 none) [1] telemetry_every [2] dive_bound
// [3] most_tight [4] gap_num [5] gap_den (den 0 = no gap target) [6] scale;
// time_limit_s < 0 = none.  incumbent: has_inc + its scaled objective + values.
// Returns the status: 0 optimal 1 feasible-gap 2 infeasible 3 timeout-no-incumbent.
int monet_bnb_solve(void* h, const int64_t* opts, double time_limit_s, const int* order, int n_order,
                    const signed char* pref, int has_inc, const int64_t* inc_obj128, const signed char* inc_vals,
                    int64_t* nodes_out, int64_t* res128 /* objective, bound, gap_num, gap_den */) {
  Problem& P = *static_cast<Problem*>(h);
  const i64 node_limit = opts[0], tel_every = opts[1];
  const bool dive_bound = opts[2] != 0, most_tight = opts[3] != 0;
  const i64 gap_num = opts[4], gap_den = opts[5];
  const i128 scale = opts[6];
  const auto t0 = std::chrono::steady_clock::now();
  auto elapsed = [&] { return std::chrono::duration<double>(std::chrono::steady_clock::now() - t0).count(); };
  P.events.clear();
  i64 nodes = 0;
  auto emit = [&](int kind, bool hi, i128 inc, bool hb, i128 bnd, bool hg, i128 gn, i128 gd) {
    P.events.push_back({kind, nodes, (i64)(elapsed() * 1000.0), hi, hb, hg, inc, bnd, gn, gd});
  };

  Prop pr(P);
  pr.reset();
  bool root_ok = true;
  {
    std::vector<int> queue;
    for (size_t i = 0; i < P.fix_var.size(); ++i)
      if (!pr.fix(P.fix_var[i], P.fix_val[i], queue)) {
        root_ok = false;
        break;
      }
    if (root_ok) root_ok = pr.propagate(queue);
  }
  if (!root_ok) {
    emit(4, false, 0, false, 0, false, 0, 0);
    *nodes_out = 0;
    return 2;
  }

  bool have_best = false;
  i128 best = 0;
  auto gap_of = [&](bool hb, i128 bnd, i128& gn, i128& gd) -> bool {  // false = no gap
    if (!have_best || !hb) return false;
    if (bnd >= best) {
      gn = 0;
      gd = 1;
      return true;
    }
    if (best == 0) return false;
    gn = best - bnd;
    gd = best;
    return true;
  };
  auto gap_ok = [&](i128 gn, i128 gd) { return gap_den != 0 && gn * (i128)gap_den <= (i128)gap_num * gd; };

  {
    const Bound b = bound(P, scale);
    emit(0, false, 0, b.ok, b.v, false, 0, 0);
  }
  if (has_inc) {
    best = rd128(inc_obj128, 0);
    have_best = true;
    P.best_assign.assign(inc_vals, inc_vals + P.n);
    emit(1, true, best, false, 0, false, 0, 0);
  }

  struct Frame {
    int var;
    int values[2];
    int nvalues;
    int tried;
    size_t mark;
    int order_pos;
    i128 entry_bound;
  };
  std::vector<Frame> frames;
  int order_pos = 0;
  bool stop = false, exhausted = false;
  auto frontier = [&](bool& hb) -> i128 {
    bool have = false;
    i128 out = 0;
    for (const Frame& f : frames)
      if (f.tried < f.nvalues && (!have || f.entry_bound < out)) {
        out = f.entry_bound;
        have = true;
      }
    if (!have) {
      hb = have_best;
      return best;
    }
    hb = true;
    return out;
  };
  auto pick_var = [&]() -> int {
    if (most_tight) return pick_most_tight(P);
    while (order_pos < n_order && P.val[order[order_pos]] != -1) ++order_pos;
    return order_pos < n_order ? order[order_pos] : -1;
  };

  bool descending = true;
  while (true) {
    if (nodes && nodes % 256 == 0) {
      if (time_limit_s >= 0 && elapsed() > time_limit_s) {
        stop = true;
        break;
      }
      if (node_limit >= 0 && nodes >= node_limit) {
        stop = true;
        break;
      }
    }
    if (descending) {
      const Bound eb = bound(P, scale);
      const bool pruned = !eb.ok || (have_best && eb.v >= best);
      const int v = pruned ? -1 : pick_var();
      if (v >= 0) {
        Frame f{v, {pref[v], 1 - pref[v]}, 2, 0, 0, order_pos, eb.v};
        if (dive_bound) {
          const size_t mark = P.trail.size();
          i128 sc[2];
          int sb[2], ns = 0;
          for (int i = 0; i < 2; ++i) {
            const int b = f.values[i];
            if (pr.assign(v, b)) {
              const Bound cb = bound(P, scale);
              if (cb.ok && (!have_best || cb.v < best)) {
                sc[ns] = cb.v;
                sb[ns] = b;
                ++ns;
              }
            }
            pr.undo_to(mark);
          }
          if (ns == 2 && sc[1] < sc[0]) {  // stable sort by bound
            std::swap(sc[0], sc[1]);
            std::swap(sb[0], sb[1]);
          }
          if (ns == 0) {
            if (frames.empty()) {
              exhausted = true;
              break;
            }
            descending = false;
            continue;
          }
          f.nvalues = ns;
          for (int i = 0; i < ns; ++i) f.values[i] = sb[i];
        }
        f.mark = P.trail.size();
        frames.push_back(f);
      } else {
        if (!pruned) {
          i128 obj = 0;
          for (size_t i = 0; i < P.obj_var.size(); ++i) obj += P.obj_cost[i] * (i128)P.val[P.obj_var[i]];
          if (!have_best || obj < best) {
            best = obj;
            have_best = true;
            P.best_assign.assign(P.val.begin(), P.val.end());
            bool hb;
            const i128 bnd = frontier(hb);
            i128 gn = 0, gd = 1;
            const bool hg = gap_of(hb, bnd, gn, gd);
            emit(2, true, best, hb, bnd, hg, gn, gd);
            if (hg && gap_ok(gn, gd)) {
              stop = true;
              break;
            }
          }
        }
        if (frames.empty()) {
          exhausted = true;
          break;
        }
        descending = false;
        continue;
      }
    }
    Frame& fr = frames.back();
    pr.undo_to(fr.mark);
    order_pos = fr.order_pos;
    if (have_best && fr.entry_bound >= best) fr.tried = fr.nvalues;
    bool advanced = false;
    while (fr.tried < fr.nvalues) {
      const int b = fr.values[fr.tried++];
      ++nodes;
      if (nodes % tel_every == 0) {
        bool hb;
        const i128 bnd = frontier(hb);
        i128 gn = 0, gd = 1;
        const bool hg = gap_of(hb, bnd, gn, gd);
        emit(3, have_best, best, hb, bnd, hg, gn, gd);
        if (have_best && hg && gap_ok(gn, gd)) {
          stop = true;
          break;
        }
      }
      if (pr.assign(fr.var, b)) {
        advanced = true;
        break;
      }
      pr.undo_to(fr.mark);
    }
    if (stop) break;
    if (advanced) {
      descending = true;
      continue;
    }
    const Frame done = fr;
    frames.pop_back();
    pr.undo_to(done.mark);
    order_pos = done.order_pos;
    if (frames.empty()) {
      exhausted = true;
      break;
    }
    descending = false;
  }
  (void)stop;
  *nodes_out = nodes;
  if (exhausted) {
    if (!have_best) {
      emit(4, false, 0, false, 0, false, 0, 0);
      return 2;
    }
    emit(4, true, best, true, best, true, 0, 1);
    wr128(res128, 0, best);
    wr128(res128, 1, best);
    wr128(res128, 2, 0);
    wr128(res128, 3, 1);
    return 0;
  }
  bool hb;
  const i128 bnd = frontier(hb);
  if (!have_best) {
    emit(4, false, 0, hb, bnd, false, 0, 0);
    wr128(res128, 1, hb ? bnd : 0);
    res128[8] = hb ? 1 : 0;
    return 3;
  }
  i128 gn = 0, gd = 1;
  const bool hg = gap_of(hb, bnd, gn, gd);
  if (hg && gn == 0) {
    emit(4, true, best, true, best, true, 0, 1);
    wr128(res128, 0, best);
    wr128(res128, 1, best);
    wr128(res128, 2, 0);
    wr128(res128, 3, 1);
    return 0;
  }
  emit(4, true, best, hb, bnd, hg, gn, gd);
  wr128(res128, 0, best);
  wr128(res128, 1, bnd);
  wr128(res128, 2, gn);
  wr128(res128, 3, gd);
  res128[8] = hg ? 1 : 0;
  return 1;
}

int monet_bnb_best(void* h, signed char* out) {
  Problem& P = *static_cast<Problem*>(h);
  if ((int)P.best_assign.size() != P.n) return 0;
  std::memcpy(out, P.best_assign.data(), P.n);
  return 1;
}

int monet_bnb_n_events(void* h) { return (int)static_cast<Problem*>(h)->events.size(); }

// event i: ints [kind, has_inc, has_bound, has_gap], int64 [nodes, elapsed_ms],
// 128-bit (hi, lo) [inc, bound, gap_num, gap_den]
int monet_bnb_event(void* h, int i, int* kinds, int64_t* counts, int64_t* vals128) {
  const Event& e = static_cast<Problem*>(h)->events[i];
  kinds[0] = e.kind;
  kinds[1] = e.has_inc;
  kinds[2] = e.has_bound;
  kinds[3] = e.has_gap;
  counts[0] = e.nodes;
  counts[1] = e.elapsed_ms;
  wr128(vals128, 0, e.inc);
  wr128(vals128, 1, e.bound);
  wr128(vals128, 2, e.gap_num);
  wr128(vals128, 3, e.gap_den);
  return 0;
}

}  // extern "C"
