// Static offset planner for the budget-capped arena.
//
// Every tensor instance of a replayed schedule has a known lifetime in ledger
// events (the alloc/free points of the reference simulator,
// pkg/src/remsched/schedule.py:344-457), so offsets are planned once before
// the step runs instead of being found by a runtime caching allocator.  The
// plan is "greedy by size": place blocks in decreasing size order at the
// lowest aligned offset that does not overlap any already placed block whose
// lifetime intersects.  The high-water mark is reported and must stay below
// the byte budget; the engine compares params + high-water with the ILP bound
// (check_schedule), which equals the ledger peak on the ResNet-50 schedules,
// so the packing has to be gap-free at the peak instant.
#include <algorithm>
#include <cstdint>
#include <numeric>
#include <vector>

#include "../../include/monet_b200.h"

namespace {

// Place blocks in the given order, each at the best-fitting gap among the
// already placed blocks whose lifetimes intersect it (else on top).
int64_t place(const std::vector<int64_t>& order, const int64_t* sizes, const int64_t* t_alloc,
              const int64_t* t_free, int64_t align, std::vector<int64_t>& offs) {
  auto rnd = [&](int64_t v) { return (v + align - 1) / align * align; };
  std::vector<int64_t> placed;
  placed.reserve(order.size());
  std::vector<std::pair<int64_t, int64_t>> busy;
  int64_t peak = 0;
  for (int64_t idx : order) {
    const int64_t need = rnd(sizes[idx]);
    if (need == 0) {  // zero-byte blocks (e.g. a split conv's wgrad anchor) take no space
      offs[idx] = 0;
      continue;
    }
    busy.clear();
    for (int64_t j : placed)
      if (t_alloc[j] < t_free[idx] && t_alloc[idx] < t_free[j])
        busy.emplace_back(offs[j], offs[j] + rnd(sizes[j]));
    std::sort(busy.begin(), busy.end());
    int64_t best = -1, best_gap = INT64_MAX, cursor = 0;
    for (auto& b : busy) {
      if (b.first > cursor) {
        const int64_t gap = b.first - cursor;
        if (gap >= need && gap < best_gap) {
          best = cursor;
          best_gap = gap;
        }
      }
      cursor = std::max(cursor, b.second);
    }
    if (best < 0) best = cursor;
    offs[idx] = best;
    peak = std::max(peak, best + need);
    placed.push_back(idx);
  }
  return peak;
}

}  // namespace

// Several deterministic orderings are tried and the lowest high-water mark
// wins (ties: the earlier strategy):
//   0 size descending (classic greedy)
//   1 "heat" descending -- the largest live-byte total over the block's
//     lifetime first, so the blocks of the global peak pack gap-free at the
//     bottom -- then size
//   2 blocks live at the peak instant first (by allocation time), then size
//   3 allocation order (what a first-fit runtime allocator would see)
//   4 lifetime length descending, 5 lifetime x size descending
// then, if none is gap-free at the peak instant, a seeded local search.
extern "C" int monet_arena_plan(int64_t count, const int64_t* sizes, const int64_t* t_alloc, const int64_t* t_free,
                                int64_t align, int64_t capacity_bytes, int64_t* offsets, int64_t* peak_bytes) {
  if (count < 0 || align <= 0) return -22;
  int64_t horizon = 1;
  for (int64_t i = 0; i < count; ++i) horizon = std::max(horizon, t_free[i] + 1);
  auto rnd = [&](int64_t v) { return (v + align - 1) / align * align; };
  std::vector<int64_t> live(horizon + 1, 0);  // live rounded bytes per event time
  for (int64_t i = 0; i < count; ++i) {
    live[t_alloc[i]] += rnd(sizes[i]);
    live[t_free[i]] -= rnd(sizes[i]);
  }
  int64_t t_peak = 0, run = 0, best_live = -1;
  for (int64_t t = 0; t < horizon; ++t) {
    run += live[t];
    live[t] = run;
    if (run > best_live) {
      best_live = run;
      t_peak = t;
    }
  }
  std::vector<int64_t> heat(count, 0);
  for (int64_t i = 0; i < count; ++i)
    for (int64_t t = t_alloc[i]; t < t_free[i]; ++t) heat[i] = std::max(heat[i], live[t]);

  std::vector<int64_t> base(count);
  std::iota(base.begin(), base.end(), 0);
  auto by_size = [&](int64_t a, int64_t b) {
    if (sizes[a] != sizes[b]) return sizes[a] > sizes[b];
    return t_alloc[a] < t_alloc[b];
  };
  std::vector<std::vector<int64_t>> orders(6, base);
  std::stable_sort(orders[0].begin(), orders[0].end(), by_size);
  std::stable_sort(orders[1].begin(), orders[1].end(), [&](int64_t a, int64_t b) {
    if (heat[a] != heat[b]) return heat[a] > heat[b];
    return by_size(a, b);
  });
  std::stable_sort(orders[2].begin(), orders[2].end(), [&](int64_t a, int64_t b) {
    const bool pa = t_alloc[a] <= t_peak && t_peak < t_free[a], pb = t_alloc[b] <= t_peak && t_peak < t_free[b];
    if (pa != pb) return pa;
    if (pa) return t_alloc[a] < t_alloc[b];
    return by_size(a, b);
  });
  std::stable_sort(orders[3].begin(), orders[3].end(), [&](int64_t a, int64_t b) {
    if (t_alloc[a] != t_alloc[b]) return t_alloc[a] < t_alloc[b];
    return a < b;
  });
  std::stable_sort(orders[4].begin(), orders[4].end(), [&](int64_t a, int64_t b) {
    const int64_t la = t_free[a] - t_alloc[a], lb = t_free[b] - t_alloc[b];
    if (la != lb) return la > lb;
    return by_size(a, b);
  });
  std::stable_sort(orders[5].begin(), orders[5].end(), [&](int64_t a, int64_t b) {
    const double aa = (double)(t_free[a] - t_alloc[a]) * sizes[a], ab = (double)(t_free[b] - t_alloc[b]) * sizes[b];
    if (aa != ab) return aa > ab;
    return by_size(a, b);
  });
  std::vector<int64_t> offs(count), best_offs, best_order;
  int64_t best = INT64_MAX;
  for (const auto& order : orders) {
    const int64_t peak = place(order, sizes, t_alloc, t_free, align, offs);
    if (peak < best) {
      best = peak;
      best_offs = offs;
      best_order = order;
    }
    if (best == best_live) break;  // gap-free at the peak: optimal
  }
  // Still fragmented (few, huge, long-lived blocks -- VGG's 2 GiB activations):
  // deterministic local search over the placement order, 1-3 random swaps per
  // trial (fixed-seed LCG), accepting non-worsening orders, until gap-free.
  if (count > 1 && best > best_live) {
    uint64_t rng = 0x9E3779B97F4A7C15ull;
    auto next = [&](int64_t m) {
      rng = rng * 6364136223846793005ull + 1442695040888963407ull;
      return (int64_t)((rng >> 33) % (uint64_t)m);
    };
    std::vector<int64_t> trial;
    const int64_t budget_ops = 400000000;  // ~ trials * count^2 placement work
    const int64_t trials = std::max<int64_t>(64, std::min<int64_t>(8000, budget_ops / (count * count)));
    for (int64_t it = 0; it < trials && best > best_live; ++it) {
      trial = best_order;
      const int64_t swaps = 1 + next(3);
      for (int64_t k = 0; k < swaps; ++k) std::swap(trial[next(count)], trial[next(count)]);
      const int64_t peak = place(trial, sizes, t_alloc, t_free, align, offs);
      if (peak <= best) {
        best = peak;
        best_offs = offs;
        best_order = trial;
      }
    }
  }
  if (count == 0) best = 0;
  std::copy(best_offs.begin(), best_offs.end(), offsets);
  *peak_bytes = best;
  if (capacity_bytes > 0 && best > capacity_bytes) return -12;
  return 0;
}
