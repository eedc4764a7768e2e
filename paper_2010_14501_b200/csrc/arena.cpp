// Static offset planner for the budget-capped arena.
//
// Every tensor instance of a replayed schedule has a known lifetime in ledger
// events (the alloc/free points of the reference simulator,
// pkg/src/remsched/schedule.py:344-457), so offsets are planned once before
// the step runs instead of being found by a runtime caching allocator.  The
// plan is "greedy by size": place blocks in decreasing size order at the
// lowest aligned offset that does not overlap any already placed block whose
// lifetime intersects.  The high-water mark is reported and must stay below
// the byte budget (and is compared with the ILP bound by the engine).
#include <algorithm>
#include <cstdint>
#include <numeric>
#include <vector>

#include "../../include/monet_b200.h"

extern "C" int monet_arena_plan(int64_t count, const int64_t* sizes, const int64_t* t_alloc, const int64_t* t_free,
                                int64_t align, int64_t capacity_bytes, int64_t* offsets, int64_t* peak_bytes) {
  if (count < 0 || align <= 0) return -22;
  std::vector<int64_t> order(count);
  std::iota(order.begin(), order.end(), 0);
  std::stable_sort(order.begin(), order.end(), [&](int64_t a, int64_t b) {
    if (sizes[a] != sizes[b]) return sizes[a] > sizes[b];
    return t_alloc[a] < t_alloc[b];
  });
  auto rnd = [&](int64_t v) { return (v + align - 1) / align * align; };
  std::vector<int64_t> placed;  // indices already assigned, kept sorted by offset
  placed.reserve(count);
  int64_t peak = 0;
  std::vector<std::pair<int64_t, int64_t>> busy;  // [begin, end) of conflicting placed blocks
  for (int64_t idx : order) {
    const int64_t need = rnd(std::max<int64_t>(sizes[idx], 1));
    busy.clear();
    for (int64_t j : placed) {
      if (t_alloc[j] < t_free[idx] && t_alloc[idx] < t_free[j]) busy.emplace_back(offsets[j], offsets[j] + rnd(std::max<int64_t>(sizes[j], 1)));
    }
    std::sort(busy.begin(), busy.end());
    // best fit: smallest gap that holds the block, else the end
    int64_t best = -1, best_gap = INT64_MAX, cursor = 0;
    for (auto& b : busy) {
      if (b.first > cursor) {
        int64_t gap = b.first - cursor;
        if (gap >= need && gap < best_gap) {
          best = cursor;
          best_gap = gap;
        }
      }
      cursor = std::max(cursor, b.second);
    }
    if (best < 0) best = cursor;
    offsets[idx] = best;
    peak = std::max(peak, best + need);
    placed.push_back(idx);
  }
  *peak_bytes = peak;
  if (capacity_bytes > 0 && peak > capacity_bytes) return -12;
  return 0;
}
