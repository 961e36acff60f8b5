// topological_order (graph.py:424-443): Kahn's algorithm with a min-heap of node ranks, so
// ties go to the lexicographically smallest id (node index == rank of the id string).  Host
// C++ in libdfsim_b200.so: the drop-in's exact order for one graph (the batched kernels use
// any valid order, which gives the same critical-path bits).
#include <cstdint>
#include <functional>
#include <queue>
#include <vector>

#include "dfsim_b200.h"

extern "C" int32_t dfsim_topological_order(int32_t n, const int32_t *succ_off, const int32_t *succ_idx,
                                           const int32_t *indeg, int32_t *order) {
    if (n < 0 || (n > 0 && (!succ_off || !indeg || !order))) return -1;
    std::vector<int32_t> left(indeg, indeg + n);
    std::priority_queue<int32_t, std::vector<int32_t>, std::greater<int32_t>> heap;
    for (int32_t v = 0; v < n; v++)
        if (left[v] == 0) heap.push(v);
    int32_t k = 0;
    while (!heap.empty()) {
        const int32_t v = heap.top();
        heap.pop();
        order[k++] = v;
        for (int32_t j = succ_off[v]; j < succ_off[v + 1]; j++)
            if (--left[succ_idx[j]] == 0) heap.push(succ_idx[j]);
    }
    return k;  // < n: some node is on a cycle (or waits on a dangling input)
}
