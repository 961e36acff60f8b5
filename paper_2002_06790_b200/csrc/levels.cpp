// Host C++ (in libdfsim_b200.so) for the per-class tables that used to be numpy loops in
// prepare.py: the Kahn level order of a class and the K4 v2 (level-group) critical-path plan.
// Both run once per topology class; at C3 / C4 sizes (45 / 18 classes of 2-10 k nodes and
// ~700 levels) the numpy versions cost ~30 + ~13 ms per class of one-shot setup.
//
// dfsim_level_order: Kahn waves, level = longest edge count from a source; each wave is
//   sorted by rank.  Any reverse topological order gives the same critical-path bits
//   (graph.py:463-469); the level order makes each schedule row contiguous
//   per level.
// dfsim_cp_levels_plan: the K4 v2 tables (see prepare.py's module docstring): groups of <=
//   `group` positions of one level, prefetch chunks of <= `chunk` positions, suffix values
//   read within the next chunk in shared-memory slots (interval colouring over the reverse
//   processing steps), the rest in an L2-resident spill row, prefetched with the reading
//   chunk.
#include <algorithm>
#include <cstdint>
#include <vector>

#include "dfsim_b200.h"

extern "C" int32_t dfsim_level_order(int32_t n, const int32_t *succ_off, const int32_t *succ_idx,
                                     const int32_t *indeg, int32_t *order, int32_t *level, int32_t *level_off) {
    if (n < 0 || (n > 0 && (!succ_off || !indeg || !order || !level || !level_off))) return -2;
    std::vector<int32_t> left(indeg, indeg + n), frontier, next;
    for (int32_t v = 0; v < n; v++) {
        level[v] = -1;
        if (left[v] == 0) frontier.push_back(v);
    }
    int32_t k = 0, lv = 0;
    level_off[0] = 0;
    while (!frontier.empty()) {
        std::sort(frontier.begin(), frontier.end());
        next.clear();
        for (int32_t v : frontier) {
            order[k++] = v;
            level[v] = lv;
            for (int32_t j = succ_off[v]; j < succ_off[v + 1]; j++)
                if (--left[succ_idx[j]] == 0) next.push_back(succ_idx[j]);
        }
        level_off[++lv] = k;
        frontier.swap(next);
    }
    return k == n ? lv : -1;  // -1: a cycle (or a dangling input) leaves nodes unordered
}

extern "C" int32_t dfsim_cp_levels_plan(int32_t n, const int32_t *succ_off, const int32_t *succ_idx,
                                        const int32_t *indeg, const int32_t *order, const int32_t *level_off,
                                        int32_t n_levels, int32_t group, int32_t chunk, int32_t *group_off,
                                        int32_t *chunk_off, int32_t *slot_of_pos, int32_t *spill_of_pos,
                                        int32_t *spill_off, int32_t *spill_list, int32_t *cp_succ,
                                        int32_t *cp_succ_abs, uint32_t *cp_meta, uint32_t *pinfo, int32_t *info) {
    if (n <= 0 || group <= 0 || chunk < group || n_levels <= 0) return -2;
    const int32_t E = succ_off[n];
    std::vector<int32_t> pos(n);
    for (int32_t p = 0; p < n; p++) pos[order[p]] = p;
    // groups of <= group positions inside each level; chunks of whole groups, <= chunk positions
    int32_t ng = 0;
    group_off[0] = 0;
    for (int32_t l = 0; l < n_levels; l++)
        for (int32_t p = level_off[l]; p < level_off[l + 1]; p += group)
            group_off[++ng] = std::min(level_off[l + 1], p + group);
    int32_t nc = 0, start = 0;
    chunk_off[0] = 0;
    for (int32_t g = 1; g <= ng; g++)
        if (group_off[g] - group_off[start] > chunk) chunk_off[++nc] = start = g - 1;
    if (chunk_off[nc] != ng) chunk_off[++nc] = ng;
    std::vector<int32_t> group_of(n), chunk_of(n);
    for (int32_t g = 0, c = 0; g < ng; g++) {
        while (chunk_off[c + 1] <= g) c++;
        for (int32_t p = group_off[g]; p < group_off[g + 1]; p++) group_of[p] = g, chunk_of[p] = c;
    }
    // edges in rank-CSR order: reader u (the producer, whose suffix reads it), value v (consumer)
    std::vector<uint8_t> near(E);
    std::vector<int32_t> last_near(n, -1);
    std::vector<uint8_t> spill_flag(n, 0);
    for (int32_t u = 0; u < n; u++) {
        const int32_t pu = pos[u], step = ng - 1 - group_of[pu];
        for (int32_t j = succ_off[u]; j < succ_off[u + 1]; j++) {
            const int32_t pv = pos[succ_idx[j]];
            near[j] = chunk_of[pu] >= chunk_of[pv] - 1;
            if (near[j])
                last_near[pv] = std::max(last_near[pv], step);
            else
                spill_flag[pv] = 1;
        }
    }
    // slot colouring in processing order (groups last to first); a slot frees after its last reader
    std::vector<int32_t> freel;
    std::vector<std::vector<int32_t>> release(ng + 1);
    int32_t nslots = 0;
    for (int32_t g = ng - 1; g >= 0; g--) {
        const int32_t step = ng - 1 - g;
        if (step >= 1) {
            auto &r = release[step - 1];
            freel.insert(freel.end(), r.begin(), r.end());
            r.clear();
        }
        for (int32_t p = group_off[g]; p < group_off[g + 1]; p++) {
            slot_of_pos[p] = 0xFFFF;
            if (last_near[p] < 0) continue;
            int32_t sl;
            if (!freel.empty()) {
                sl = freel.back();
                freel.pop_back();
            } else {
                sl = nslots++;
            }
            slot_of_pos[p] = sl;
            release[last_near[p]].push_back(sl);
        }
    }
    int32_t n_long = 0;
    for (int32_t p = 0; p < n; p++) spill_of_pos[p] = spill_flag[p] ? n_long++ : 0xFFFF;
    // (reading chunk, spill index) pairs, unique and sorted: each chunk's spill list
    std::vector<int64_t> pairs;
    for (int32_t u = 0; u < n; u++)
        for (int32_t j = succ_off[u]; j < succ_off[u + 1]; j++)
            if (!near[j])
                pairs.push_back(static_cast<int64_t>(chunk_of[pos[u]]) << 32 | spill_of_pos[pos[succ_idx[j]]]);
    std::sort(pairs.begin(), pairs.end());
    pairs.erase(std::unique(pairs.begin(), pairs.end()), pairs.end());
    const int32_t nl = static_cast<int32_t>(pairs.size());
    for (int32_t c = 0; c <= nc; c++) spill_off[c] = 0;
    for (int32_t i = 0; i < nl; i++) {
        spill_off[(pairs[i] >> 32) + 1]++;
        spill_list[i] = static_cast<int32_t>(pairs[i] & 0xFFFFFFFF);
    }
    int32_t max_reads = 0;
    for (int32_t c = 0; c < nc; c++) {
        max_reads = std::max(max_reads, spill_off[c + 1]);
        spill_off[c + 1] += spill_off[c];
    }
    const int32_t slot_region = (std::max(nslots, 1) + 1) / 2 * 2;
    const int32_t stage = (2 * chunk + max_reads + 1) / 2 * 2;
    // successor entries by reading position (rank-CSR order within a reader)
    int32_t e = 0;
    for (int32_t p = 0; p < n; p++) {
        const int32_t u = order[p], c = chunk_of[p], deg = succ_off[u + 1] - succ_off[u];
        cp_meta[p] = (static_cast<uint32_t>(e) & 0xFFFF) | static_cast<uint32_t>(std::min(deg, 255)) << 16 |
                     static_cast<uint32_t>(indeg[u] == 0) << 24;
        for (int32_t j = succ_off[u]; j < succ_off[u + 1]; j++, e++) {
            const int32_t pv = pos[succ_idx[j]];
            if (near[j]) {
                cp_succ[e] = cp_succ_abs[e] = slot_of_pos[pv];
            } else {
                const int64_t key = static_cast<int64_t>(c) << 32 | spill_of_pos[pv];
                const int32_t b = static_cast<int32_t>(std::lower_bound(pairs.begin(), pairs.end(), key) - pairs.begin())
                                  - spill_off[c];
                cp_succ[e] = 0x8000 | b;
                cp_succ_abs[e] = slot_region + (c & 1) * stage + 2 * chunk + b;
            }
        }
        const bool hs = slot_of_pos[p] != 0xFFFF, sp = spill_flag[p];
        pinfo[p] = (hs ? static_cast<uint32_t>(slot_of_pos[p]) & 0x7FFF : 0u) | static_cast<uint32_t>(hs) << 15 |
                   (sp ? static_cast<uint32_t>(spill_of_pos[p]) & 0x7FFF : 0u) << 16 | static_cast<uint32_t>(sp) << 31;
    }
    info[0] = ng;
    info[1] = nc;
    info[2] = nslots;
    info[3] = n_long;
    info[4] = max_reads;
    info[5] = nl;
    info[6] = slot_region;
    info[7] = stage;
    return 0;
}
