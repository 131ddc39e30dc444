// fate_host.cpp -- host-side (CPU, native) preparation for the FATE scorer.
//
// Horizon windows: for each stage v, its descendants x with level offset
// l = level(x) - level(v) in 1..levels, bucketed by l and sorted ascending
// (= the reference's _descendants_by_level restricted to the offsets the
// tail reads, costs.py:294-299, :354-379).  Levels are longest-path depths,
// so any descendant at offset l is reachable in <= l hops: a BFS bounded at
// `levels` hops finds every descendant the tail can use, without walking the
// whole downstream DAG like the reference does.
#include <algorithm>
#include <cstdint>
#include <string>
#include <vector>

#include "fate.h"

namespace {

struct WindowScratch {
    std::vector<int32_t> stamp;
    std::vector<int32_t> frontier, next;
    std::vector<std::vector<int32_t>> buckets;
    int32_t epoch = 0;
};

// Collects the buckets of stage v into ws.buckets[0..levels-1].
void window_of(int32_t v, const int32_t* ch_ptr, const int32_t* ch_idx, const int32_t* level,
               int32_t levels, WindowScratch& ws) {
    ++ws.epoch;
    for (auto& bk : ws.buckets) bk.clear();
    ws.frontier.assign(1, v);
    const int32_t lv = level[v];
    for (int32_t hop = 0; hop < levels && !ws.frontier.empty(); ++hop) {
        ws.next.clear();
        for (int32_t u : ws.frontier) {
            for (int32_t e = ch_ptr[u]; e < ch_ptr[u + 1]; ++e) {
                const int32_t c = ch_idx[e];
                if (ws.stamp[c] == ws.epoch) continue;
                ws.stamp[c] = ws.epoch;
                ws.next.push_back(c);
                const int32_t off = level[c] - lv;
                if (off >= 1 && off <= levels) ws.buckets[off - 1].push_back(c);
            }
        }
        ws.frontier.swap(ws.next);
    }
    for (auto& bk : ws.buckets) std::sort(bk.begin(), bk.end());
}

}  // namespace

extern "C" {

int fate_windows_count_host(int32_t n_stages, const int32_t* ch_ptr, const int32_t* ch_idx,
                            const int32_t* level, int32_t levels, int64_t* n_items) {
    if (n_stages < 0 || levels < 0 || !n_items || (n_stages > 0 && (!ch_ptr || !level)))
        return FATE_EINVAL;
    WindowScratch ws;
    ws.stamp.assign((size_t)n_stages, 0);
    ws.buckets.resize((size_t)levels);
    int64_t total = 0;
    if (levels > 0) {
        for (int32_t v = 0; v < n_stages; ++v) {
            window_of(v, ch_ptr, ch_idx, level, levels, ws);
            for (auto& bk : ws.buckets) total += (int64_t)bk.size();
        }
    }
    *n_items = total;
    return 0;
}

int fate_windows_build_host(int32_t n_stages, const int32_t* ch_ptr, const int32_t* ch_idx,
                            const int32_t* level, int32_t levels, int64_t* ptr_out,
                            int32_t* idx_out) {
    if (n_stages < 0 || levels < 0 || !ptr_out) return FATE_EINVAL;
    WindowScratch ws;
    ws.stamp.assign((size_t)n_stages, 0);
    ws.buckets.resize((size_t)levels);
    int64_t pos = 0;
    ptr_out[0] = 0;
    for (int32_t v = 0; v < n_stages; ++v) {
        if (levels > 0) window_of(v, ch_ptr, ch_idx, level, levels, ws);
        for (int32_t l = 0; l < levels; ++l) {
            for (int32_t x : ws.buckets[l]) idx_out[pos++] = x;
            ptr_out[(int64_t)v * levels + l + 1] = pos;
        }
    }
    return 0;
}

// Window parents: per (stage v, level l) the distinct parents p != v of the
// bucket's descendants, ascending -- the stages whose output location decides
// whether the level's tail chain has any locality op (costs.py:332-348).
static void wpar_of(int64_t vl, int32_t v, const int64_t* win_ptr, const int32_t* win_idx,
                    const int32_t* par_ptr, const int32_t* par_idx, std::vector<int32_t>& out) {
    out.clear();
    for (int64_t i = win_ptr[vl]; i < win_ptr[vl + 1]; ++i) {
        const int32_t x = win_idx[i];
        for (int32_t e = par_ptr[x]; e < par_ptr[x + 1]; ++e)
            if (par_idx[e] != v) out.push_back(par_idx[e]);
    }
    std::sort(out.begin(), out.end());
    out.erase(std::unique(out.begin(), out.end()), out.end());
}

int fate_window_parents_host(int32_t n_stages, int32_t levels, const int64_t* win_ptr,
                             const int32_t* win_idx, const int32_t* par_ptr,
                             const int32_t* par_idx, int64_t* ptr_out, int32_t* idx_out,
                             int64_t* n_out) {
    if (n_stages < 0 || levels < 0 || !n_out) return FATE_EINVAL;
    std::vector<int32_t> buf;
    int64_t pos = 0;
    if (ptr_out) ptr_out[0] = 0;
    for (int32_t v = 0; v < n_stages; ++v) {
        for (int32_t l = 0; l < levels; ++l) {
            const int64_t vl = (int64_t)v * levels + l;
            wpar_of(vl, v, win_ptr, win_idx, par_ptr, par_idx, buf);
            if (idx_out)
                for (size_t k = 0; k < buf.size(); ++k) idx_out[pos + (int64_t)k] = buf[k];
            pos += (int64_t)buf.size();
            if (ptr_out) ptr_out[vl + 1] = pos;
        }
    }
    *n_out = pos;
    return 0;
}

}  // extern "C"
