// fate_synth.cpp -- native batch generator for layered synthetic workloads.
//
// Produces, directly in the fate_bank / fate_state SoA layout, the instances
// the reference pipeline
//     synth_generate(SuiteSpec(kind="synthetic", depth, width, density, seed))
//       -> finalize_dag (assign_roles / assign_models / assign_devices)
//     make_instance(dag, batch, seed)
// would build (benchgen.py:247-393), plus the canonical scenario state of
// SURVEY.md §8(d) (paper_2605_07238_b200/scenarios.py), for thousands of
// instances at once.  It replays CPython's Mersenne Twister
// (random.Random(int): init_by_array over the 32-bit words of the seed;
// random() = genrand_res53; randrange(n) = getrandbits rejection) and the
// FNV-1a stable hash (hashutil.py:15-22) exactly, so the output is identical
// to packing the Python objects (checked by tests/test_fastgen.py).
#include <algorithm>
#include <cstdint>
#include <cstdlib>
#include <cstring>
#include <string>
#include <vector>

#include "fate.h"

namespace {

// ---- CPython-compatible MT19937 ---------------------------------------------
struct PyMT {
    uint32_t mt[624];
    int mti = 625;

    void init_genrand(uint32_t s) {
        mt[0] = s;
        for (mti = 1; mti < 624; mti++)
            mt[mti] = 1812433253u * (mt[mti - 1] ^ (mt[mti - 1] >> 30)) + (uint32_t)mti;
    }
    void init_by_array(const uint32_t* key, int klen) {
        init_genrand(19650218u);
        int i = 1, j = 0;
        for (int k = (624 > klen ? 624 : klen); k; k--) {
            mt[i] = (mt[i] ^ ((mt[i - 1] ^ (mt[i - 1] >> 30)) * 1664525u)) + key[j] + (uint32_t)j;
            i++;
            j++;
            if (i >= 624) { mt[0] = mt[623]; i = 1; }
            if (j >= klen) j = 0;
        }
        for (int k = 623; k; k--) {
            mt[i] = (mt[i] ^ ((mt[i - 1] ^ (mt[i - 1] >> 30)) * 1566083941u)) - (uint32_t)i;
            i++;
            if (i >= 624) { mt[0] = mt[623]; i = 1; }
        }
        mt[0] = 0x80000000u;
        mti = 624;
    }
    void seed_int(uint64_t n) {  // random.seed(int) for n >= 0
        uint32_t key[2];
        int klen = 0;
        key[klen++] = (uint32_t)(n & 0xffffffffu);
        if (n >> 32) key[klen++] = (uint32_t)(n >> 32);
        init_by_array(key, klen);
    }
    uint32_t next() {
        static const uint32_t mag01[2] = {0x0u, 0x9908b0dfu};
        uint32_t y;
        if (mti >= 624) {
            int kk;
            for (kk = 0; kk < 624 - 397; kk++) {
                y = (mt[kk] & 0x80000000u) | (mt[kk + 1] & 0x7fffffffu);
                mt[kk] = mt[kk + 397] ^ (y >> 1) ^ mag01[y & 1u];
            }
            for (; kk < 623; kk++) {
                y = (mt[kk] & 0x80000000u) | (mt[kk + 1] & 0x7fffffffu);
                mt[kk] = mt[kk + (397 - 624)] ^ (y >> 1) ^ mag01[y & 1u];
            }
            y = (mt[623] & 0x80000000u) | (mt[0] & 0x7fffffffu);
            mt[623] = mt[396] ^ (y >> 1) ^ mag01[y & 1u];
            mti = 0;
        }
        y = mt[mti++];
        y ^= (y >> 11);
        y ^= (y << 7) & 0x9d2c5680u;
        y ^= (y << 15) & 0xefc60000u;
        y ^= (y >> 18);
        return y;
    }
    double random() {
        uint32_t a = next() >> 5, b = next() >> 6;
        return (a * 67108864.0 + b) * (1.0 / 9007199254740992.0);
    }
    uint32_t randbelow(uint32_t n) {
        int k = 0;
        while ((1ull << k) <= n) k++;  // n.bit_length()
        uint32_t r = next() >> (32 - k);
        while (r >= n) r = next() >> (32 - k);
        return r;
    }
};

// ---- FNV-1a over "a|b|c" -----------------------------------------------------
struct Fnv {
    uint64_t h = 0xCBF29CE484222325ull;
    bool first = true;
    Fnv& part(const std::string& s) {
        if (!first) byte('|');
        first = false;
        for (unsigned char c : s) byte(c);
        return *this;
    }
    Fnv& part(long long v) { return part(std::to_string(v)); }
    void byte(unsigned char c) {
        h ^= c;
        h *= 0x100000001B3ull;
    }
};

std::string sid_of(int n) {
    char buf[32];
    snprintf(buf, sizeof buf, "s%02d", n);
    return buf;
}

// ROLE_KINDS order (model.py:17-29)
enum { PROMPT_PREP, RETRIEVAL, ROUTING, DECOMPOSITION, WORKER, MERGE, AGGREGATION,
       SUMMARIZATION, VALIDATION, VERIFICATION, FINAL_SYNTHESIS, N_KINDS };

}  // namespace

extern "C" {

// Catalog description passed from Python (all host pointers).
typedef struct fate_synth_catalog {
    int32_t n_devices;
    const char* const* device_names;  // sorted device ids
    int32_t n_models;                 // catalog aliases sorted; model id = rank
    int32_t role_row[N_KINDS];        // bank role-table row per role kind
    int32_t role_shard[N_KINDS];      // shard_eligible
    int32_t role_max_tok[N_KINDS];
    int32_t role_out_tok[N_KINDS];
    int32_t role_keep[N_KINDS];
    int32_t role_reuse[N_KINDS];
    const int32_t* role_models_ptr;   // [N_KINDS+1] CSR into role_models
    const int32_t* role_models;       // model ids in config order
} fate_synth_catalog;

typedef struct fate_synth_out {
    int32_t n_instances, n_stages_per, n_edges, batch, n_devices, kappa_cap;
    int32_t* st_model; int32_t* st_role; int32_t* st_prompt; int32_t* st_out; int32_t* st_group;
    int32_t* st_flags; int32_t* st_shard; int32_t* st_level;
    int32_t* par_ptr; int32_t* par_idx; int32_t* ch_ptr; int32_t* ch_idx;
    int32_t* q_prompt;
    double* clock; int32_t* frontier_level; int32_t* loc;
    int32_t* residency; double* dev_free; int32_t* kappa_n; int32_t* kappa;
} fate_synth_out;

void fate_synth_free(fate_synth_out* o) {
    if (!o) return;
    void* ptrs[] = {o->st_model, o->st_role, o->st_prompt, o->st_out, o->st_group, o->st_flags,
                    o->st_shard, o->st_level, o->par_ptr, o->par_idx, o->ch_ptr, o->ch_idx,
                    o->q_prompt, o->clock, o->frontier_level, o->loc, o->residency, o->dev_free,
                    o->kappa_n, o->kappa};
    for (void* p : ptrs) free(p);
    free(o);
}

// Instance i uses seed seed0 + i and scenario seed scen0 + i.
int fate_synth_layered(int32_t n_inst, int64_t seed0, int64_t scen0, int32_t depth, int32_t width,
                       double density, int32_t batch, const fate_synth_catalog* cat,
                       fate_synth_out** result) {
    if (n_inst < 1 || depth < 1 || width < 1 || batch < 0 || !cat || !result ||
        cat->n_devices < 1 || cat->n_devices > FATE_MAX_DEVICES || cat->n_models < 1)
        return FATE_EINVAL;
    const int V = depth * width, D = cat->n_devices, M = cat->n_models;
    // sorted-id rank of the creation index (ids "s%02d" compare as strings)
    std::vector<std::string> names(V);
    for (int n = 0; n < V; ++n) names[n] = sid_of(n);
    std::vector<int> order(V), rank(V);
    for (int n = 0; n < V; ++n) order[n] = n;
    std::sort(order.begin(), order.end(), [&](int a, int b) { return names[a] < names[b]; });
    for (int r = 0; r < V; ++r) rank[order[r]] = r;

    fate_synth_out* o = (fate_synth_out*)calloc(1, sizeof(fate_synth_out));
    const size_t NS = (size_t)n_inst * V;
    o->n_instances = n_inst; o->n_stages_per = V; o->batch = batch; o->n_devices = D;
    o->kappa_cap = M;  // at most one pg:<alias> entry per model
    auto I32 = [](size_t n) { return (int32_t*)calloc(n ? n : 1, sizeof(int32_t)); };
    o->st_model = I32(NS); o->st_role = I32(NS); o->st_prompt = I32(NS); o->st_out = I32(NS);
    o->st_group = I32(NS); o->st_flags = I32(NS); o->st_shard = I32(NS); o->st_level = I32(NS);
    o->par_ptr = I32(NS + 1); o->ch_ptr = I32(NS + 1);
    o->q_prompt = I32((size_t)n_inst * batch);
    o->clock = (double*)calloc(n_inst, sizeof(double));
    o->frontier_level = I32(n_inst);
    o->loc = I32(NS);
    o->residency = I32((size_t)n_inst * D);
    o->dev_free = (double*)calloc((size_t)n_inst * D, sizeof(double));
    o->kappa_n = I32((size_t)n_inst * D);
    o->kappa = I32((size_t)n_inst * D * M * 4);

    std::vector<int32_t> par_all, ch_all;
    std::vector<std::vector<int>> ups(V), downs(V);
    std::vector<int> level(V), indeg(V), outdeg(V), kind(V), model(V);
    std::vector<int> lw(depth);
    static const int EARLY[] = {PROMPT_PREP, RETRIEVAL, ROUTING, DECOMPOSITION};
    static const int MERGE_B[] = {MERGE, AGGREGATION};
    static const int LATE[] = {SUMMARIZATION, VALIDATION, VERIFICATION, FINAL_SYNTHESIS};
    int32_t par_pos = 0, ch_pos = 0;
    for (int ii = 0; ii < n_inst; ++ii) {
        const long long seed = seed0 + ii, scen = scen0 + ii;
        const std::string wid = "synthetic-d" + std::to_string(depth) + "w" + std::to_string(width) +
                                "-s" + std::to_string(seed);
        for (int n = 0; n < V; ++n) { ups[n].clear(); downs[n].clear(); }
        // synth_generate edges (benchgen.py:373-386)
        PyMT rng;
        rng.seed_int((uint64_t)seed);
        for (int d = 1; d < depth; ++d) {
            for (int i = 0; i < width; ++i) {
                const int v = d * width + i;
                for (int j = 0; j < width; ++j)
                    if (rng.random() < density) ups[v].push_back((d - 1) * width + j);
                if (ups[v].empty()) ups[v].push_back((d - 1) * width + (int)rng.randbelow(width));
            }
        }
        for (int v = 0; v < V; ++v)
            for (int u : ups[v]) downs[u].push_back(v);
        // annotations: layered DAG -> level = layer (every stage has a parent
        // in the previous layer)
        for (int v = 0; v < V; ++v) {
            level[v] = v / width;
            indeg[v] = (int)ups[v].size();
            outdeg[v] = (int)downs[v].size();
        }
        std::fill(lw.begin(), lw.end(), width);
        const int max_level = depth - 1;
        // assign_roles + assign_models (benchgen.py:247-316)
        for (int v = 0; v < V; ++v) {
            const int lvl = level[v], ind = indeg[v], outd = outdeg[v];
            const int here_w = lw[lvl], prev_w = lvl >= 1 ? lw[lvl - 1] : 1;
            const int* bucket;
            int blen;
            static const int WORKER_B[] = {WORKER};
            if (ind == 0 || (lvl <= 1 && here_w >= 3)) { bucket = EARLY; blen = 4; }
            else if (lvl < max_level && outd >= 3) { bucket = WORKER_B; blen = 1; }
            else if (ind >= 3 || (ind >= 2 && 2 * ind >= prev_w)) { bucket = MERGE_B; blen = 2; }
            else if (outd == 0 || lvl == max_level) { bucket = LATE; blen = 4; }
            else { bucket = WORKER_B; blen = 1; }
            Fnv hr;
            hr.part(names[v]).part(seed);
            kind[v] = bucket[hr.h % (uint64_t)blen];
            const int k = kind[v];
            const int c0 = cat->role_models_ptr[k], c1 = cat->role_models_ptr[k + 1];
            if (c1 <= c0) { fate_synth_free(o); return FATE_EINVAL; }
            Fnv hm;
            hm.part(wid).part(names[v]).part(seed);
            model[v] = cat->role_models[c0 + (int)(hm.h % (uint64_t)(c1 - c0))];
        }
        // pack stages in sorted-id order
        const size_t g0 = (size_t)ii * V;
        for (int r = 0; r < V; ++r) {
            const int v = order[r], k = kind[v];
            const size_t g = g0 + r;
            o->st_model[g] = model[v];
            o->st_role[g] = cat->role_row[k];
            o->st_prompt[g] = cat->role_max_tok[k] / 4;
            o->st_out[g] = cat->role_out_tok[k];
            o->st_group[g] = cat->role_reuse[k] ? model[v] : -1;  // group "pg:<alias>" -> model id
            o->st_flags[g] = (cat->role_reuse[k] ? FATE_STAGE_CACHE_REUSE : 0) |
                             (cat->role_keep[k] ? FATE_STAGE_KEEP_CACHE : 0);
            o->st_shard[g] = cat->role_shard[k] ? 2 : 1;
            o->st_level[g] = level[v];
            std::vector<int> pu, cd;
            for (int u : ups[v]) pu.push_back(rank[u]);
            for (int c : downs[v]) cd.push_back(rank[c]);
            std::sort(pu.begin(), pu.end());
            std::sort(cd.begin(), cd.end());
            o->par_ptr[g] = par_pos;
            o->ch_ptr[g] = ch_pos;
            for (int x : pu) { par_all.push_back((int32_t)(g0 + x)); par_pos++; }
            for (int x : cd) { ch_all.push_back((int32_t)(g0 + x)); ch_pos++; }
        }
        // make_queries (benchgen.py:343-353)
        for (int q = 0; q < batch; ++q) {
            Fnv hq;
            hq.part(wid).part("query").part(q).part(seed);
            o->q_prompt[(size_t)ii * batch + q] = 200 + (int32_t)(hq.h % 600ull);
        }
        // scenario state (scenarios.build_scenario)
        Fnv hl;
        hl.part(wid).part("L").part(scen);
        const int cut = 1 + (int)(hl.h % (uint64_t)(max_level > 0 ? max_level : 1));
        const double clock = 1000.0 * cut;
        o->clock[ii] = clock;
        o->frontier_level[ii] = cut;
        int32_t* loc = o->loc + g0;
        int32_t* kn = o->kappa_n + (size_t)ii * D;
        int32_t* kap = o->kappa + (size_t)ii * D * M * 4;
        // entry store per device: group -> (tokens, model, sticky, survived), insertion ordered
        struct Ent { int group, tokens, model; bool sticky, survived; };
        std::vector<std::vector<Ent>> store(D);
        for (int r = 0; r < V; ++r) {
            const int v = order[r];
            loc[r] = -1;
            if (level[v] >= cut) continue;
            Fnv h;
            h.part(wid).part("loc").part(names[v]).part(scen);
            const int first = (int)(h.h % (uint64_t)D);
            const size_t g = g0 + r;
            int shards[2] = {first, -1};
            int n_sh = 1;
            if (o->st_shard[g] == 2 && ((h.h >> 8) & 1ull)) { shards[1] = (first + 1) % D; n_sh = 2; }
            // plurality device of the output shards, ties -> smallest id
            int best = first;
            if (n_sh == 2) {
                const int n0 = batch / 2 + (batch % 2), n1 = batch / 2;
                if (n1 > n0) best = shards[1];
                else if (n1 == n0) best = std::min(shards[0], shards[1]);
            }
            loc[r] = best;
            if ((o->st_flags[g] & FATE_STAGE_KEEP_CACHE) && o->st_group[g] != -1) {
                for (int j = 0; j < n_sh; ++j) {
                    auto& st = store[shards[j]];
                    bool found = false;
                    for (auto& e : st) {
                        if (e.group == o->st_group[g]) {
                            e.tokens = std::max(e.tokens, (int)o->st_prompt[g]);
                            e.model = o->st_model[g];
                            e.sticky = true;
                            e.survived = false;
                            found = true;
                            break;
                        }
                    }
                    if (!found) st.push_back({o->st_group[g], o->st_prompt[g], o->st_model[g], true, false});
                }
            }
        }
        for (int d = 0; d < D; ++d) {
            Fnv h;
            h.part(wid).part("dev").part(cat->device_names[d]).part(scen);
            const int m = (int)(h.h % (uint64_t)M);
            // _evict_on_switch (state.py:224-234): groups visited in sorted order;
            // the outcome per entry does not depend on the visiting order
            auto& st = store[d];
            std::vector<Ent> kept;
            for (auto& e : st) {
                if (e.model == m) { e.survived = false; kept.push_back(e); }
                else if (e.sticky && !e.survived) { e.survived = true; kept.push_back(e); }
            }
            st.swap(kept);
            o->residency[(size_t)ii * D + d] = m;
            o->dev_free[(size_t)ii * D + d] =
                ((h.h >> 16) & 1ull) ? clock + 12.5 * (double)((h.h >> 8) % 4ull) : clock - 5.0;
            kn[d] = (int)st.size();
            for (size_t k = 0; k < st.size(); ++k) {
                int32_t* e = kap + ((size_t)d * M + k) * 4;
                e[0] = st[k].group; e[1] = st[k].tokens; e[2] = st[k].model; e[3] = 0;
            }
        }
    }
    o->par_ptr[NS] = par_pos;
    o->ch_ptr[NS] = ch_pos;
    o->n_edges = par_pos;
    o->par_idx = I32(par_all.size());
    o->ch_idx = I32(ch_all.size());
    std::copy(par_all.begin(), par_all.end(), o->par_idx);
    std::copy(ch_all.begin(), ch_all.end(), o->ch_idx);
    *result = o;
    return 0;
}

}  // extern "C"
