// fate_mirror.cu -- device-resident incremental execution-state mirror and GPU
// ready set.
//
// The scorer's input state s_t = (residency, device_free, prefix store,
// output locations, clock) of ONE running workflow instance lives in HBM and
// is updated in place from the executor's transition events, instead of
// snapshotting the whole ExecutionState on the host and packing / uploading it
// every wave (reference executor.py:200 snapshot -> our pack_states).  The
// events restate ExecutionState's transitions (reference state.py:130-272):
//
//   COMMIT(v, slots)        commit_stage           (state.py:130-135): a new
//                           progress record (a stage can be re-committed while
//                           a task of an earlier commit still runs)
//   START(v, d, finish)     on_task_start          (state.py:137-167):
//                           model switch -> _evict_on_switch (state.py:220-234)
//                           and residency; device_free = finish; first start
//                           of a stage clears its commit
//   COMPLETE(v, d, finish,  on_task_complete       (state.py:169-181):
//            queries)       clock = max(clock, finish); _seed_prefixes
//                           (state.py:236-256, _merge_entry state.py:258-266);
//                           when the stage's last slot finishes: completed,
//                           output location = plurality device of the shards
//                           (output_device, state.py:96-108), children's
//                           remaining-parent counters decremented
//
// Events of a wave are applied in order by one thread (they are few and
// strictly sequential); the ready set (model.py:306-319) is one thread per
// stage over the remaining-parent counters plus the claimed flags, compacted
// per warp (ascending within a warp; warps append in completion order, so the
// set is unordered across warps -- DeviceMirror.ready() sorts it).  The mirror's arrays ARE a
// one-scenario fate_state: fate_score reads them directly.
#include <cuda_runtime.h>

#include <cstdint>
#include <cstring>
#include <string>
#include <vector>

#include "fate.h"
#include "fate_internal.h"

struct fate_mirror {
    int device = 0;
    int D = 0, V = 0, cap = 0, nq = 0;
    int32_t stage_off = 0;     // global index of the instance's first stage
    int32_t empty_model = -1;  // model id of "" (entries seeded by model-less stages)
    // device arrays (fate_state of one scenario + bookkeeping)
    int32_t* scen_inst = nullptr;
    double* scen_clock = nullptr;
    int64_t* scen_loc_off = nullptr;
    int32_t* scen_done_level = nullptr;
    int32_t* loc = nullptr;        // [V]
    int32_t* residency = nullptr;  // [D]
    double* dev_free = nullptr;    // [D]
    int32_t* kappa_n = nullptr;    // [D]
    int32_t* kappa = nullptr;      // [D*cap*4] (group, tokens, model, flags: 1 sticky, 2 survived)
    int32_t* status = nullptr;     // [V] bit0 completed, bit1 committed
    int32_t* running = nullptr;    // [V] running tasks
    int32_t* slots = nullptr;      // [V] committed slot count
    int32_t* finished = nullptr;   // [V] finished slots
    int32_t* remaining = nullptr;  // [V] uncompleted parents
    int32_t* shard_q = nullptr;    // [V*D] finished queries per (stage, device)
    int32_t* q_group = nullptr;    // [nq] query prefix group id (-1 None)
    int32_t* q_tokens = nullptr;   // [nq] group_tokens(group, prompt) (state.py:79-85)
    int32_t* error = nullptr;      // [1] 0 ok, else a FATE_MIRROR_E* code
    // bank pieces the events read (device pointers of the bank)
    const int32_t* st_model = nullptr;
    const int32_t* st_group = nullptr;
    const int32_t* st_prompt = nullptr;
    const int32_t* st_flags = nullptr;
    const int32_t* st_level = nullptr;
    const int32_t* ch_ptr = nullptr;
    const int32_t* ch_idx = nullptr;
    const int32_t* par_ptr = nullptr;
    // event staging
    void* ev = nullptr;
    size_t ev_cap = 0;
    int32_t* evq = nullptr;
    size_t evq_cap = 0;
    int32_t* ready_n = nullptr;  // [1]
};

namespace {

constexpr int E_OK = 0, E_KAPPA = 1, E_STATE = 2;

struct MirrorArgs {
    int D, V, cap, stage_off, empty_model;
    int32_t *loc, *residency, *kappa_n, *kappa, *status, *running, *slots, *finished, *remaining,
        *shard_q, *done_level, *error;
    double *dev_free, *clock;
    const int32_t *q_group, *q_tokens, *st_model, *st_group, *st_prompt, *st_flags, *st_level,
        *ch_ptr, *ch_idx;
};

__device__ void merge_entry(const MirrorArgs& a, int d, int group, int tokens, int model,
                            bool sticky) {
    int32_t* kap = a.kappa + (size_t)d * a.cap * 4;
    const int n = a.kappa_n[d];
    for (int k = 0; k < n; ++k) {
        int32_t* e = kap + 4 * k;
        if (e[0] == group) {
            e[1] = e[1] > tokens ? e[1] : tokens;
            e[2] = model;
            e[3] = (e[3] & 1) | (sticky ? 1 : 0);  // sticky |= new; survived = False
            return;
        }
    }
    if (n >= a.cap) {
        atomicExch(a.error, E_KAPPA);
        return;
    }
    int32_t* e = kap + 4 * n;
    e[0] = group;
    e[1] = tokens;
    e[2] = model;
    e[3] = sticky ? 1 : 0;
    a.kappa_n[d] = n + 1;
}

__device__ void evict_on_switch(const MirrorArgs& a, int d, int new_model) {
    // iteration order does not matter: each entry's fate depends on itself
    int32_t* kap = a.kappa + (size_t)d * a.cap * 4;
    const int n = a.kappa_n[d];
    int w = 0;
    for (int k = 0; k < n; ++k) {
        int32_t e0 = kap[4 * k], e1 = kap[4 * k + 1], e2 = kap[4 * k + 2], e3 = kap[4 * k + 3];
        bool keep = true;
        if (e2 == new_model) {
            e3 &= ~2;  // survived = False
        } else if ((e3 & 1) && !(e3 & 2)) {
            e3 |= 2;  // sticky entry survives one switch
        } else {
            keep = false;
        }
        if (keep) {  // compaction keeps dict order (insertion order of survivors)
            kap[4 * w] = e0;
            kap[4 * w + 1] = e1;
            kap[4 * w + 2] = e2;
            kap[4 * w + 3] = e3;
            ++w;
        }
    }
    a.kappa_n[d] = w;
}

__global__ void fate_mirror_apply_kernel(MirrorArgs a, const fate_event* ev, int n_ev,
                                         const int32_t* evq) {
    if (threadIdx.x != 0 || blockIdx.x != 0) return;
    for (int i = 0; i < n_ev; ++i) {
        const fate_event e = ev[i];
        const int v = e.stage - a.stage_off;
        if (v < 0 || v >= a.V || (e.kind != FATE_EV_COMMIT && (e.device < 0 || e.device >= a.D))) {
            atomicExch(a.error, E_STATE);
            return;
        }
        if (e.kind == FATE_EV_COMMIT) {
            // commit_stage replaces the stage's progress record: slot count,
            // finished shards (and so the output-location tally) start over
            a.status[v] |= 2;
            a.slots[v] = e.slots;
            a.finished[v] = 0;
            for (int x = 0; x < a.D; ++x) a.shard_q[(size_t)v * a.D + x] = 0;
        } else if (e.kind == FATE_EV_START) {
            const int d = e.device;
            const int m = a.st_model[e.stage];
            if (m >= 0 && a.residency[d] != m) {
                evict_on_switch(a, d, m);
                a.residency[d] = m;
            }
            a.dev_free[d] = e.time;
            a.status[v] &= ~2;  // first start clears the commit (later starts: no-op)
            a.running[v] += 1;
        } else if (e.kind == FATE_EV_COMPLETE) {
            const int d = e.device;
            a.clock[0] = a.clock[0] > e.time ? a.clock[0] : e.time;
            a.running[v] -= 1;
            // _seed_prefixes: model is stage.model or ""
            const int m = a.st_model[e.stage];
            const int mid = m >= 0 ? m : a.empty_model;
            const bool keep_cache = a.st_flags[e.stage] & FATE_STAGE_KEEP_CACHE;
            const int g = a.st_group[e.stage];
            if (keep_cache && g != -1) merge_entry(a, d, g, a.st_prompt[e.stage], mid, true);
            for (int k = 0; k < e.nq; ++k) {
                const int q = evq[e.q0 + k];
                const int qg = a.q_group[q];
                if (qg == -1) continue;
                merge_entry(a, d, qg, a.q_tokens[q], mid, keep_cache);
            }
            // per (stage, device): 2 * queries + 1 once the device holds a shard
            int32_t& sq = a.shard_q[(size_t)v * a.D + d];
            sq = (sq | 1) + 2 * e.nq;
            a.finished[v] += 1;
            if (a.finished[v] == a.slots[v]) {
                a.status[v] |= 1;
                // output_device: the shard device with the most output queries,
                // ties (including all-empty shards) -> smallest device id
                int best = -1, bc = -1;
                for (int x = 0; x < a.D; ++x) {
                    const int c = a.shard_q[(size_t)v * a.D + x];
                    if ((c & 1) && (c >> 1) > bc) {
                        bc = c >> 1;
                        best = x;
                    }
                }
                a.loc[v] = best;
                const int lvl = a.st_level[e.stage];
                if (lvl > a.done_level[0]) a.done_level[0] = lvl;
                for (int c = a.ch_ptr[e.stage]; c < a.ch_ptr[e.stage + 1]; ++c)
                    a.remaining[a.ch_idx[c] - a.stage_off] -= 1;
            }
        }
    }
}

// ready_set (model.py:306-319): not completed, not running, not committed,
// every parent completed; ascending within each warp's slice, warp slices in
// completion order (the host sorts)
__global__ void fate_mirror_ready_kernel(int V, int stage_off, const int32_t* status,
                                         const int32_t* running, const int32_t* remaining,
                                         int32_t* out, int32_t* n_out) {
    const int v = blockIdx.x * blockDim.x + threadIdx.x;
    const bool r = v < V && status[v] == 0 && running[v] == 0 && remaining[v] == 0;
    const unsigned bal = __ballot_sync(0xffffffffu, r);
    int base = 0;
    if ((threadIdx.x & 31) == 0 && bal) base = atomicAdd(n_out, __popc(bal));
    base = __shfl_sync(0xffffffffu, base, 0);
    if (r) out[base + __popc(bal & ((1u << (threadIdx.x & 31)) - 1u))] = v + stage_off;
}

__global__ void fate_mirror_init_kernel(int V, const int32_t* par_ptr, int stage_off,
                                        int32_t* remaining) {
    const int v = blockIdx.x * blockDim.x + threadIdx.x;
    if (v < V) remaining[v] = par_ptr[stage_off + v + 1] - par_ptr[stage_off + v];
}

int cuda_fail(cudaError_t e, const char* what) {
    return fate_internal_fail((int)e, std::string(what) + ": " + cudaGetErrorString(e));
}

MirrorArgs args_of(fate_mirror* m) {
    MirrorArgs a;
    a.D = m->D;
    a.V = m->V;
    a.cap = m->cap;
    a.stage_off = m->stage_off;
    a.empty_model = m->empty_model;
    a.loc = m->loc;
    a.residency = m->residency;
    a.kappa_n = m->kappa_n;
    a.kappa = m->kappa;
    a.status = m->status;
    a.running = m->running;
    a.slots = m->slots;
    a.finished = m->finished;
    a.remaining = m->remaining;
    a.shard_q = m->shard_q;
    a.done_level = m->scen_done_level;
    a.error = m->error;
    a.dev_free = m->dev_free;
    a.clock = m->scen_clock;
    a.q_group = m->q_group;
    a.q_tokens = m->q_tokens;
    a.st_model = m->st_model;
    a.st_group = m->st_group;
    a.st_prompt = m->st_prompt;
    a.st_flags = m->st_flags;
    a.st_level = m->st_level;
    a.ch_ptr = m->ch_ptr;
    a.ch_idx = m->ch_idx;
    return a;
}

}  // namespace

extern "C" {

int fate_mirror_create(const fate_bank* bank, int32_t inst, int32_t kappa_cap,
                       const int32_t* q_group_host, const int32_t* q_tokens_host,
                       int32_t empty_model, void* stream, fate_mirror** out) {
    if (!bank || !out || kappa_cap < 1 || kappa_cap > FATE_MAX_KAPPA || inst < 0 ||
        inst >= bank->n_instances)
        return fate_internal_fail(FATE_EINVAL, "fate_mirror_create: bad arguments");
    int32_t off = 0, nst = 0, nq = 0;
    cudaError_t e;
    // the instance's stage range and query count come from the (device) bank
    if ((e = cudaMemcpy(&off, bank->inst_stage_off + inst, 4, cudaMemcpyDeviceToHost)) ||
        (e = cudaMemcpy(&nst, bank->inst_n_stages + inst, 4, cudaMemcpyDeviceToHost)) ||
        (e = cudaMemcpy(&nq, bank->inst_n_queries + inst, 4, cudaMemcpyDeviceToHost)))
        return cuda_fail(e, "fate_mirror_create: bank");
    auto* m = new fate_mirror();
    cudaGetDevice(&m->device);
    m->D = bank->n_devices;
    m->V = nst;
    m->cap = kappa_cap;
    m->nq = nq;
    m->stage_off = off;
    m->empty_model = empty_model;
    m->st_model = bank->st_model;
    m->st_group = bank->st_group;
    m->st_prompt = bank->st_prompt;
    m->st_flags = bank->st_flags;
    m->st_level = bank->st_level;
    m->ch_ptr = bank->ch_ptr;
    m->ch_idx = bank->ch_idx;
    m->par_ptr = bank->par_ptr;
    const size_t V = (size_t)nst, D = (size_t)m->D;
    struct A {
        void** p;
        size_t bytes;
    } allocs[] = {
        {(void**)&m->scen_inst, 4},
        {(void**)&m->scen_clock, 8},
        {(void**)&m->scen_loc_off, 8},
        {(void**)&m->scen_done_level, 4},
        {(void**)&m->loc, 4 * V},
        {(void**)&m->residency, 4 * D},
        {(void**)&m->dev_free, 8 * D},
        {(void**)&m->kappa_n, 4 * D},
        {(void**)&m->kappa, 16 * D * (size_t)kappa_cap},
        {(void**)&m->status, 4 * V},
        {(void**)&m->running, 4 * V},
        {(void**)&m->slots, 4 * V},
        {(void**)&m->finished, 4 * V},
        {(void**)&m->remaining, 4 * V},
        {(void**)&m->shard_q, 4 * V * D},
        {(void**)&m->q_group, 4 * (size_t)(nq > 0 ? nq : 1)},
        {(void**)&m->q_tokens, 4 * (size_t)(nq > 0 ? nq : 1)},
        {(void**)&m->error, 4},
        {(void**)&m->ready_n, 4},
    };
    for (auto& al : allocs) {
        if ((e = cudaMalloc(al.p, al.bytes ? al.bytes : 4)) != cudaSuccess) {
            fate_mirror_destroy(m);
            return cuda_fail(e, "fate_mirror_create: cudaMalloc");
        }
    }
    cudaStream_t s = static_cast<cudaStream_t>(stream);
    // initial state (ExecutionState.initial, state.py:60-69): nothing resident,
    // no prefixes, every device free at 0, clock 0
    const int32_t zero = 0, none = -1;
    const double dz = 0.0;
    const int64_t lz = 0;
    std::vector<int32_t> ones_v(V > D ? V : D, -1);
    if ((e = cudaMemcpyAsync(m->scen_inst, &inst, 4, cudaMemcpyHostToDevice, s)) ||
        (e = cudaMemcpyAsync(m->scen_clock, &dz, 8, cudaMemcpyHostToDevice, s)) ||
        (e = cudaMemcpyAsync(m->scen_loc_off, &lz, 8, cudaMemcpyHostToDevice, s)) ||
        (e = cudaMemcpyAsync(m->scen_done_level, &none, 4, cudaMemcpyHostToDevice, s)) ||
        (e = cudaMemcpyAsync(m->loc, ones_v.data(), 4 * V, cudaMemcpyHostToDevice, s)) ||
        (e = cudaMemcpyAsync(m->residency, ones_v.data(), 4 * D, cudaMemcpyHostToDevice, s)) ||
        (e = cudaMemsetAsync(m->dev_free, 0, 8 * D, s)) ||
        (e = cudaMemsetAsync(m->kappa_n, 0, 4 * D, s)) ||
        (e = cudaMemsetAsync(m->kappa, 0, 16 * D * kappa_cap, s)) ||
        (e = cudaMemsetAsync(m->status, 0, 4 * V, s)) ||
        (e = cudaMemsetAsync(m->running, 0, 4 * V, s)) ||
        (e = cudaMemsetAsync(m->slots, 0, 4 * V, s)) ||
        (e = cudaMemsetAsync(m->finished, 0, 4 * V, s)) ||
        (e = cudaMemsetAsync(m->shard_q, 0, 4 * V * D, s)) ||
        (e = cudaMemcpyAsync(m->error, &zero, 4, cudaMemcpyHostToDevice, s)) ||
        (nq > 0 && ((e = cudaMemcpyAsync(m->q_group, q_group_host, 4 * (size_t)nq,
                                          cudaMemcpyHostToDevice, s)) ||
                    (e = cudaMemcpyAsync(m->q_tokens, q_tokens_host, 4 * (size_t)nq,
                                         cudaMemcpyHostToDevice, s))))) {
        fate_mirror_destroy(m);
        return cuda_fail(e, "fate_mirror_create: init");
    }
    if (V > 0) {
        fate_mirror_init_kernel<<<(unsigned)((V + 127) / 128), 128, 0, s>>>(
            (int)V, bank->par_ptr, off, m->remaining);
        fate_internal_count_launches(1);
    }
    // host-side staging values above are stack/vector memory: finish the copies
    if ((e = cudaStreamSynchronize(s)) != cudaSuccess) {
        fate_mirror_destroy(m);
        return cuda_fail(e, "fate_mirror_create: sync");
    }
    *out = m;
    return 0;
}

int fate_mirror_destroy(fate_mirror* m) {
    if (!m) return 0;
    void* ps[] = {m->scen_inst, m->scen_clock, m->scen_loc_off, m->scen_done_level, m->loc,
                  m->residency, m->dev_free, m->kappa_n, m->kappa, m->status, m->running,
                  m->slots, m->finished, m->remaining, m->shard_q, m->q_group, m->q_tokens,
                  m->error, m->ready_n, m->ev, m->evq};
    for (void* p : ps)
        if (p) cudaFree(p);
    delete m;
    return 0;
}

int fate_mirror_apply(fate_mirror* m, const fate_event* events, int32_t n_events,
                      const int32_t* event_queries, int32_t n_event_queries, void* stream) {
    if (!m || n_events < 0 || n_event_queries < 0 || (n_events > 0 && !events))
        return fate_internal_fail(FATE_EINVAL, "fate_mirror_apply: bad arguments");
    if (n_events == 0) return 0;
    cudaError_t e;
    const size_t eb = sizeof(fate_event) * (size_t)n_events;
    if (eb > m->ev_cap) {
        if (m->ev) cudaFree(m->ev);
        m->ev = nullptr;
        if ((e = cudaMalloc(&m->ev, 2 * eb)) != cudaSuccess) return cuda_fail(e, "fate_mirror_apply");
        m->ev_cap = 2 * eb;
    }
    const size_t qb = 4 * (size_t)(n_event_queries > 0 ? n_event_queries : 1);
    if (qb > m->evq_cap) {
        if (m->evq) cudaFree(m->evq);
        m->evq = nullptr;
        if ((e = cudaMalloc((void**)&m->evq, 2 * qb)) != cudaSuccess)
            return cuda_fail(e, "fate_mirror_apply");
        m->evq_cap = 2 * qb;
    }
    cudaStream_t s = static_cast<cudaStream_t>(stream);
    if ((e = cudaMemcpyAsync(m->ev, events, eb, cudaMemcpyHostToDevice, s)) ||
        (n_event_queries > 0 &&
         (e = cudaMemcpyAsync(m->evq, event_queries, 4 * (size_t)n_event_queries,
                              cudaMemcpyHostToDevice, s))))
        return cuda_fail(e, "fate_mirror_apply: H2D");
    fate_mirror_apply_kernel<<<1, 32, 0, s>>>(args_of(m), static_cast<const fate_event*>(m->ev),
                                               n_events, m->evq);
    fate_internal_count_launches(1);
    e = cudaGetLastError();
    return e == cudaSuccess ? 0 : cuda_fail(e, "fate_mirror_apply_kernel");
}

int fate_mirror_state(const fate_mirror* m, fate_state* out) {
    if (!m || !out) return fate_internal_fail(FATE_EINVAL, "fate_mirror_state: NULL");
    out->n_scenarios = 1;
    out->kappa_cap = m->cap;
    out->scen_inst = m->scen_inst;
    out->scen_clock = m->scen_clock;
    out->scen_loc_off = m->scen_loc_off;
    out->scen_done_level = m->scen_done_level;
    // fate_score indexes loc by global stage index minus the instance offset
    out->loc = m->loc;
    out->residency = m->residency;
    out->dev_free = m->dev_free;
    out->kappa_n = m->kappa_n;
    out->kappa = m->kappa;
    return 0;
}

int fate_mirror_ready(fate_mirror* m, int32_t* out_dev, int32_t* n_out, void* stream) {
    if (!m || !out_dev || !n_out) return fate_internal_fail(FATE_EINVAL, "fate_mirror_ready: NULL");
    cudaStream_t s = static_cast<cudaStream_t>(stream);
    cudaError_t e;
    int32_t err = 0;
    if ((e = cudaMemcpyAsync(&err, m->error, 4, cudaMemcpyDeviceToHost, s)) ||
        (e = cudaMemsetAsync(m->ready_n, 0, 4, s)))
        return cuda_fail(e, "fate_mirror_ready");
    if (m->V > 0) {
        fate_mirror_ready_kernel<<<(unsigned)((m->V + 127) / 128), 128, 0, s>>>(
            m->V, m->stage_off, m->status, m->running, m->remaining, out_dev, m->ready_n);
        fate_internal_count_launches(1);
    }
    if ((e = cudaMemcpyAsync(n_out, m->ready_n, 4, cudaMemcpyDeviceToHost, s)) ||
        (e = cudaStreamSynchronize(s)) != cudaSuccess)
        return cuda_fail(e, "fate_mirror_ready");
    if (err == E_KAPPA)
        return fate_internal_fail(FATE_ETOOBIG, "fate_mirror: prefix entries exceed kappa_cap");
    if (err != E_OK) return fate_internal_fail(FATE_EINVAL, "fate_mirror: event out of range");
    return 0;
}

}  // extern "C"
