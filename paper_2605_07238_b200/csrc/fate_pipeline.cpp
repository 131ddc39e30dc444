// fate_pipeline.cpp -- the host-buffer entry of the scorer (native, C ABI).
//
// The reference's consumer hands the scorer HOST objects and reads HOST
// results (wfsched.planner.build_problem -> FrontierProblem, planner.py:75-98).
// fate_pipeline_score is that boundary for a whole batch: per-scenario state
// and the work list come from (pinned) host memory in the wire format of
// fate.h (fixed-size scenario records, loc rows, 16-byte items -- any
// scenario range is one contiguous copy), Psi / S / completion go back to
// host memory, and the static bank stays resident in HBM.
//
// The batch is cut into scenario-aligned chunks.  All H2D copies go on one
// stream, back to back; each chunk's scoring waits only for its own inputs
// (event), and its D2H copies, on a third stream, only for its scoring; so
// the H2D copy of chunk i+1, the scoring of chunk i and the D2H copy of chunk
// i-1 overlap (two copy engines + the SMs) with no false stream ordering
// between a D2H and a later H2D.  A
// chunk costs three H2D copies, one unpack launch (wire records -> the
// fate_state SoA the scoring kernels read), one scoring launch and one D2H
// copy per output: every copy-engine transfer has a fixed ~2 us setup cost,
// so the copy count per chunk, not the byte count, is what limits chunking.
#include <cuda_runtime.h>

#include <algorithm>
#include <cstdio>
#include <cstdlib>
#include <cstdint>
#include <cstring>
#include <string>
#include <vector>

#include <nvtx3/nvToolsExt.h>

#include "fate.h"
#include "fate_internal.h"

struct fate_pipeline {
    int device = 0;
    int n_chunks = 8;
    size_t h2d_bytes = 0, d2h_bytes = 0;  // of the last fate_pipeline_score call
    // streams[0] = H2D copies, streams[1] = D2H copies, streams[2..] = scoring
    std::vector<cudaStream_t> streams;
    std::vector<cudaEvent_t> done;      // per stream: joined into the caller's stream
    std::vector<cudaEvent_t> in_ready;  // per chunk: its H2D copies landed
    std::vector<cudaEvent_t> scored;    // per chunk: its scoring launch finished
    cudaEvent_t start = nullptr;
    std::vector<int> qslots;  // reserved ticket-queue slot per compute stream
    // captured graph of the last fate_pipeline_capture (replayed as a whole)
    cudaStream_t cap = nullptr;
    cudaGraphExec_t exec = nullptr;
    long long launches_per_replay = 0;
    bool invalidated = false;  // a later call outgrew the captured workspaces
    // device workspaces (grown on demand): wire-format staging + the SoA the
    // kernels read
    struct Buf {
        void* p = nullptr;
        size_t cap = 0;
    };
    Buf rec, items, loc8, scen_inst, scen_clock, scen_loc_off, scen_done_level, loc, residency,
        dev_free, kappa_n, kappa, w_scen, w_stage, w_psi_off, psi, sched, completion;
    std::vector<Buf*> all() {
        return {&rec, &items, &loc8, &scen_inst, &scen_clock, &scen_loc_off, &scen_done_level, &loc,
                &residency, &dev_free, &kappa_n, &kappa, &w_scen, &w_stage, &w_psi_off, &psi,
                &sched, &completion};
    }
};

namespace {

int cuda_fail(cudaError_t e, const char* what) {
    return fate_internal_fail((int)e, std::string(what) + ": " + cudaGetErrorString(e));
}

int grow(fate_pipeline* p, fate_pipeline::Buf& b, size_t bytes) {
    if (bytes <= b.cap) return 0;
    if (p->exec) {
        // a captured graph addresses the old workspaces: it must be recaptured
        cudaGraphExecDestroy(p->exec);
        p->exec = nullptr;
        p->invalidated = true;
    }
    if (b.p) cudaFree(b.p);
    b.p = nullptr;
    b.cap = 0;
    const size_t want = std::max<size_t>(bytes + bytes / 4, 256);
    cudaError_t e = cudaMalloc(&b.p, want);
    if (e != cudaSuccess) return cuda_fail(e, "fate_pipeline: cudaMalloc");
    b.cap = want;
    return 0;
}

struct Copy {
    void* dst;
    const void* src;
    size_t bytes;
};

}  // namespace

extern "C" {

int fate_pipeline_create(int device, int n_chunks, int n_streams, fate_pipeline** out) {
    if (!out) return fate_internal_fail(FATE_EINVAL, "fate_pipeline_create: out is NULL");
    if (n_chunks < 1 || n_streams < 1 || n_chunks > 1024 || n_streams > 16)
        return fate_internal_fail(FATE_EINVAL, "fate_pipeline_create: bad chunk/stream count");
    cudaError_t e = cudaSetDevice(device);
    if (e != cudaSuccess) return cuda_fail(e, "fate_pipeline_create: cudaSetDevice");
    auto* p = new fate_pipeline();
    p->device = device;
    p->n_chunks = n_chunks;
    p->streams.resize(2 + n_streams);
    p->done.resize(2 + n_streams);
    for (int i = 0; i < 2 + n_streams; ++i) {
        if ((e = cudaStreamCreateWithFlags(&p->streams[i], cudaStreamNonBlocking)) != cudaSuccess ||
            (e = cudaEventCreateWithFlags(&p->done[i], cudaEventDisableTiming)) != cudaSuccess) {
            fate_pipeline_destroy(p);
            return cuda_fail(e, "fate_pipeline_create");
        }
    }
    for (int i = 0; i < n_streams; ++i) p->qslots.push_back(fate_internal_reserve_queue_slot());
    p->in_ready.resize(n_chunks);
    p->scored.resize(n_chunks);
    for (int i = 0; i < n_chunks; ++i) {
        if ((e = cudaEventCreateWithFlags(&p->in_ready[i], cudaEventDisableTiming)) != cudaSuccess ||
            (e = cudaEventCreateWithFlags(&p->scored[i], cudaEventDisableTiming)) != cudaSuccess) {
            fate_pipeline_destroy(p);
            return cuda_fail(e, "fate_pipeline_create");
        }
    }
    if ((e = cudaEventCreateWithFlags(&p->start, cudaEventDisableTiming)) != cudaSuccess) {
        fate_pipeline_destroy(p);
        return cuda_fail(e, "fate_pipeline_create");
    }
    *out = p;
    return 0;
}

int fate_pipeline_destroy(fate_pipeline* p) {
    if (!p) return 0;
    int prev = 0;
    cudaGetDevice(&prev);
    cudaSetDevice(p->device);
    for (auto s : p->streams)
        if (s) cudaStreamSynchronize(s);
    for (auto* b : p->all())
        if (b->p) cudaFree(b->p);
    for (auto s : p->streams)
        if (s) cudaStreamDestroy(s);
    for (auto* v : {&p->done, &p->in_ready, &p->scored})
        for (auto ev : *v)
            if (ev) cudaEventDestroy(ev);
    if (p->start) cudaEventDestroy(p->start);
    if (p->exec) cudaGraphExecDestroy(p->exec);
    for (int q : p->qslots) fate_internal_release_queue_slot(q);
    if (p->cap) cudaStreamDestroy(p->cap);
    cudaSetDevice(prev);
    delete p;
    return 0;
}

}  // extern "C"

namespace {

enum class Mode { direct, size_only, capture };

// Validates the batch, sizes the workspaces and enqueues the chunked
// H2D -> unpack -> score -> D2H pipeline after the work on `caller` (which
// then waits for all of it).  Used directly (fate_pipeline_score) or under
// stream capture (fate_pipeline_capture).
int enqueue(fate_pipeline* p, const fate_bank* bank, const fate_weights* w,
            const fate_windows* win, const fate_derived* der, const fate_host_batch* hb,
            double* psi_host, double* sched_host, double* completion_host, cudaStream_t caller,
            Mode mode) {
    const bool capturing = mode == Mode::capture;
    if (!p || !bank || !hb || !psi_host)
        return fate_internal_fail(FATE_EINVAL, "fate_pipeline_score: NULL argument");
    const int D = bank->n_devices;
    const int S = hb->n_scenarios;
    const int W = hb->n_items;
    const int cap = hb->kappa_cap;
    if (D < 1 || D > FATE_MAX_DEVICES || S < 0 || W < 0 || cap < 1 || cap > FATE_MAX_KAPPA ||
        hb->n_loc < 0 || hb->n_psi < 0)
        return fate_internal_fail(FATE_EINVAL, "fate_pipeline_score: bad sizes");
    if (W == 0) return 0;
    if (!hb->scen_rec || !hb->items || (hb->n_loc > 0 && !hb->loc))
        return fate_internal_fail(FATE_EINVAL, "fate_pipeline_score: NULL batch array");
    const size_t RB = FATE_SCEN_REC_BYTES(D, cap);
    const fate_item* it = hb->items;
    {
        // branch-free pass (this runs on the host before any copy is enqueued)
        unsigned bad = (unsigned)it[0].scen >= (unsigned)S;
        for (int i = 1; i < W; ++i)
            bad |= ((unsigned)it[i].scen >= (unsigned)S) | (it[i].scen < it[i - 1].scen) |
                   (it[i].psi_off < it[i - 1].psi_off);
        if (bad)
            return fate_internal_fail(FATE_EINVAL,
                                      "fate_pipeline_score: items must be scenario-major (scenario "
                                      "in range), psi_off non-decreasing");
    }
    // psi_off == n_psi is a trailing item without candidates (no eligible
    // device); the device Psi workspace carries 64 * D slack entries past
    // n_psi, so even an item whose bound the host cannot see (the bank is
    // device-resident) never writes outside the workspace -- only [0, n_psi)
    // is copied back
    if (it[0].psi_off < 0 || it[W - 1].psi_off > hb->n_psi)
        return fate_internal_fail(FATE_EINVAL, "fate_pipeline_score: psi_off out of range");
    const auto loc_off = [&](int s) -> int64_t {
        int64_t v;
        std::memcpy(&v, (const char*)hb->scen_rec + (size_t)s * RB + 8, 8);
        return v;
    };
    for (int s = 0; s < S; ++s) {
        const int64_t o = loc_off(s);
        if (o < 0 || o > hb->n_loc || (s > 0 && o < loc_off(s - 1)))
            return fate_internal_fail(FATE_EINVAL,
                                      "fate_pipeline_score: loc_off must be nondecreasing, in range");
    }
    p->h2d_bytes = 0;
    p->d2h_bytes = 0;

    int rc;
    if ((rc = grow(p, p->rec, RB * (size_t)S)) || (rc = grow(p, p->items, 16 * (size_t)W)) ||
        (rc = grow(p, p->scen_inst, 4 * (size_t)S)) || (rc = grow(p, p->scen_clock, 8 * (size_t)S)) ||
        (rc = grow(p, p->scen_loc_off, 8 * (size_t)S)) ||
        (rc = grow(p, p->scen_done_level, 4 * (size_t)S)) ||
        (rc = grow(p, p->loc, 4 * (size_t)hb->n_loc)) || (rc = grow(p, p->loc8, (size_t)hb->n_loc)) ||
        (rc = grow(p, p->residency, 4 * (size_t)S * D)) ||
        (rc = grow(p, p->dev_free, 8 * (size_t)S * D)) || (rc = grow(p, p->kappa_n, 4 * (size_t)S * D)) ||
        (rc = grow(p, p->kappa, 16 * (size_t)S * D * cap)) || (rc = grow(p, p->w_scen, 4 * (size_t)W)) ||
        (rc = grow(p, p->w_stage, 4 * (size_t)W)) || (rc = grow(p, p->w_psi_off, 8 * (size_t)W)) ||
        (rc = grow(p, p->psi, 8 * ((size_t)hb->n_psi + 64 * (size_t)D))))
        return rc;
    if (sched_host && (rc = grow(p, p->sched, 8 * (size_t)W * D))) return rc;
    if (completion_host && (rc = grow(p, p->completion, 8 * (size_t)W * D))) return rc;
    if (mode == Mode::size_only) return 0;

    fate_state dst{};
    dst.n_scenarios = S;
    dst.kappa_cap = cap;
    dst.scen_inst = (const int32_t*)p->scen_inst.p;
    dst.scen_clock = (const double*)p->scen_clock.p;
    dst.scen_loc_off = (const int64_t*)p->scen_loc_off.p;
    dst.scen_done_level = (const int32_t*)p->scen_done_level.p;
    dst.loc = (const int32_t*)p->loc.p;
    dst.residency = (const int32_t*)p->residency.p;
    dst.dev_free = (const double*)p->dev_free.p;
    dst.kappa_n = (const int32_t*)p->kappa_n.p;
    dst.kappa = (const int32_t*)p->kappa.p;
    fate_out dout{};
    dout.psi = (double*)p->psi.p;
    dout.sched = sched_host ? (double*)p->sched.p : nullptr;
    dout.completion = completion_host ? (double*)p->completion.p : nullptr;
    dout.tail = nullptr;

    // scenario-aligned chunk boundaries (even split; measured on B200: uneven
    // first chunks did not help, the D2H stream is the bound either way)
    std::vector<int> bounds{0};
    for (int c = 1; c < p->n_chunks; ++c) {
        int i = (int)(((long long)W * c) / p->n_chunks);
        while (i > 0 && i < W && it[i].scen == it[i - 1].scen) ++i;
        if (i > bounds.back() && i < W) bounds.push_back(i);
    }
    bounds.push_back(W);

    // FATE_PIPE_TRACE=1 (-DFATE_AB experiment builds only): per-chunk timeline
    // on stderr (diagnostic; synchronizes)
#ifdef FATE_AB
    static const bool trace_env = getenv("FATE_PIPE_TRACE") != nullptr;
#else
    constexpr bool trace_env = false;
#endif
    const bool trace = trace_env && !capturing;
    std::vector<cudaEvent_t> tev;
    const auto mark = [&](cudaStream_t st) {
        if (!trace) return;
        cudaEvent_t ev;
        cudaEventCreate(&ev);
        cudaEventRecord(ev, st);
        tev.push_back(ev);
    };
    mark(caller);
    if (trace) {
        for (const void* hp : {(const void*)psi_host, hb->scen_rec, (const void*)hb->items}) {
            cudaPointerAttributes at{};
            cudaError_t pe = cudaPointerGetAttributes(&at, hp);
            fprintf(stderr, "[fate_pipeline] host ptr %p: type %d (%s)\n", hp, (int)at.type,
                    cudaGetErrorString(pe));
        }
    }
    cudaError_t e = cudaEventRecord(p->start, caller);
    if (e != cudaSuccess) return cuda_fail(e, "fate_pipeline_score: record");
    for (auto s : p->streams)
        if ((e = cudaStreamWaitEvent(s, p->start, 0)) != cudaSuccess)
            return cuda_fail(e, "fate_pipeline_score: wait");

    char* drec = (char*)p->rec.p;
    // Three passes, in this host order: every H2D copy, then every scoring
    // launch, then every D2H copy.  Copy engines are fed from shared hardware
    // queues: a D2H enqueued before a later chunk's H2D would sit at the head
    // of its queue waiting for its scoring event and hold that H2D back
    // (measured: each chunk's inputs then landed only after the previous
    // chunk's kernel).  Dependencies are per chunk (events), so chunk i's
    // scoring still starts as soon as its own inputs land.
    struct Chunk {
        int i0, i1, sa, sb;
        int64_t l0, l1, p0, p1;
    };
    std::vector<Chunk> ch;
    for (size_t c = 0; c + 1 < bounds.size(); ++c) {
        Chunk k;
        k.i0 = bounds[c];
        k.i1 = bounds[c + 1];
        // only the scenarios this chunk's items read travel
        k.sa = it[k.i0].scen;
        k.sb = it[k.i1 - 1].scen + 1;
        k.l0 = loc_off(k.sa);
        k.l1 = k.sb < S ? loc_off(k.sb) : hb->n_loc;
        k.p0 = it[k.i0].psi_off;
        k.p1 = k.i1 < W ? it[k.i1].psi_off : hb->n_psi;
        ch.push_back(k);
    }
    cudaStream_t sh = p->streams[0], sd = p->streams[1];
    const auto comp = [&](size_t c) { return p->streams[2 + c % (p->streams.size() - 2)]; };
    nvtxRangePushA("fate_pipeline:h2d");
    for (size_t c = 0; c < ch.size(); ++c) {
        const Chunk& k = ch[c];
        const Copy h2d[] = {
            {drec + RB * k.sa, (const char*)hb->scen_rec + RB * k.sa, RB * (size_t)(k.sb - k.sa)},
            {(int8_t*)p->loc8.p + k.l0, hb->loc + k.l0, (size_t)(k.l1 - k.l0)},
            {(fate_item*)p->items.p + k.i0, it + k.i0, 16 * (size_t)(k.i1 - k.i0)},
        };
        for (const Copy& cp : h2d) {
            if (cp.bytes == 0) continue;
            if ((e = cudaMemcpyAsync(cp.dst, cp.src, cp.bytes, cudaMemcpyHostToDevice, sh)) !=
                cudaSuccess)
                return cuda_fail(e, "fate_pipeline_score: H2D");
            p->h2d_bytes += cp.bytes;
        }
        mark(sh);
        if ((e = cudaEventRecord(p->in_ready[c], sh)) != cudaSuccess)
            return cuda_fail(e, "fate_pipeline_score: H2D event");
    }
    nvtxRangePop();
    nvtxRangePushA("fate_pipeline:score");
    for (size_t c = 0; c < ch.size(); ++c) {
        const Chunk& k = ch[c];
        cudaStream_t s = comp(c);
        if ((e = cudaStreamWaitEvent(s, p->in_ready[c], 0)) != cudaSuccess)
            return cuda_fail(e, "fate_pipeline_score: H2D wait");
        mark(s);
        if ((rc = fate_internal_unpack(drec, (size_t)RB, k.sa, k.sb, D, cap,
                                       (const fate_item*)p->items.p, k.i0, k.i1,
                                       (const int8_t*)p->loc8.p, k.l0, k.l1, &dst,
                                       (int32_t*)p->w_scen.p, (int32_t*)p->w_stage.p,
                                       (int64_t*)p->w_psi_off.p, s)))
            return rc;
        fate_work cw{};
        cw.n_items = k.i1 - k.i0;
        cw.scen = (const int32_t*)p->w_scen.p + k.i0;
        cw.stage = (const int32_t*)p->w_stage.p + k.i0;
        cw.psi_off = (const int64_t*)p->w_psi_off.p + k.i0;
        // per-item output rows are indexed by the chunk-local item, Psi by psi_off
        fate_out co = dout;
        if (co.sched) co.sched += (size_t)k.i0 * D;
        if (co.completion) co.completion += (size_t)k.i0 * D;
        mark(s);
        fate_internal_set_queue_slot(p->qslots[c % p->qslots.size()]);
        rc = fate_score(bank, w, win, der, &dst, &cw, &co, s);
        fate_internal_set_queue_slot(-1);
        if (rc) return rc;
        mark(s);
        if ((e = cudaEventRecord(p->scored[c], s)) != cudaSuccess)
            return cuda_fail(e, "fate_pipeline_score: score event");
    }
    nvtxRangePop();
    nvtxRangePushA("fate_pipeline:d2h");
    for (size_t c = 0; c < ch.size(); ++c) {
        const Chunk& k = ch[c];
        const size_t ni = (size_t)(k.i1 - k.i0);
        if ((e = cudaStreamWaitEvent(sd, p->scored[c], 0)) != cudaSuccess)
            return cuda_fail(e, "fate_pipeline_score: score wait");
        const Copy d2h[] = {
            {psi_host + k.p0, (const double*)p->psi.p + k.p0, 8 * (size_t)(k.p1 - k.p0)},
            {sched_host ? sched_host + (size_t)k.i0 * D : nullptr,
             dout.sched ? dout.sched + (size_t)k.i0 * D : nullptr, 8 * ni * D},
            {completion_host ? completion_host + (size_t)k.i0 * D : nullptr,
             dout.completion ? dout.completion + (size_t)k.i0 * D : nullptr, 8 * ni * D},
        };
        for (const Copy& cp : d2h) {
            if (!cp.dst || cp.bytes == 0) continue;
            if ((e = cudaMemcpyAsync(cp.dst, cp.src, cp.bytes, cudaMemcpyDeviceToHost, sd)) !=
                cudaSuccess)
                return cuda_fail(e, "fate_pipeline_score: D2H");
            p->d2h_bytes += cp.bytes;
        }
        mark(sd);
    }
    nvtxRangePop();
    if (trace) {
        cudaDeviceSynchronize();
        fprintf(stderr, "[fate_pipeline] chunk: h2d_end unpack_start score_start score_end d2h_end (us)\n");
        // marks: [0] origin, then nc H2D ends, then 3 per chunk (unpack,
        // score start, score end), then nc D2H ends
        const size_t nc = ch.size();
        for (size_t c = 0; c < nc; ++c) {
            const size_t idx[5] = {1 + c, 1 + nc + 3 * c, 2 + nc + 3 * c, 3 + nc + 3 * c,
                                   1 + 4 * nc + c};
            float t[5];
            for (int k = 0; k < 5; ++k) cudaEventElapsedTime(&t[k], tev[0], tev[idx[k]]);
            fprintf(stderr, "[fate_pipeline] %zu: %.1f %.1f %.1f %.1f %.1f\n", c, 1e3 * t[0],
                    1e3 * t[1], 1e3 * t[2], 1e3 * t[3], 1e3 * t[4]);
        }
        for (auto ev : tev) cudaEventDestroy(ev);
    }
    for (size_t i = 0; i < p->streams.size(); ++i) {
        if ((e = cudaEventRecord(p->done[i], p->streams[i])) != cudaSuccess ||
            (e = cudaStreamWaitEvent(caller, p->done[i], 0)) != cudaSuccess)
            return cuda_fail(e, "fate_pipeline_score: join");
    }
    return 0;
}

}  // namespace

extern "C" {

int fate_pipeline_score(fate_pipeline* p, const fate_bank* bank, const fate_weights* w,
                        const fate_windows* win, const fate_derived* der,
                        const fate_host_batch* hb, double* psi_host, double* sched_host,
                        double* completion_host, void* stream) {
    return enqueue(p, bank, w, win, der, hb, psi_host, sched_host, completion_host,
                   static_cast<cudaStream_t>(stream), Mode::direct);
}

int fate_pipeline_capture(fate_pipeline* p, const fate_bank* bank, const fate_weights* w,
                          const fate_windows* win, const fate_derived* der,
                          const fate_host_batch* hb, double* psi_host, double* sched_host,
                          double* completion_host) {
    if (!p) return fate_internal_fail(FATE_EINVAL, "fate_pipeline_capture: NULL handle");
    if (p->exec) {
        cudaGraphExecDestroy(p->exec);
        p->exec = nullptr;
    }
    p->invalidated = false;
    cudaError_t e;
    if (!p->cap && (e = cudaStreamCreateWithFlags(&p->cap, cudaStreamNonBlocking)) != cudaSuccess)
        return cuda_fail(e, "fate_pipeline_capture: stream");
    // workspaces are (re)allocated outside the capture: validate and size them
    // with a pass that enqueues nothing (W == 0 batches capture nothing)
    int rc0 = enqueue(p, bank, w, win, der, hb, psi_host, sched_host, completion_host, p->cap,
                      Mode::size_only);
    if (rc0) return rc0;
    if (hb->n_items == 0) return 0;
    if ((e = cudaStreamBeginCapture(p->cap, cudaStreamCaptureModeThreadLocal)) != cudaSuccess)
        return cuda_fail(e, "fate_pipeline_capture: begin");
    const long long before = fate_internal_launches();
    int rc = enqueue(p, bank, w, win, der, hb, psi_host, sched_host, completion_host, p->cap,
                     Mode::capture);
    p->launches_per_replay = fate_internal_launches() - before;
    fate_internal_count_launches(-p->launches_per_replay);  // counted when replayed
    cudaGraph_t g = nullptr;
    e = cudaStreamEndCapture(p->cap, &g);
    if (rc) {
        if (g) cudaGraphDestroy(g);
        return rc;
    }
    if (e != cudaSuccess) return cuda_fail(e, "fate_pipeline_capture: end");
    e = cudaGraphInstantiate(&p->exec, g, 0);
    cudaGraphDestroy(g);
    if (e != cudaSuccess) return cuda_fail(e, "fate_pipeline_capture: instantiate");
    return 0;
}

int fate_pipeline_replay(fate_pipeline* p, void* stream) {
    if (!p || !p->exec)
        return fate_internal_fail(FATE_ENOTREADY,
                                  p && p->invalidated
                                      ? "fate_pipeline_replay: workspaces reallocated by a larger "
                                        "batch since the capture; capture again"
                                      : "fate_pipeline_replay: nothing captured");
    cudaError_t e = cudaGraphLaunch(p->exec, static_cast<cudaStream_t>(stream));
    if (e != cudaSuccess) return cuda_fail(e, "fate_pipeline_replay");
    fate_internal_count_launches(p->launches_per_replay);
    return 0;
}

int fate_pipeline_bytes(const fate_pipeline* p, int64_t* h2d, int64_t* d2h) {
    if (!p || !h2d || !d2h) return fate_internal_fail(FATE_EINVAL, "fate_pipeline_bytes: NULL");
    *h2d = (int64_t)p->h2d_bytes;
    *d2h = (int64_t)p->d2h_bytes;
    return 0;
}

int fate_pipeline_device_psi(const fate_pipeline* p, const double** psi_dev) {
    if (!p || !psi_dev) return fate_internal_fail(FATE_EINVAL, "fate_pipeline_device_psi: NULL");
    if (!p->psi.p) return fate_internal_fail(FATE_ENOTREADY, "fate_pipeline_device_psi: no run yet");
    *psi_dev = (const double*)p->psi.p;
    return 0;
}

}  // extern "C"
