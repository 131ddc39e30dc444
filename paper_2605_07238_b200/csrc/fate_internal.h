// fate_internal.h -- shared by the library's translation units (not ABI).
#ifndef FATE_INTERNAL_H
#define FATE_INTERNAL_H
#include <cuda_runtime.h>

#include <cstddef>
#include <string>

#include "fate.h"

// Records msg as fate_last_error() and returns code.
int fate_internal_fail(int code, const std::string& msg);

// Library-wide kernel launch counter (fate_launch_count).
long long fate_internal_launches();
void fate_internal_count_launches(long long n);

// v6 ticket-queue slots: reserve one for a pipeline compute stream (-1 when
// none is left), release it, and select the slot of this thread's next
// scoring launch (-1 = the rotating direct-launch slots).
int fate_internal_reserve_queue_slot();
void fate_internal_release_queue_slot(int slot);
void fate_internal_set_queue_slot(int slot);

// Scatter wire-format scenario records [s0, s1) and items [i0, i1) (device
// copies of fate_host_batch) into the fate_state / fate_work SoA of dst.
// Wire loc rows [l0, l1) (int8) are widened into dst->loc.
int fate_internal_unpack(const void* rec, size_t rec_bytes, int s0, int s1, int D, int cap,
                         const fate_item* items, int i0, int i1, const int8_t* loc8, int64_t l0,
                         int64_t l1, const fate_state* dst, int32_t* w_scen, int32_t* w_stage,
                         int64_t* w_psi_off, cudaStream_t s);

#endif
