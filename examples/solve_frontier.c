/* solve_frontier.c -- the C ABI from plain C, no Python (host-only entry
 * points, so it runs on a machine without a GPU).
 *
 *   gcc -std=c11 -I include examples/solve_frontier.c \
 *       -L paper_2605_07238_b200 -lfate -Wl,-rpath,$PWD/paper_2605_07238_b200 \
 *       -o /tmp/solve_frontier && /tmp/solve_frontier
 *
 * Builds the three-stage frontier below in the fate_frontier CSR layout
 * (stage -> slot rows -> candidates, devices ascending within a slot, the
 * order the reference's _stage_options visits them, planner.py:101-147) and
 * solves it with fate_solve_frontier, the native wfsched.planner.solve_frontier
 * (planner.py:150-214).  Prints one line:
 *   abi=<v> n=<k> sel=<stage:slot:device,...> objective=<x> optimal=<0|1> nodes=<n>
 */
#include <stdint.h>
#include <stdio.h>

#include "fate.h"

int main(void) {
    /* stage 0: slot 0 on d0 (5.0) / d1 (3.0); slot 1 on d0 (0.5) / d1 (0.25)
     * stage 1: slot 0 on d0 (4.0) / d1 (6.0)
     * stage 2: slot 0 on d2 only (-1.0: a negative option is never kept) */
    const int32_t slot_ptr[] = {0, 2, 3, 4};
    const int32_t cand_ptr[] = {0, 2, 4, 6, 7};
    const int32_t cand_dev[] = {0, 1, 0, 1, 0, 1, 2};
    const double cand_psi[] = {5.0, 3.0, 0.5, 0.25, 4.0, 6.0, -1.0};
    fate_frontier fr = {3, 3, slot_ptr, cand_ptr, cand_dev, cand_psi};
    int32_t st[3], sl[3], dv[3];
    fate_selection out = {0};
    out.capacity = 3;
    out.stage = st;
    out.slot = sl;
    out.device = dv;
    const int rc = fate_solve_frontier(&fr, 0.25, 0, &out);
    if (rc != 0) {
        fprintf(stderr, "fate_solve_frontier: %s (status %d)\n", fate_last_error(), rc);
        return 1;
    }
    printf("abi=%d n=%d sel=", fate_abi_version(), out.n);
    for (int k = 0; k < out.n; ++k) printf("%s%d:%d:%d", k ? "," : "", st[k], sl[k], dv[k]);
    printf(" objective=%.17g optimal=%d nodes=%lld\n", out.objective, out.optimal,
           (long long)out.nodes);
    return 0;
}
