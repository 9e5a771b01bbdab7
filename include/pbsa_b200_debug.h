/*
 * pbsa_b200_debug.h -- test / experiment hooks of libpbsa_b200.so.  NOT part of the drop-in boundary
 * (include/pbsa_b200.h): nothing a production caller of the PBSA ops needs, kept out of the public
 * header so the operator API stays exactly the reference's.  Used by tests/ and tools/ only.
 */
#ifndef PBSA_B200_DEBUG_H
#define PBSA_B200_DEBUG_H

#include "pbsa_b200.h"

#ifdef __cplusplus
extern "C" {
#endif

/* One 128-row query tile against one 64-row KV slot through the tcgen05 path.
 * q [128][d], k/v [64][d] bf16 (device); s_out [128][64] f32 = q k^T; o_out [128][d] f32 =
 * bf16(s_out) v.  Validates descriptors / TMEM layouts. */
int pbsa_debug_tile(const void* q, const void* k, const void* v, int d, float* s_out,
                    float* o_out, void* stream);

/* Fault injection for negative controls (`verify --fault drop-sink`): "drop-sink" makes
 * K4 rank the sink blocks together with the dynamic candidates (sinks can then be evicted by Top-C,
 * violating the sink-retention rule of SPEC.md:204,228), "" / NULL clears it.  Process-wide; affects
 * every later pbsa_mem_commit.  PBSA_EINVAL for an unknown fault name. */
int pbsa_debug_set_fault(const char* name);

/* Handshake-timeline stamps of CTA 0 (builds with -DPBSA_K3_TRACE only; tools/k3_timeline.py,
 * tools/bwd_timeline.py).  NULL turns them off. */
void pbsa_debug_trace_buffer(void* buf);
void pbsa_debug_bwd_trace_buffer(void* buf);

#ifdef __cplusplus
}
#endif
#endif /* PBSA_B200_DEBUG_H */
