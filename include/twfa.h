/* twfa.h -- C ABI of the B200 (sm_100a) executor for Twill schedules.
 *
 * Drop-in boundary. The reference (weftsched, /root/reference/proj) exposes
 * its scheduler as C++ (the headers under include/weftsched/), a CLI (`weftsched joint |
 * codegen | sim | validate`, src/cli.cpp:376-473) and pybind11 bindings that
 * exchange the SAME JSON documents (bindings/module.cpp:219-249). Its only
 * consumer of a solved schedule is `synthesize` (codegen.cpp:43-189 /
 * codegen.hpp:49), which renders a text listing that the paper then
 * hand-compiled to CUDA. This library is the compiled
 * consumer in that position: it takes the problem JSON and the solution JSON
 * exactly as `weftsched joint` writes them (solution_to_json, cli.cpp:68-94)
 * and executes the loop on the GPU. Nothing here re-solves a schedule.
 *
 * Conventions (mirroring the reference, cli.hpp:11-13, cli.cpp:462-471):
 *   return 0 success, 1 domain error (malformed document, schedule the
 *   executor cannot realize), 2 usage error (bad arguments / unsupported
 *   shape), 3 CUDA error. The message of the last failure on the calling
 *   thread is returned by twfa_last_error(). No C++ exception crosses this
 *   boundary. Plans are immutable after creation and may be shared between
 *   threads and devices; launches are ordered on the caller's stream.
 * Device buffers are caller-owned (raw device pointers, e.g. torch tensors).
 */
#ifndef TWFA_H
#define TWFA_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define TWFA_OK 0
#define TWFA_EDOMAIN 1
#define TWFA_EUSAGE 2
#define TWFA_ECUDA 3

typedef struct twfa_plan twfa_plan;

/* Interface version of this header (bumped on ABI changes). */
int twfa_abi_version(void);

/* Thread-local message of the last failed call ("" after a success). */
const char* twfa_last_error(void);

/* Lower a solved schedule into an executable plan.
 * Replaces the reference consumer chain solution_from_json (cli.cpp:96-155)
 * -> reconstruct (cli.cpp:161-168) -> synthesize (codegen.cpp:43-189):
 * same document checks (unknown keys, M covering every node inside
 * [0, L - eff], streaming rewrite re-applied when streaming_depths is set),
 * same stage / region semantics. On success *out owns the plan. */
int twfa_plan_create(const char* problem_json, const char* solution_json, twfa_plan** out);

/* The reference's schedule checker on a (problem, solution) pair without
 * lowering it: validate_program (sim.cpp:79-311) over the tables
 * expand_solution (sim.cpp:57-77) builds from the reconstructed solution
 * (cli.cpp:161-168), restated. Writes the JSON list [[family, message], ...]
 * the reference's binding returns (bindings/module.cpp:176-184; "[]" when
 * the schedule is exact) into buf (at most cap bytes including the NUL);
 * *needed receives the full size. Returns 1 for malformed documents.
 * twfa_plan_create runs the same checks and rejects any violation. */
int twfa_schedule_validate(const char* problem_json, const char* solution_json, char* buf, size_t cap,
                           size_t* needed);

/* Release a plan (NULL is ignored). */
void twfa_plan_destroy(twfa_plan* plan);

/* JSON description of the lowered plan (I, L, copies, per-node stage, slot
 * and warp, per-warp trip programs, ring depths). Writes at most `cap` bytes
 * including the terminating NUL; *needed receives the full size. Plays the
 * role of emit_listing / program_to_json (codegen.hpp:51-56). */
int twfa_plan_describe(const twfa_plan* plan, char* buf, size_t cap, size_t* needed);

/* Copy the raw device plan (struct TwfaDevicePlan, plan.h) for inspection. */
int twfa_plan_raw(const twfa_plan* plan, void* dst, size_t cap, size_t* needed);

/* FA forward, bf16, head dim 128, on the calling device:
 *   O = softmax(scale * Q K^T [+ causal mask]) V,   lse = log-sum-exp per row.
 * q, k, v, o: [B, H, S, 128] contiguous bf16 device buffers; lse: [B, H, S]
 * fp32 or NULL. causal: key j visible to query i iff j <= i. stream: a
 * cudaStream_t (NULL = legacy default stream). The plan must come from an
 * FA-forward loop problem. Plans with 128-key K/V tiles and an unsplit S run
 * as clusters of two CTAs (tcgen05 cta_group::2; environment TWFA_PAIR=0
 * selects one CTA per work tile, with bit-identical results). */
int twfa_fa_fwd(const twfa_plan* plan, const void* q, const void* k, const void* v, void* o, float* lse,
                int B, int H, int S, int D, int causal, float softmax_scale, void* stream);

/* Same as twfa_fa_fwd, additionally recording the issue trace of CTA 0:
 * per warp w, trace[w * cap * 8] = number of records n, followed by n records
 * of 8 uint32 {node, iteration, trip, t_issue, t_ready, t_done, work tile
 * ordinal, iterations of that work tile} (clock64 low words; device buffer of
 * num_warps * cap * 8 uint32, zeroed by the caller). */
int twfa_fa_fwd_traced(const twfa_plan* plan, const void* q, const void* k, const void* v, void* o,
                       float* lse, int B, int H, int S, int D, int causal, float softmax_scale,
                       uint32_t* trace, uint32_t cap, void* stream);

/* Host-buffer form of twfa_fa_fwd for CPU callers (the reference's C++ host,
 * the CLI, ctypes): synchronous; on return O (and lse) are in the caller's
 * buffers. The (b, h) pairs are streamed in chunks through a pipeline: host
 * -> device copies of chunk i + 1 and device -> host copies of chunk i - 1
 * overlap the kernel on chunk i (three CUDA streams). Page-locked caller
 * buffers (cudaMallocHost / cudaHostRegister) are DMA'd directly; pageable
 * ones are staged through pinned slots by host threads. Device buffers,
 * pinned slots and streams are cached per calling thread. */
int twfa_fa_fwd_host(const twfa_plan* plan, const uint16_t* q, const uint16_t* k, const uint16_t* v,
                     uint16_t* o, float* lse, int B, int H, int S, int D, int causal, float softmax_scale);

/* FA backward (the paper's second workload), bf16, head
 * dim 128, from an FA-backward plan (problem fa_backward_problem, solved by
 * the reference scheduler):
 *   dQ = scale dS K,  dK = scale dS^T Q,  dV = P^T dO,
 *   P = exp(scale Q K^T - lse),  dS = P (dO V^T - rowsum(dO O)).
 * q, k, v, o, dout, dq, dk, dv: [B, H, S, 128] contiguous bf16 device
 * buffers; lse: [B, H, S] fp32 from the forward (natural log). workspace: a
 * device buffer of at least twfa_fa_bwd_workspace_size(B, H, S, D) bytes
 * (fp32 dQ accumulator and rowsum(dO O)); contents are overwritten. */
int twfa_fa_bwd_workspace_size(int B, int H, int S, int D, size_t* bytes);
int twfa_fa_bwd(const twfa_plan* plan, const void* q, const void* k, const void* v, const void* o,
                const void* dout, const float* lse, void* dq, void* dk, void* dv, void* workspace,
                size_t workspace_bytes, int B, int H, int S, int D, int causal, float softmax_scale,
                void* stream);

/* Same as twfa_fa_bwd, additionally recording the issue trace of CTA 0 in
 * the layout of twfa_fa_fwd_traced (records {node, iteration, trip, t_issue,
 * 0, t_done, work item ordinal, Q iterations of that item}). */
int twfa_fa_bwd_traced(const twfa_plan* plan, const void* q, const void* k, const void* v, const void* o,
                       const void* dout, const float* lse, void* dq, void* dk, void* dv, void* workspace,
                       size_t workspace_bytes, int B, int H, int S, int D, int causal, float softmax_scale,
                       uint32_t* trace, uint32_t cap, void* stream);

/* GEMM mainloop plan: C[M,N] = A[M,K] * B[N,K]^T, bf16 in/out, fp32 accumulate.
 * M % 256 == 0, N % 256 == 0, K % 64 == 0 (one CTA pair per 256 x 256 output tile). */
int twfa_gemm(const twfa_plan* plan, const void* a, const void* b, void* c, int M, int N, int K,
              void* stream);

/* Persistent grid size used by the launches (number of SMs of the current device). */
int twfa_grid_size(int* out);

#ifdef __cplusplus
}
#endif
#endif
