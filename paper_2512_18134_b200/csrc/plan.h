// KernelPlan: the lowered form of a Twill joint schedule, consumed by the
// sm_100a kernels. Plain-old-data so it can be passed by value as a kernel
// parameter (__grid_constant__) and copied to the device unchanged.
//
// It is the device-side counterpart of the reference's PipelinedProgram
// (/root/reference/proj/include/weftsched/codegen.hpp:32-42): instead of a
// text listing per region, every hardware warp gets the ordered list of loop
// ops it issues in one steady-state trip, each tagged with its stage
// (M div I, codegen.cpp:63). Trip r of the realized loop runs op v on
// iteration r - stage(v); trips with r < max_stage form the prologue and
// trips past the last iteration the epilogue, so prologue / steady state /
// epilogue are exactly the region split of codegen.cpp:51-52.
#pragma once
#include <stdint.h>

#define TWFA_MAX_NODES 20
#define TWFA_MAX_WARPS 16
#define TWFA_MAX_TILES 2

enum TwfaOpKind : uint8_t {
  TWFA_OP_LDK = 0,  // TMA load of the K tile (streamed, variable latency)
  TWFA_OP_LDV = 1,  // TMA load of the V tile
  TWFA_OP_S = 2,    // S_k = Q_k K^T            (tcgen05.mma, SS, into TMEM)
  TWFA_OP_MX = 3,   // row max of S_k, rescale factor -> correction
  TWFA_OP_EX = 4,   // P_k = exp2(S_k - m), row sum, P -> TMEM (bf16)
  TWFA_OP_CR = 5,   // O_k *= exp2(m_old - m_new)  (TMEM read-modify-write)
  TWFA_OP_PV = 6,   // O_k += P_k V             (tcgen05.mma, TS, into TMEM)
  TWFA_OP_LDA = 7,  // GEMM: TMA load of the A k-block
  TWFA_OP_LDB = 8,  // GEMM: TMA load of the B k-block
  TWFA_OP_MMA = 9,  // GEMM: D += A B^T over one k-block
  // S_k as two N = 64 GEMMs: SA_k (keys 0-63 -> columns 0-63) overwrites only
  // S columns MX_k has already read, SB_k (keys 64-127 -> columns 64-127)
  // the columns P_k (bf16) is aliased over; see fa_forward_problem(split_s)
  TWFA_OP_SA = 10,
  TWFA_OP_SB = 11,
  // FA backward (one 128-key K/V tile per CTA, iterations over 128-row Q
  // tiles; see fa_backward_problem in tools/make_problems.py)
  TWFA_OP_LDQ = 12,  // TMA load of Q_i (streamed)
  TWFA_OP_LDO = 13,  // TMA load of dO_i (streamed)
  TWFA_OP_ST = 14,   // S^T = K Q_i^T           (tcgen05.mma SS)
  TWFA_OP_DP = 15,   // dP^T = V dO_i^T         (tcgen05.mma SS)
  TWFA_OP_EXB = 16,  // P^T = exp2(S^T - LSE_i) -> TMEM (bf16)
  TWFA_OP_DS = 17,   // dS^T = P^T (dP^T - D_i) -> TMEM (bf16) and smem
  TWFA_OP_DV = 18,   // dV += P^T dO_i          (tcgen05.mma TS)
  TWFA_OP_DK = 19,   // dK += dS^T Q_i          (tcgen05.mma TS)
  TWFA_OP_DQ = 20,   // dQ_i = dS K             (tcgen05.mma SS, A MN-major)
  TWFA_OP_RD = 21,   // dQ_i -> global fp32 accumulator (TMA reduce-add)
  TWFA_OP_COUNT = 22
};

struct alignas(16) TwfaPlanOp {  // 16 bytes: one vector load on the device
  uint8_t node;        // index in the problem graph (declaration order)
  uint8_t kind;        // TwfaOpKind
  uint8_t tile;        // Q sub-tile k for S/MX/EX/CR/PV, else 0
  uint8_t stage;       // M(v) div I
  uint8_t slot;        // M(v) mod I  (cycle inside the steady-state trip)
  uint8_t warp_start;  // A(v)
  uint8_t warp_count;  // warps_required(v)
  uint8_t order;       // rank inside the trip on its warp(s)
  uint8_t flags;       // TWFA_OPF_*
  uint8_t pad[7];
};

// MX_k is immediately followed by EX_k (same stage) in the trip program of
// every warp of its warpgroup: the kernel keeps the S row in registers
// between the two ops instead of re-reading it from tensor memory.
#define TWFA_OPF_FUSE_NEXT 1
// S_k is issued by the same thread as PV_k, after PV_k(i-1) in program order:
// tcgen05.mma ops of one thread execute in issue order, so S_k(i) cannot
// overwrite the P_k(i-1) columns before PV_k(i-1) has read them and the
// issue needs no wait on PV_k's completion (the PV_k -> S_k, delta 1, d 0
// edge of the loop graph is realized by program order alone).
#define TWFA_OPF_INORDER 2
// EX_k whose work is done by the fused MX_k right before it (FUSE_NEXT).
#define TWFA_OPF_FUSED 4
// FA backward: the last tensor-core reader of its streamed ring slot in the
// iteration (releases Q_i / dO_i with its commit).
#define TWFA_OPF_RELEASE 8
// FA backward ST: DS runs on another warpgroup and reads P^T(i-1) back from
// the S^T columns; S^T(i) waits for that read (edge DS -> ST, delta 1).
#define TWFA_OPF_WAIT_PREAD 16

// Kind of the workload the plan drives.
enum TwfaPlanFamily : int32_t { TWFA_FAMILY_FA_FWD = 1, TWFA_FAMILY_GEMM = 2, TWFA_FAMILY_FA_BWD = 3 };

struct TwfaDevicePlan {
  int32_t family;      // TwfaPlanFamily
  int32_t ii;          // I
  int32_t length;      // L
  int32_t copies;      // ceil(L / I)
  int32_t max_stage;   // max over nodes of M div I (== copies - 1 or less)
  int32_t num_nodes;
  int32_t num_warps;   // machine.num_warps: CTA = num_warps x 32 threads (+ extra)
  int32_t num_tiles;   // Q sub-tiles per CTA (number of S_k nodes)
  int32_t k_depth;     // smem ring depth of the streamed K (or A) loads
  int32_t v_depth;     // smem ring depth of the streamed V (or B) loads
  int32_t load_warp;   // warp issuing the TMA loads (and the per-tile Q load)
  // Streamed loads issue `prefetch` iterations ahead of their schedule slot:
  // the ring of depth D hides the load latency (the reference's streaming
  // rewrite, jointsolve.cpp:511-524), bounded so a same-warp consumer never
  // waits on a slot its own warp frees later.
  int32_t k_prefetch;
  int32_t v_prefetch;
  // S ring depth in tensor memory (delta of the PV_k -> S_k edge, 1 or 2) and
  // the K/V tile it implies: the 128 S/P columns of a sub-tile hold s_depth
  // tiles of kv_tile = 128 / s_depth keys.
  int32_t s_depth;
  int32_t kv_tile;
  int32_t s_split;  // S_k is SA_k + SB_k (P_k at columns 64-127)
  int32_t cr_warp[TWFA_MAX_TILES];  // warpgroup start running CR_k (+ epilogue of tile k)
  int32_t sm_warp[TWFA_MAX_TILES];  // warpgroup start running MX_k / EX_k
  int32_t mma_warp;                 // GEMM: warp issuing MMA
  // Unit-order tokens: the EX ops share one capacity-1 unit (MUFU) and the
  // modulo schedule orders them inside the trip; the kernel realizes that
  // reservation order with a token passed EX -> EX in slot order.
  int32_t heavy_wg_mask;            // bit w: warpgroup w runs MX/EX (gets the big register budget)
  int32_t q_warp;                   // FA forward: idle warp that loads the Q tiles (-1: the load warp)
  int32_t ex_ring_len;              // 0 = no token (stages differ / single EX)
  uint8_t ex_ring[TWFA_MAX_TILES];  // tiles of the EX ops in slot order
  TwfaPlanOp ops[TWFA_MAX_NODES];
  // per-warp trip programs: indices into ops[], in issue order
  uint8_t prog[TWFA_MAX_WARPS][TWFA_MAX_NODES];
  uint8_t prog_len[TWFA_MAX_WARPS];
};
