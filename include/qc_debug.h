/*
 * qc_debug.h -- host-only introspection of libqc's planner (no GPU needed).
 *
 * qc_debug_plan lowers an op list with the canonical layout, applies block
 * fusion and the fused-pass planner exactly as qc_run_circuit would, and
 * reports the plan's shape.  With compile_jit != 0 it also generates and
 * NVRTC-compiles the specialised kernel of every pass for sm_100a (no launch).
 * Used by the CPU test-suite to check planner invariants and the code
 * generator; not part of the hot path.
 */
#ifndef QC_DEBUG_H_
#define QC_DEBUG_H_
#include "qc.h"

#ifdef __cplusplus
extern "C" {
#endif

typedef struct qc_plan_stats {
    int64_t gates;        /* input gates                                    */
    int64_t relabels;     /* SWAPs turned into relabels                     */
    int64_t blocks;       /* ops after block fusion                         */
    int64_t passes;       /* fused tile passes                              */
    int64_t substages;    /* register sub-stages over all passes            */
    int64_t fused_ops;    /* encoded ops over all passes                    */
    int64_t phase_runs;   /* phase-run ops over all passes                  */
    int64_t blob_bytes;   /* packed op blob bytes                           */
    int32_t tile_bits;
    int32_t jit_compiled; /* passes compiled by NVRTC (compile_jit != 0)    */
    int64_t remap_swaps;  /* row-bit <-> tile-bit remap swaps (remap != 0)  */
    int64_t restore_passes; /* swap-only passes restoring the input layout  */
    double flops_per_amp; /* algorithmic flops per amplitude of the fused ops */
    int64_t swz_substages;  /* sub-stages with >= 2 slot bits among the smem
                               bank-group bits (lane-XOR select network)     */
} qc_plan_stats;

/* tile_bits / row_bits 0 = default; remap as QC_OPT_REMAP.  errbuf (may be
 * NULL) receives a message on error. */
qc_status qc_debug_plan(int n, qc_precision p, const qc_gate* ops, size_t n_ops, int tile_bits,
                        int row_bits, int block_fusion, int remap, int compile_jit, qc_plan_stats* out,
                        char* errbuf, size_t errlen);

/* Sharded-state exchange arithmetic (host only): the runs of local indices
 * (offset, count in amplitudes) that rank `rank` sends to -- and receives
 * from -- `partner` when rank bit g is swapped with local bit l (n_loc local
 * qubits).  Returns the run count in n_runs (fills at most max_runs). */
qc_status qc_debug_exchange_runs(int n_loc, int rank, int g, int l, int* partner, uint64_t* offsets,
                                 uint64_t* counts, int max_runs, int* n_runs);

/* The sharded schedule qc_run_circuit would execute from the canonical
 * layout (host only, deterministic): steps[4*i..] = (kind, g, l, gates) with
 * kind 0 = fused local segment of `gates` gates, 1 = exchange of rank bit g
 * with local bit l (gates = 1: one of the exchanges at the end that return
 * the layout to the one the SWAP relabels alone give).  layout_out (n ints,
 * may be NULL) = final layout. */
qc_status qc_debug_dist_schedule(int n, int world, int relabel, const qc_gate* ops, size_t n_ops,
                                 int* steps, int max_steps, int* n_steps, int* layout_out);
/* Same, for a QC_OPT_EXCHANGE mode (0/1: exchanges; 2: pair segments, kind 2
 * = pair segment of `gates` gates on rank bit g, l = -1). */
qc_status qc_debug_dist_schedule_ex(int n, int world, int relabel, int exchange_mode, const qc_gate* ops,
                                    size_t n_ops, int* steps, int max_steps, int* n_steps, int* layout_out);

/* Group plans (QC_OPT_EXCHANGE 3, host arithmetic): for a pass with tile bit
 * set T over an n-bit index sharded over `world` ranks (rank bits n-p..n-1),
 * rank `rank`'s tile range [tile0, tile0+count) of the pass's 2^(n-|T|)
 * tiles, the number j of rank bits in T, and owners[h] = the rank holding
 * sub-tile h (its T-rank bits = h) for h < 2^j (-1 beyond). */
qc_status qc_debug_group_split(int n, int world, uint64_t tile_bits_set, int rank, uint64_t* tile0,
                               uint64_t* count, int* j, int* owners);

/* Run one qubit-swap exchange of physical rank bit g with local bit l on a
 * sharded state (collective; enqueued on the state's stream); the layout is
 * updated.  Used to time NVLink exchanges in isolation. */
qc_status qc_debug_exchange(qc_state* s, int g, int l);

/* The TMA box decomposition of a tile (host only; QC_OPT_TMA_MODE 0): the
 * tile's physical bit set T over an nbits-bit index -> dims (<= 5) starting
 * at starts[0..dims) (starts[dims] = nbits), box widths boxbits[d] (tile bits
 * at the bottom of dim d), and xmask = tile bits beyond the 5th run relative
 * to starts[4] (one box per combination).  Returns QC_ERR_UNSUPPORTED if the
 * tile needs more than 16 boxes (the pass then moves gather4 rows). */
qc_status qc_debug_box_layout(uint64_t tile_bits_set, int nbits, int dbl, int* dims, int* starts,
                              int* boxbits, uint32_t* xmask);

/* Measurement utility (needs a GPU): the FMA throughput of the current device
 * in TFLOP/s (2 flops per FMA), FP64 (dbl != 0) or FP32, from a kernel of 8
 * independent FMA chains per thread (best of 3 timed launches).  bench.py
 * uses it as the ALU roofline peak of the fused pass. */
qc_status qc_debug_fma_peak(int dbl, double* tflops);

#ifdef __cplusplus
}
#endif
#endif
