/*
 * qc.h -- C ABI of the B200-native state-vector gate engine (libqc.so).
 *
 * The library applies a quantum circuit's 1- and 2-qubit gates to a
 * 2^n-amplitude complex state vector resident in B200 HBM.  It implements the
 * hot path of qclab++ (arXiv 2303.00123).  Citations "P:n" are PAPER.md lines.
 *
 * Semantics fixed by the paper:
 *   - Each gate is psi = (I_l (x) U (x) I_r) phi            eq:kron.
 *   - Qubit numbering is Definition 1: qubit 0 is the MOST
 *     significant bit of the amplitude index; qubit q is bit n-1-q.
 *   - 1-qubit gates = 2^{n-1} independent 2x2 matvecs (Alg. alg:1q);
 *     controlled 1-qubit gates update the control-selected half (Alg.
 *     alg:ctrl-1q, all four control cases); 2-qubit gates are
 *     2^{n-2} 4x4 matvecs on any (non-contiguous) qubit pair (Alg. alg:2q,
 *     P:883-919); SWAP and CNOT are pure element moves (P:852-854,
 *     P:921-938); a doubly controlled gate touches a quarter.
 *   - A circuit is the ordered product of its gates.
 *   Matrix conventions the paper leaves open are DESIGN.md readings R1-R14
 *   (R1: the 4x4 of a 2-qubit gate is indexed big-endian over the LISTED
 *   qubit order, i.e. eq:kron, not Alg. alg:2q read literally; R4: gate
 *   matrices; R11: X/CNOT/SWAP/CCX are bit-exact moves).
 *
 * Data layout: the state is one device buffer of 2^n interleaved complex
 * numbers (QC_COMPLEX64: 2 x float, 8 B; QC_COMPLEX128: 2 x double, 16 B).
 * The library may keep the amplitudes in a PERMUTED bit order (SWAP gates are
 * applied as relabels when QC_OPT_RELABEL_SWAP is on); qc_state_read /
 * qc_state_write always speak canonical (Definition 1) order.
 *
 * Ownership: the state owns its device memory (qc_state_create*), except for
 * qc_state_wrap, where the caller keeps ownership and guarantees lifetime.
 * Every host pointer argument is borrowed for the duration of the call only.
 *
 * Errors: every call returns a qc_status; qc_last_error() returns a
 * thread-local message for the last failing call on this thread.  Argument
 * validation happens BEFORE any device work, so on QC_ERR_INVALID_ARG the
 * state is unchanged (qc_run_circuit validates the whole list first).
 * Asynchronous CUDA failures surface at the next call that checks the stream
 * and mark the state failed: every later call returns QC_ERR_STATE_FAILED.
 *
 * Threading: a qc_state is not thread-safe; distinct states are independent.
 * apply/run enqueue on the state's CUDA stream and return; read, norm2 and
 * sync block until the stream is drained.
 */
#ifndef QC_H_
#define QC_H_

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define QC_ABI_VERSION 1

typedef enum {
    QC_OK = 0,
    QC_ERR_INVALID_ARG = 1,   /* bad n, qubit out of range / repeated, NULL, NaN theta, range */
    QC_ERR_OUT_OF_MEMORY = 2, /* device allocation failed (message states s*2^n bytes) */
    QC_ERR_CUDA = 3,          /* a CUDA runtime call failed */
    QC_ERR_NCCL = 4,          /* reserved for the sharded layer */
    QC_ERR_UNSUPPORTED = 5,   /* valid request this build does not implement */
    QC_ERR_STATE_FAILED = 6   /* an earlier asynchronous failure poisoned the state */
} qc_status;

typedef enum {
    QC_COMPLEX64 = 0,   /* interleaved 2 x float32 per amplitude (8 B)  */
    QC_COMPLEX128 = 1   /* interleaved 2 x float64 per amplitude (16 B) */
} qc_precision;

/* Gate kinds.  "qubits" lists controls first.  Matrices:
 *   H = [[1,1],[1,-1]]/sqrt2;  X, Y, Z per P:617-631;  P(t) = diag(1, e^{it});
 *   RX(t) = exp(-i t X/2), RY(t) = exp(-i t Y/2), RZ(t) = diag(e^{-it/2}, e^{it/2});
 *   CNOT/CZ/CP/CU1: 1 control + target;  CCX: 2 controls + target (Toffoli);
 *   SWAP: P:921-930;  U1: any 2x2;  U2: any 4x4 on (qubits[0], qubits[1]),
 *   row/column index = 2*bit(qubits[0]) + bit(qubits[1]) (eq:kron, R1).     */
typedef enum {
    QC_H = 0, QC_X = 1, QC_Y = 2, QC_Z = 3, QC_P = 4, QC_RX = 5, QC_RY = 6, QC_RZ = 7,
    QC_CNOT = 8, QC_CZ = 9, QC_CP = 10, QC_SWAP = 11,
    QC_U1 = 12, QC_CU1 = 13, QC_U2 = 14, QC_CCX = 15,
    QC_MGATE = 16   /* generic gate: qubits[0] = index into the qc_mgate table of
                       qc_run_circuit_ex (other fields ignored, flags must be 0) */
} qc_op;

#define QC_CTRL_ONES 0xFFFFFFFFu  /* default: every control must be |1> */

/* One gate of an op list (288 bytes, 8-byte aligned). */
typedef struct qc_gate {
    int32_t op;          /* qc_op                                                    */
    int32_t qubits[3];   /* listed qubits (controls first); entries past arity ignored */
    uint32_t ctrl_state; /* bit t = required state of listed control t (low nctrl bits) */
    uint32_t flags;      /* reserved, must be 0                                      */
    double theta;        /* P, RX, RY, RZ, CP (finite); ignored otherwise            */
    double m[32];        /* U1/CU1: 2x2, U2: 4x4; interleaved re,im; row-major       */
} qc_gate;

typedef struct qc_state qc_state;  /* opaque handle */

typedef enum {
    QC_OPT_FUSION = 0,        /* 1 (default): fused tile passes; 0: one kernel per gate    */
    QC_OPT_RELABEL_SWAP = 1,  /* 1 (default): SWAP = relabel (0 bytes moved); 0: data move  */
    QC_OPT_USE_GRAPH = 2,     /* 1 (default): replay repeated circuits as CUDA graphs       */
    QC_OPT_TILE_BITS = 3,     /* 0 (default): auto (64 KiB tiles); else 4..13               */
    QC_OPT_CTAS = 4,          /* 0 (default): one CTA per SM; else grid size of fused passes */
    QC_OPT_BLOCK_FUSION = 5,  /* 1 (default): merge gates on <= 2 qubits into exact blocks    */
    QC_OPT_JIT = 6,           /* 1 (default): specialise repeated fused plans with NVRTC
                                 (and plans whose passes span >= 2^30 amplitudes from the
                                 first run); 0: never (AOT interpreting kernel); 2: from
                                 the first run                                              */
    QC_OPT_ROW_BITS = 7,      /* 0 (default): auto -- with the box transport the planner plans
                                 3..6 (c128) / 4..7 (c64) row bits and keeps the plan a host
                                 cost model prefers; else the contiguous row bits of a tile  */
    QC_OPT_TMA_MODE = 8,      /* 0 (default): one 5-D TMA box per tile (dims = the runs of
                                 consecutive tile bits, coordinates = the outer bits above
                                 each run; several boxes when > 5 runs), gather4 rows for a
                                 pass whose runs do not fit; 1: one cp.async.bulk per row;
                                 2: TMA tile::gather4/scatter4 rows only (4 rows/request)    */
    QC_OPT_REMAP = 9,         /* 1 (default): a fused pass may end by swapping row bits with
                                 tile bits the next pass needs (a relabel, like SWAP);
                                 0: the row bits keep their qubits                           */
    QC_OPT_EXCHANGE = 10      /* sharded states (NCCL, and the loopback, which runs the same
                                 schedules on one GPU), how gates on rank-bit qubits are
                                 served (collective: set the same value on every rank):
                                 0 (default): NCCL send/recv of 256 MiB chunks into two
                                   ping-pong staging buffers on a second stream, each chunk's
                                   copy into place overlapping the next chunk's transfer;
                                 1: peer-to-peer -- every rank maps the others' state buffers
                                   (CUDA IPC handles all-gathered over NCCL) and one kernel
                                   per run swaps the two halves directly over NVLink (loads +
                                   stores, no staging copy); the pair splits each run in two
                                   and brackets the kernel with a pairwise NCCL token barrier;
                                 2: collective-fused pair passes -- a run of gates whose only
                                   non-diagonal rank-bit qubit is g is planned over the local
                                   bits + g; ranks r and r ^ 2^(g-n_loc) split every pass's
                                   tiles, and a pass whose tile holds g moves the two tile
                                   halves from / to both shards directly (TMA over the IPC-
                                   mapped partner buffer): the exchange is fused into the
                                   pass and the layout does not change (no swap back).  A
                                   gate on two rank-bit qubits at once falls back to 1;
                                 3: group plan -- the whole circuit planned once over all n
                                   bits like a single-GPU state; a pass whose tile holds j
                                   rank bits moves its 2^j sub-tiles from / to 2^j shards
                                   (one tensor map per shard), the P ranks splitting its
                                   tiles; passes without rank bits stay in the own shard.
                                   No exchanges, no layout change; spanning passes are
                                   bracketed by world barriers                          */
} qc_option;

/* Counters of the most recent qc_run_circuit / qc_apply_gate. */
typedef struct qc_info {
    int32_t n;
    int32_t precision;        /* qc_precision */
    void* device_ptr;         /* amplitudes (physical order, see layout)        */
    void* stream;             /* cudaStream_t the state enqueues on             */
    int32_t layout[64];       /* layout[q] = physical bit position of qubit q   */
    int32_t layout_is_canonical;
    int64_t last_gates;       /* gates in the last run                          */
    int64_t last_passes;      /* fused tile passes (or per-gate kernels)        */
    int64_t last_launches;    /* kernels launched by the last run               */
    int64_t last_relabels;    /* SWAPs applied as relabels                      */
    int32_t last_graph;       /* 1 if the last run replayed a CUDA graph        */
    int32_t tile_bits;        /* k of the last fused run                        */
    int64_t last_blocks;      /* ops after block fusion (fused runs)            */
    int32_t last_jit;         /* 1 if the last run used NVRTC-specialised passes */
    int32_t world;            /* ranks the state is sharded over (1: not sharded) */
    int32_t rank;             /* this rank                                       */
    int32_t n_local;          /* qubits per shard (n - log2 world)               */
    int32_t sharding;         /* 0 single GPU, 1 loopback (all shards here), 2 NCCL */
    int64_t last_exchanges;   /* qubit-swap exchanges in the last run            */
    double last_flops_per_amp; /* fused runs: algorithmic flops per amplitude of the
                                  plan's fused ops (complex arithmetic counted;
                                  the ALU roofline numerator, qc_debug.h)      */
    int64_t last_pair_segments; /* sharded runs with QC_OPT_EXCHANGE 2: pair segments
                                   (gates on one rank-bit qubit run in place over
                                   the pair's two shards, no exchange); with 3:
                                   passes whose tiles span several shards       */
} qc_info;

/* Generic gate: any number of controls and a dense
 * 2^k x 2^k matrix on k = n_targ <= 4 targets.  P:942-946 -- every further
 * qubit is one more inserted index bit ("2 additional bit masks")
 * -- a doubly controlled gate updates only the block where both controls hold
 * (here: every control t equals bit t of ctrl_state).  The embedded operator
 * over the listed qubits is the identity except that block, which holds the
 * matrix; matrix rows/columns are big-endian over the listed TARGETS (first
 * target = most significant index bit, eq:kron P:407-412, reading R1).
 * Exact structure is detected (a diagonal / permutation 2x2 runs as a phase /
 * move, X under controls is bit-exact).  88 bytes, 8-byte aligned. */
#define QC_MGATE_MAX_QUBITS 16
#define QC_MGATE_MAX_TARGETS 4
typedef struct qc_mgate {
    int32_t n_ctrl;            /* controls, listed first: 0..15                    */
    int32_t n_targ;            /* targets after them: 1..4                          */
    int32_t qubits[QC_MGATE_MAX_QUBITS];  /* distinct, in [0,n); past n_ctrl+n_targ ignored */
    uint32_t ctrl_state;       /* bit t = required state of listed control t        */
    uint32_t flags;            /* reserved, must be 0                               */
    const double* matrix;      /* 2^k x 2^k complex, interleaved re,im, row-major;
                                  borrowed for the call (copied before return)     */
} qc_mgate;

/* ---------------------------------------------------------------- lifetime */

/* Sharded states (north star: shard the vector across B200s by
 * its top log2(P) qubits, remap global<->local qubits by NCCL pairwise
 * send/recv).  A state over P = 2^p ranks keeps 2^(n-p) amplitudes per rank;
 * physical bits >= n-p are rank bits.  Gates whose non-diagonal targets are
 * local run fused on each shard (rank-bit controls and diagonal bits are
 * per-rank constants); a non-diagonal target on a rank bit triggers a
 * qubit-swap exchange with the partner rank (half a shard per direction).
 * Every rank must make the same calls with the same arguments (collective). */

/* 128-byte NCCL unique id for qc_state_create_dist (call on one rank, then
 * broadcast, e.g. over torch.distributed). */
qc_status qc_nccl_unique_id(void* out128);

/* One process per GPU: this rank's shard of an n-qubit state over `world`
 * ranks (power of two), initialised to |0...0>; creates an NCCL communicator
 * from `nccl_unique_id` (collective).  n - log2(world) >= 8. */
qc_status qc_state_create_dist(int n, qc_precision p, int rank, int world,
                               const void* nccl_unique_id, qc_state** out);

/* All `world` shards in ONE process and ONE device buffer (2^n amplitudes):
 * the sharded schedule and exchange arithmetic run exactly as with NCCL but
 * exchanges are device swaps of the same runs.  For validation on one GPU. */
qc_status qc_state_create_loopback(int n, qc_precision p, int world, qc_state** out);

/* Allocate an n-qubit state on the current CUDA device, initialised to |0...0>,
 * with its own non-blocking stream.  1 <= n <= 40.  Returns NULL on error
 * (qc_last_error() says why; out of memory names the s*2^n byte count). */
qc_state* qc_state_create(int n, qc_precision p);

/* As qc_state_create, on `device`, enqueuing on `cuda_stream` (a cudaStream_t;
 * NULL = the library creates a non-blocking stream). */
qc_status qc_state_create_ex(int n, qc_precision p, int device, void* cuda_stream,
                             qc_state** out);

/* Borrow caller-owned device memory of s*2^n bytes (e.g. a torch tensor) and a
 * stream.  Contents are taken as the state in canonical order. */
qc_status qc_state_wrap(int n, qc_precision p, void* dev_ptr, void* cuda_stream,
                        qc_state** out);

/* Synchronise the stream and free everything the state owns.  NULL is a no-op. */
void qc_state_destroy(qc_state* s);

/* ------------------------------------------------------------ initial data */

/* |k>, canonical index k < 2^n.  Resets the layout to canonical. */
qc_status qc_state_init_basis(qc_state* s, uint64_t k);

/* The seeded random state of DESIGN.md's input recipe, generated on device:
 *   re_i = u(sm(seed,2i))*c, im_i = u(sm(seed,2i+1))*c, c = sqrt(1.5/2^n),
 *   sm = counter-based splitmix64, u(x) = (x>>11)*2^-52 - 1;
 * complex64 rounds each double to float.  Resets the layout to canonical. */
qc_status qc_state_init_random(qc_state* s, uint64_t seed);

/* --------------------------------------------------------------- the path */

/* Apply one gate with its own per-gate kernel (no fusion).  `qubits` holds
 * arity(op) distinct qubits in [0,n), controls first (controls = |1>).
 * `matrix`: NULL for H X Y Z CNOT CZ SWAP CCX; one double theta for P RX RY RZ
 * CP; 8 doubles (2x2) for U1 and CU1; 32 doubles (4x4) for U2, interleaved
 * re,im, row-major.  Enqueued; returns without waiting. */
qc_status qc_apply_gate(qc_state* s, qc_op op, const int* qubits, const double* matrix);

/* Apply n_ops gates in order (Alg. 1-3 semantics, eq:kron product).  The
 * whole list is validated first (all-or-nothing).  With QC_OPT_FUSION the
 * planner groups gates into fused tile passes (one HBM round trip each);
 * otherwise one kernel per gate.  Enqueued; returns without waiting. */
qc_status qc_run_circuit(qc_state* s, const qc_gate* ops, size_t n_ops);

/* One generic gate with its own per-gate kernel (no fusion): validated
 * (controls + targets distinct and in range, 1 <= n_targ <= 4, n_ctrl +
 * n_targ <= 16, finite matrix, flags 0), then enqueued. */
qc_status qc_apply_mgate(qc_state* s, const qc_mgate* g);

/* qc_run_circuit with generic gates: an op with op == QC_MGATE stands for
 * mgates[qubits[0]] (0 <= qubits[0] < n_mgates).  Same semantics, fusion,
 * plan caching (keyed by the referenced gates' contents) and all-or-nothing
 * validation as qc_run_circuit; mgates and their matrices are borrowed for
 * the call only.  qc_run_circuit(s, ops, n) == qc_run_circuit_ex(s, ops, n,
 * NULL, 0). */
qc_status qc_run_circuit_ex(qc_state* s, const qc_gate* ops, size_t n_ops,
                            const qc_mgate* mgates, size_t n_mgates);

/* ------------------------------------------------------------------ I/O */

/* Copy canonical amplitudes [first, first+count) to host memory (count*s
 * bytes).  Blocks.  Undoes any pending relabel on the fly (gather kernel).
 * NCCL-sharded states: the layout must be canonical (qc_state_canonicalize)
 * and the range inside this rank's shard [rank*2^(n-p), (rank+1)*2^(n-p)). */
qc_status qc_state_read(qc_state* s, uint64_t first, uint64_t count, void* host_dst);

/* Write canonical amplitudes [first, first+count) from host memory.  Blocks
 * until the copy has been consumed.  Leaves the layout unchanged. */
qc_status qc_state_write(qc_state* s, uint64_t first, uint64_t count, const void* host_src);

/* Read canonical amplitudes [first, first+count) into host_dst and replace
 * them with host_src: the same as qc_state_read then qc_state_write, but in
 * 256 MiB chunks with the upload of chunk c (a second copy stream) overlapping
 * the read-back of chunk c+1 -- PCIe / C2C links are full duplex, so handing
 * a result back and loading the next input costs about one direction.  Chunk
 * c is uploaded only after it has been read, so host_src == host_dst uploads
 * exactly what was read (the two buffers must be identical or disjoint).
 * Blocks.  Same range / layout rules as
 * qc_state_read (a non-canonical single-GPU layout: read, then write). */
qc_status qc_state_readwrite(qc_state* s, uint64_t first, uint64_t count, void* host_dst, const void* host_src);

/* Permute the amplitudes back to canonical order in place (no-op if already). */
qc_status qc_state_canonicalize(qc_state* s);

/* Block until all enqueued work on the state's stream is done; report any
 * asynchronous CUDA failure. */
qc_status qc_state_sync(qc_state* s);

/* sum_i |psi_i|^2 in double (device reduction).  Blocks. */
qc_status qc_state_norm2(qc_state* s, double* out);

/* ---------------------------------------------------------- configuration */

qc_status qc_set_option(qc_state* s, qc_option opt, int64_t value);
qc_status qc_get_info(const qc_state* s, qc_info* out);

/* ------------------------------------------------------------ openQASM 2.0
 * The paper's I/O statement (P:6: "provides I/O through openQASM"); grammar
 * per SPEC S:442-495: header `OPENQASM 2.0;`, the literal
 * `include "qelib1.inc";`, exactly one `qreg`, gate statements h x y z,
 * p|u1, rx ry rz, cx|CX, cz, cp|cu1, swap, ccx with constant angle
 * expressions (+ - * /, unary minus, parentheses, numbers, pi), `//`
 * comments.  creg / measure / reset / barrier / if / gate definitions /
 * a second qreg are rejected.  Host-only (no device work, no state).
 *
 * qc_qasm_parse: text (NUL-terminated, borrowed) -> *n_qubits and the gate
 *   list in program order; writes min(cap, count) gates to `ops` (may be
 *   NULL to query) and always sets *n_ops = count.  Errors: QC_ERR_INVALID_ARG
 *   with "line:col: what" in qc_last_error().
 * qc_qasm_emit: gate list -> text ("OPENQASM 2.0;\ninclude \"qelib1.inc\";\n
 *   qreg q[n];\n" + one statement per gate, angles with 17 significant
 *   digits; P -> u1, CP -> cu1, CNOT -> cx).  Writes at most cap-1 bytes + NUL
 *   to buf (may be NULL to query) and always sets *len = full length.
 *   Errors: QC_ERR_INVALID_ARG (invalid gate), QC_ERR_UNSUPPORTED (U1 / CU1 /
 *   U2 generic matrices or |0> controls: no qelib1 name). */
qc_status qc_qasm_parse(const char* text, int* n_qubits, qc_gate* ops, size_t cap, size_t* n_ops);
qc_status qc_qasm_emit(int n, const qc_gate* ops, size_t n_ops, char* buf, size_t cap, size_t* len);

/* Thread-local message of the last failing call ("" if none). */
const char* qc_last_error(void);

/* Library version string ("qc-b200 <abi> sm_100a"). */
const char* qc_version(void);

#ifdef __cplusplus
}
#endif
#endif /* QC_H_ */
