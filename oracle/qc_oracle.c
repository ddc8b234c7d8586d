/*
 * qc_oracle.c -- TEST INFRASTRUCTURE ONLY.
 *
 * A plain, slow, obviously-correct CPU state-vector simulator used to check
 * the CUDA path.  Only tests/, __graft_entry__.smoke() and bench.py's
 * cpu_baseline / --impl reference leg may load it.  It shares no code, header,
 * table or constant with paper_2303_00123_b200/ (the product), and the product
 * never loads it.
 *
 * What it computes (PAPER.md = "P:n"):
 *   Each gate is  psi = (I_l (x) U (x) I_r) phi       eq:kron, P:407-412,
 *   with non-contiguous / reordered / controlled gates being the same operator
 *   with its qubits permuted into place.  Index bits follow
 *   Definition 1: qubit q is bit position n-1-q (qubit 0 = MSB).
 *   A circuit is the ordered product of its gates.
 *
 * Algorithm ("per-amplitude bit extraction"):
 *   U  <- embed(op)                        2^k x 2^k complex double, built here
 *   gm <- OR_t 2^(n-1-q_t)
 *   for i in [0, 2^n):  if (i & gm) continue
 *       idx[c] = i | sum_t bit(c, k-1-t) * 2^(n-1-q_t)   (first listed qubit
 *                                                        = MSB of c, eq:kron)
 *       v[c] = phi[idx[c]];  phi[idx[r]] = sum_c U[r][c] v[c]   (fixed order)
 *   No bit masks m_L/m_C/m_R, no specialisations, always double precision.
 *
 * Gate matrices (reading R4; the paper defines only X, Y, Z, SWAP):
 *   H = [[1,1],[1,-1]]/sqrt2    X, Y, Z per P:617-631    P(t) = diag(1, e^{it})
 *   RX(t) = [[c,-is],[-is,c]]   RY(t) = [[c,-s],[s,c]]    RZ(t) = diag(e^{-it/2}, e^{it/2})
 *   (c = cos(t/2), s = sin(t/2));  SWAP per P:921-938;  CNOT/CZ/CP/CU1/CCX:
 *   identity except the block where the controls equal ctrl_state.
 *
 * Parity pins: see tests/test_oracle.py (brute-force numpy.kron, the paper's
 * index tables fig:1q / fig:ctrl-1q / fig:dctrl-1q, FFT closed form, QFT o
 * QFT^-1, TFXY zero-angle identity and parity sector, unitarity).
 */
#include <complex.h>
#include <math.h>
#include <stdint.h>
#include <stdlib.h>
#include <string.h>
#ifdef _OPENMP
#include <omp.h>
#endif

/* The oracle's own op codes (the Python wrapper maps names to these). */
enum {
    ORC_H = 0, ORC_X, ORC_Y, ORC_Z, ORC_P, ORC_RX, ORC_RY, ORC_RZ,
    ORC_CNOT, ORC_CZ, ORC_CP, ORC_SWAP, ORC_U1, ORC_CU1, ORC_U2, ORC_CCX,
    ORC_NKINDS
};

typedef struct {
    int32_t kind;
    int32_t nq;          /* number of listed qubits (controls first)        */
    int32_t q[3];        /* paper qubit numbers                             */
    uint32_t ctrl_state; /* bit t = required state of listed control t      */
    double theta;
    double m[32];        /* U1/CU1: 2x2, U2: 4x4, interleaved re,im, row-major */
} orc_op;

static const int orc_arity[ORC_NKINDS] = {1, 1, 1, 1, 1, 1, 1, 1, 2, 2, 2, 2, 1, 2, 2, 3};
static const int orc_nctrl[ORC_NKINDS] = {0, 0, 0, 0, 0, 0, 0, 0, 1, 1, 1, 0, 0, 1, 0, 2};

/* 2x2 target matrix V of a (possibly controlled) 1-qubit op. */
static void target_2x2(const orc_op* op, double complex V[2][2]) {
    const double t = op->theta;
    const double c = cos(t / 2.0), s = sin(t / 2.0);
    const double h = 1.0 / sqrt(2.0);
    memset(V, 0, sizeof(double complex) * 4);
    switch (op->kind) {
    case ORC_H:  V[0][0] = h; V[0][1] = h; V[1][0] = h; V[1][1] = -h; break;
    case ORC_X: case ORC_CNOT: case ORC_CCX:
                 V[0][1] = 1.0; V[1][0] = 1.0; break;
    case ORC_Y:  V[0][1] = -I; V[1][0] = I; break;
    case ORC_Z: case ORC_CZ:
                 V[0][0] = 1.0; V[1][1] = -1.0; break;
    case ORC_P: case ORC_CP:
                 V[0][0] = 1.0; V[1][1] = cexp(I * t); break;
    case ORC_RX: V[0][0] = c; V[0][1] = -I * s; V[1][0] = -I * s; V[1][1] = c; break;
    case ORC_RY: V[0][0] = c; V[0][1] = -s; V[1][0] = s; V[1][1] = c; break;
    case ORC_RZ: V[0][0] = cexp(-I * t / 2.0); V[1][1] = cexp(I * t / 2.0); break;
    case ORC_U1: case ORC_CU1:
        for (int r = 0; r < 2; r++)
            for (int cc = 0; cc < 2; cc++)
                V[r][cc] = op->m[2 * (2 * r + cc)] + I * op->m[2 * (2 * r + cc) + 1];
        break;
    default: break;
    }
}

/* Embedded 2^k x 2^k matrix over the op's listed qubits (first = MSB).
 * Returns k, or -1 for an unknown op.  U is row-major, dim <= 8.          */
int orc_embed(const orc_op* op, double complex* U) {
    if (op->kind < 0 || op->kind >= ORC_NKINDS) return -1;
    const int k = orc_arity[op->kind];
    const int d = 1 << k;
    memset(U, 0, sizeof(double complex) * d * d);
    if (op->kind == ORC_SWAP) {
        U[0 * 4 + 0] = 1.0; U[1 * 4 + 2] = 1.0; U[2 * 4 + 1] = 1.0; U[3 * 4 + 3] = 1.0;
        return k;
    }
    if (op->kind == ORC_U2) {
        for (int r = 0; r < 4; r++)
            for (int c = 0; c < 4; c++)
                U[r * 4 + c] = op->m[2 * (4 * r + c)] + I * op->m[2 * (4 * r + c) + 1];
        return k;
    }
    double complex V[2][2];
    target_2x2(op, V);
    const int nc = orc_nctrl[op->kind];
    if (nc == 0) {
        for (int r = 0; r < 2; r++)
            for (int c = 0; c < 2; c++) U[r * 2 + c] = V[r][c];
        return k;
    }
    /* controlled: identity, except the 2x2 block where control t (local bit
     * nc-t, i.e. listed order MSB first) equals bit t of ctrl_state. */
    for (int r = 0; r < d; r++) U[r * d + r] = 1.0;
    int cp = 0;
    for (int t = 0; t < nc; t++)
        cp |= (int)((op->ctrl_state >> t) & 1u) << (nc - 1 - t);
    for (int a = 0; a < 2; a++)
        for (int b = 0; b < 2; b++) U[(cp * 2 + a) * d + (cp * 2 + b)] = V[a][b];
    return k;
}

/* Validate one op against n.  0 = ok. */
static int orc_check(int n, const orc_op* op) {
    if (op->kind < 0 || op->kind >= ORC_NKINDS) return 1;
    const int k = orc_arity[op->kind];
    if (op->nq != k) return 2;
    for (int t = 0; t < k; t++) {
        if (op->q[t] < 0 || op->q[t] >= n) return 3;
        for (int u = 0; u < t; u++)
            if (op->q[u] == op->q[t]) return 4;
    }
    if (!isfinite(op->theta)) return 5;
    return 0;
}

/* Apply one gate in place: the plain loop of the header comment. */
static void orc_apply_one(int n, double complex* phi, const orc_op* op) {
    double complex U[64];
    const int k = orc_embed(op, U);
    const int d = 1 << k;
    uint64_t bit[3];
    uint64_t gm = 0;
    for (int t = 0; t < k; t++) {
        bit[t] = (uint64_t)1 << (n - 1 - op->q[t]);
        gm |= bit[t];
    }
    const int64_t N = (int64_t)1 << n;
#pragma omp parallel for schedule(static)
    for (int64_t i = 0; i < N; i++) {
        if (((uint64_t)i & gm) != 0) continue;
        uint64_t idx[8];
        double complex v[8];
        for (int c = 0; c < d; c++) {
            uint64_t x = (uint64_t)i;
            for (int t = 0; t < k; t++)
                if ((c >> (k - 1 - t)) & 1) x |= bit[t];
            idx[c] = x;
            v[c] = phi[x];
        }
        for (int r = 0; r < d; r++) {
            double complex acc = 0.0;
            for (int c = 0; c < d; c++) acc += U[r * d + c] * v[c];
            phi[idx[r]] = acc;
        }
    }
}

/* Apply an op list in order.  Validates the whole list first (nothing is
 * touched on error).  Returns 0, or 100*op_index + reason + 1 on error.    */
int64_t orc_run(int n, double complex* phi, const orc_op* ops, int64_t n_ops,
                int nthreads) {
    if (n < 1 || n > 40 || !phi || (n_ops > 0 && !ops)) return -1;
    for (int64_t g = 0; g < n_ops; g++) {
        int e = orc_check(n, &ops[g]);
        if (e) return 100 * g + e + 1;
    }
#ifdef _OPENMP
    if (nthreads > 0) omp_set_num_threads(nthreads);
#else
    (void)nthreads;
#endif
    for (int64_t g = 0; g < n_ops; g++) orc_apply_one(n, phi, &ops[g]);
    return 0;
}

/* ---------------------------------------------------------------------------
 * Generic gate ("for every additional qubit
 * ... 2 additional bit masks", P:948-978 the doubly controlled gate):
 * nctrl controls listed first, then k = nq - nctrl targets carrying a dense
 * 2^k x 2^k matrix U (row/column index big-endian over the listed targets,
 * eq:kron).  The embedded 2^nq x 2^nq operator is the identity except on the
 * block where every control t equals bit t of ctrl_state, which holds U
 * (fig:dctrl-1q: a doubly controlled gate touches only that block).
 * So, for every index i with all listed bits clear, the block's amplitudes
 *     idx[c] = i | (controls set to ctrl_state) | (targets set to the bits of c)
 * are gathered and overwritten with U v (fixed summation order); every other
 * amplitude is left as is (identity rows).                                  */
typedef struct {
    int32_t nq;          /* listed qubits (controls first), 1..16          */
    int32_t nctrl;       /* 0..nq-1                                         */
    int32_t q[16];       /* paper qubit numbers                             */
    uint32_t ctrl_state; /* bit t = required state of listed control t      */
    int32_t pad;
    const double* m;     /* 2^k x 2^k, interleaved re,im, row-major         */
} orc_gop;

static int orc_gcheck(int n, const orc_gop* g) {
    if (g->nq < 1 || g->nq > 16 || g->nctrl < 0 || g->nctrl >= g->nq) return 1;
    if (g->nq - g->nctrl > 6 || !g->m) return 2;
    for (int t = 0; t < g->nq; t++) {
        if (g->q[t] < 0 || g->q[t] >= n) return 3;
        for (int u = 0; u < t; u++)
            if (g->q[u] == g->q[t]) return 4;
    }
    const int d = 1 << (g->nq - g->nctrl);
    for (int e = 0; e < 2 * d * d; e++)
        if (!isfinite(g->m[e])) return 5;
    return 0;
}

static void orc_gapply_one(int n, double complex* phi, const orc_gop* g) {
    const int k = g->nq - g->nctrl, d = 1 << k;
    double complex* U = malloc(sizeof(double complex) * d * d);
    for (int e = 0; e < d * d; e++) U[e] = g->m[2 * e] + I * g->m[2 * e + 1];
    uint64_t gm = 0, cs = 0, tbit[6];
    for (int t = 0; t < g->nq; t++) {
        const uint64_t b = (uint64_t)1 << (n - 1 - g->q[t]);
        gm |= b;
        if (t < g->nctrl) {
            if ((g->ctrl_state >> t) & 1u) cs |= b;
        } else {
            tbit[t - g->nctrl] = b;
        }
    }
    const int64_t N = (int64_t)1 << n;
#pragma omp parallel for schedule(static)
    for (int64_t i = 0; i < N; i++) {
        if (((uint64_t)i & gm) != 0) continue;
        uint64_t idx[64];
        double complex v[64];
        for (int c = 0; c < d; c++) {
            uint64_t x = (uint64_t)i | cs;
            for (int t = 0; t < k; t++)
                if ((c >> (k - 1 - t)) & 1) x |= tbit[t];
            idx[c] = x;
            v[c] = phi[x];
        }
        for (int r = 0; r < d; r++) {
            double complex acc = 0.0;
            for (int c = 0; c < d; c++) acc += U[r * d + c] * v[c];
            phi[idx[r]] = acc;
        }
    }
    free(U);
}

/* Apply a list of generic gates in order (validated first; 0 or
 * 100*index + reason + 1 on error, nothing touched).                      */
int64_t orc_run_general(int n, double complex* phi, const orc_gop* ops, int64_t n_ops,
                        int nthreads) {
    if (n < 1 || n > 40 || !phi || (n_ops > 0 && !ops)) return -1;
    for (int64_t g = 0; g < n_ops; g++) {
        int e = orc_gcheck(n, &ops[g]);
        if (e) return 100 * g + e + 1;
    }
#ifdef _OPENMP
    if (nthreads > 0) omp_set_num_threads(nthreads);
#else
    (void)nthreads;
#endif
    for (int64_t g = 0; g < n_ops; g++) orc_gapply_one(n, phi, &ops[g]);
    return 0;
}

int orc_max_threads(void) {
#ifdef _OPENMP
    return omp_get_max_threads();
#else
    return 1;
#endif
}

int orc_abi_version(void) { return 1; }
