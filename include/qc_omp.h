/*
 * qc_omp.h -- the paper's CPU implementation (libqc_omp.so): Algorithms 1-3 of
 * arXiv 2303.00123 as plain OpenMP loops over a host state vector.
 *
 * qclab++ parallelises every gate with one `#pragma omp parallel for` over the
 * paper's index loop (the CPU listing of fig:Xgate-cpu-vs-gpu P:18-36);
 * its CPU-vs-GPU experiments time exactly that.  This library is
 * that CPU program, written for the same gate semantics as libqc (include/qc.h):
 *   - generic 1-qubit gates: Alg. alg:1q, a_j = (j & m_R) +
 *     ((j & m_L) << 1), b_j = a_j + 2^{n-q-1}; X / Y / Z / P / RZ use the
 *     simplified updates of P:617-631 (Z and P touch only the b_j half);
 *   - controlled 1-qubit gates: Alg. alg:ctrl-1q with the three
 *     masks m_L, m_C, m_R of P:829-850 and the control-state increment of
 *     P:870-874; CNOT swaps half the elements; CCX inserts one more
 *     bit per control;
 *   - 2-qubit gates: Alg. alg:2q on any qubit pair, SWAP as the
 *     element swap of P:932-938.
 * Readings: R1 -- a 2-qubit matrix is indexed big-endian over the
 * LISTED qubits (eq:kron), so b_j / c_j are assigned from the listed order,
 * not from the sorted pair; R2 -- b_j = a_j + 2^{n-q-1} (the listing's
 * precedence slip); R3 -- 64-bit indices and masks (the listing's `int`
 * overflows at n = 32).
 *
 * It is a separate baseline program, never a fallback: libqc.so does not load
 * or call it, and it does not load libqc.so.  Host memory only.
 */
#ifndef QC_OMP_H_
#define QC_OMP_H_
#include "qc.h"

#ifdef __cplusplus
extern "C" {
#endif

/* Apply n_ops named gates (QC_H .. QC_CCX; QC_MGATE is QC_ERR_UNSUPPORTED) in
 * order to the caller-owned host state `x` of 2^n interleaved complex values
 * (QC_COMPLEX64: 2 x float, QC_COMPLEX128: 2 x double), canonical order
 * (Definition 1, qubit 0 = MSB), in place.  One OpenMP parallel loop per
 * gate; nthreads > 0 sets the team size (0: the OpenMP default).  The whole
 * list is validated first (QC_ERR_INVALID_ARG, state untouched).  Blocks. */
qc_status qc_omp_run(int n, qc_precision p, void* x, const qc_gate* ops, size_t n_ops, int nthreads);

/* OpenMP threads a parallel region of qc_omp_run would use (nthreads = 0). */
int qc_omp_max_threads(void);

/* Thread-local message of the last failing qc_omp_* call. */
const char* qc_omp_last_error(void);

#ifdef __cplusplus
}
#endif
#endif /* QC_OMP_H_ */
