/*
 * oracle/laplex_oracle.c -- CPU restatement of the LAPLEX reference hot path.
 *
 * TEST INFRASTRUCTURE ONLY.  This is the checker, never the product: only
 * tests/, __graft_entry__.smoke() and bench.py's cpu_baseline leg may load it.
 * It restates, function by function, the algorithms in the reference C++
 * headers (/root/reference/proj/include/laplex/{scan,operator,gradients,
 * oracle}.hpp) in plain C so that it runs on the GPU box where the reference
 * tree does not exist.  Parity is pinned by tests/test_oracle_cpu.py against
 * (a) the known-answer vectors in the reference's own tests and SPEC and
 * (b) golden fixtures produced by the compiled reference (oracle/_ref).
 *
 * Build: see oracle/Makefile (gcc -O2 -fPIC -shared, no fast-math).
 */
#include <math.h>
#include <stddef.h>
#include <stdint.h>
#include <stdlib.h>
#include <string.h>

#define LXO_OK 0
#define LXO_EMPTY_INPUT 1
#define LXO_NON_FINITE 2
#define LXO_DIMENSION_MISMATCH 3
#define LXO_PHASE_PRESENT 4
#define LXO_PHASE_ABSENT 5
#define LXO_ASYMMETRIC_COTANGENT 6

#ifdef _OPENMP
#include <omp.h>
#endif

/* Threads of the calling thread's parallel loops (OpenMP ICVs are per thread):
   callers that run several oracle calls concurrently set 1.  The results do not
   depend on it. */
void lxo_set_num_threads(int n) {
#ifdef _OPENMP
    omp_set_num_threads(n > 0 ? n : 1);
#else
    (void)n;
#endif
}

/* double instantiation */
#define REAL double
#define SFX _f64
#define EXP exp
#define COS cos
#define SIN sin
#define FABS fabs
#include "lxo_impl.inc"
#undef REAL
#undef SFX
#undef EXP
#undef COS
#undef SIN
#undef FABS

/* float instantiation (std::exp(float) == expf in libstdc++) */
#define REAL float
#define SFX _f32
#define EXP expf
#define COS cosf
#define SIN sinf
#define FABS fabsf
#include "lxo_impl.inc"
#undef REAL
#undef SFX
#undef EXP
#undef COS
#undef SIN
#undef FABS
