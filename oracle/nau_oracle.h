/* oracle/nau_oracle.h — TEST INFRASTRUCTURE, not product code.
 *
 * Plain-C restatement of the reference's particle hot path (Nauticle,
 * /root/reference/proj), used only by tests/, __graft_entry__.smoke() and
 * bench.py's cpu_baseline / reference legs as the CHECKER. The product path
 * (paper_1710_08259_b200/) never links or calls this.
 *
 * Parity pinning: every function here is checked in tests/test_oracle.py
 * against oracle/_ref/libnauticle_ref.so (the reference sources compiled
 * unmodified against oracle/shim/) and against the committed golden fixtures
 * in tests/golden/ (made by tests/golden/make_golden.py from that build).
 * Arithmetic follows the reference's operation order with no FMA contraction
 * (compiled -ffp-contract=off), so results are bitwise equal to oracle/_ref.
 */
#ifndef NAU_ORACLE_H
#define NAU_ORACLE_H

#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

enum { NOR_PERIODIC = 0, NOR_SYMMETRIC = 1, NOR_CUTOFF = 2 };

/* Operator codes: same numbering as include/nauticle_gpu.h (NAU_OP_*). */
enum {
    NOR_SPH_S = 0, NOR_SPH_D00 = 1, NOR_SPH_G11 = 2, NOR_SPH_L0 = 3, NOR_SPH_A = 4,
    NOR_DEM_HERTZ = 5, NOR_DEM_BOUNDARY = 6, NOR_GRAVITY = 7, NOR_DEM_LSD = 8, NOR_SFM = 9
};
enum { NOR_K_WENDLAND = 0, NOR_K_CUBIC = 1 };

typedef struct {
    int dim;
    int cells[3];
    double lo[3], hi[3], ext[3], cs[3];
    int kind[3];
} nor_domain;

/* A per-particle field (SoA, component-major: field[c*n + i]) or a uniform value. */
typedef struct {
    const double* field;
    double value[9];
    int rows, cols;
} nor_operand;

typedef struct {
    nor_domain dom;
    int n;
    const double* pos;      /* dim x n, component-major */
    const uint8_t* active;  /* n */
    const int* cell_of;     /* n: flat cell, -1 if inactive */
    const int* cell_start;  /* ncells */
    const int* cell_count;  /* ncells */
    const int* sorted;      /* active particles in cell order */
    long warnings;
} nor_ps;

void nor_domain_init(nor_domain* d, int dim, const int* min_cells, const int* max_cells,
                     const double* cell_size, const int* kinds);
long nor_ncells(const nor_domain* d);
int nor_cell_index(const nor_domain* d, int axis, double x);
/* Returns 0, or 1 + index of the first active particle outside a cutoff axis. */
long nor_build_cells(const nor_domain* d, int n, const double* pos, const uint8_t* active,
                     int* cell_of, int* cell_start, int* cell_count, int* sorted);
/* Returns the number of symmetric-overflow warnings; deactivates cutoff leavers. */
long nor_boundary_shift(const nor_domain* d, int n, double* pos, uint8_t* active);
void nor_neighbor_counts(nor_ps* ps, double radius, int* counts);

double nor_kernel_value(int family, int kdim, double h, double d);
double nor_kernel_dq(int family, int kdim, double h, double q);

/* out: SoA of the result shape (component-major, stride n); inactive particles
 * are left untouched. Returns 0, or an error: 1 + first offending particle
 * index is written to *bad and the return value is 1 (runtime error).
 * Operand order follows the reference's kOps[] (interactions.cpp:259-269)
 * with the kernel keyword slot removed. */
int nor_interact(int op, int kfamily, int kdim, nor_ps* ps, const nor_operand* ops, int nops,
                 double* out, int out_comps, long* bad);

/* euler: out = x + xdot*dt (ast.cpp:180-191), active particles only. */
void nor_euler(int n, int comps, const uint8_t* active, const double* x, const double* xdot,
               double dt, double* out);

/* The reference's counter RNG (random_state.hpp:22-30): out[k*n+i] = draw k of i. */
void nor_uniform_draws(uint64_t seed, int n, int ndraws, double a, double b, double* out);

#ifdef __cplusplus
}
#endif
#endif
