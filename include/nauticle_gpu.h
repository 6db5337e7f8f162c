/* include/nauticle_gpu.h — C-ABI of the B200-native Nauticle particle hot path.
 *
 * Built as paper_1710_08259_b200/libnau_b200.so (hand-written sm_100a CUDA +
 * a thin C++ host layer). No torch types, plain pointers and sizes only.
 *
 * Why the boundary sits one level above the reference's plugin type
 * (SURVEY.md §8(b)): the reference's operator plugin
 *     struct InteractionOp { name, arity_min, arity_max, kernel_slot, radius_slot,
 *                            finite_influence, Tensor (*eval)(node, int i, int level) }
 * (include/nauticle/interactions.hpp:13-21, registry kOps[] src/interactions.cpp:259-269)
 * is called once per particle i from Case::solve_equation's thread blocks
 * (src/case.cpp:31-54). Across a C ABI to a GPU that would be one launch per
 * particle, so every entry point here is a whole-field operation that takes
 * over the per-equation loop instead. Each function names the reference code it
 * replaces. Ownership: a context owns all device memory; the host keeps names,
 * shapes and equation trees and maps names to field ids.
 *
 * Threading: a context is bound to one host thread and one CUDA stream; calls
 * are stream-ordered and asynchronous unless they return host data. Device-side
 * failures (zero density, cut-off leavers at cell build, non-finite results)
 * are latched in a device error word and surface at the next nau_sync() (or any
 * call that returns host data) — the reference throws nauticle::Error{Runtime|Nan}
 * (include/nauticle/error.hpp:10-69) at the same points.
 *
 * Data order: fields live on the device in CELL order (sorted by the last
 * nau_build_cells). Every host-facing array (upload/download/tables/counts) is
 * in ORIGINAL particle-index order, as the reference's std::vector<Tensor> is.
 */
#ifndef NAUTICLE_GPU_H
#define NAUTICLE_GPU_H

#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

typedef struct nau_ctx nau_ctx;

typedef enum {
    NAU_OK = 0,
    NAU_ERR_RUNTIME = 1, /* nauticle::ErrorKind::Runtime */
    NAU_ERR_NAN = 2,     /* nauticle::ErrorKind::Nan (case.cpp:46-53 audit) */
    NAU_ERR_CUDA = 3,
    NAU_ERR_ARG = 4,     /* ≙ Assembly/Parse errors of bad calls */
    NAU_ERR_COMM = 5
} nau_status;

/* BoundaryKind (include/nauticle/domain.hpp:8) */
enum { NAU_PERIODIC = 0, NAU_SYMMETRIC = 1, NAU_CUTOFF = 2 };

/* Interaction operators: one per kOps[] row (src/interactions.cpp:259-269),
 * plus NAU_OP_DEM_LSD, the linear spring-dashpot law BASELINE cfg3 needs. */
enum {
    NAU_OP_SPH_S = 0,        /* sph_S   (A, m, rho, K, R)  interactions.cpp:40-58   */
    NAU_OP_SPH_D00 = 1,      /* sph_D00 (A, m, rho, K, R)  interactions.cpp:60-79   */
    NAU_OP_SPH_G11 = 2,      /* sph_G11 (A, m, rho, K, R)  interactions.cpp:81-102  */
    NAU_OP_SPH_L0 = 3,       /* sph_L0  (A, m, rho, K, R)  interactions.cpp:104-126 */
    NAU_OP_SPH_A = 4,        /* sph_A   (v, m, rho, K, R)  interactions.cpp:128-150 */
    NAU_OP_DEM_HERTZ = 5,    /* dem_l   (v,R,E,nu,m,cf,Rs) interactions.cpp:152-188 */
    NAU_OP_DEM_BOUNDARY = 6, /* dem_boundary_force         interactions.cpp:190-193 */
    NAU_OP_GRAVITY = 7,      /* nbody_gravity (m, G, eps)  interactions.cpp:195-214 */
    NAU_OP_DEM_LSD = 8,      /* dem_lsd (v,R,kn,en,m,cf,Rs) new: linear spring-dashpot + Coulomb */
    NAU_OP_SFM = 9,          /* sfm (v, v0, r_d, R, A, B, k, c, m, tau)  interactions.cpp:216-257 */
    NAU_OP_COUNT = 10
};

/* Smoothing-kernel families: Wendland (keywords Wp5D220, src/kernel.cpp:9-69)
 * and the cubic spline (keywords Wc3D220, new). */
enum { NAU_K_WENDLAND = 0, NAU_K_CUBIC = 1 };

/* Mirror of InteractionOp's metadata (interactions.hpp:13-21). */
typedef struct {
    const char* name;
    int op;
    int arity_min, arity_max;
    int kernel_slot; /* operand that must be a kernel keyword, -1 if none */
    int radius_slot; /* operand holding the influence radius, -1 if none  */
    int finite_influence;
} nau_op_info;

/* ≙ find_interaction(name) (interactions.cpp:273-277). Returns NAU_ERR_ARG if unknown. */
nau_status nau_find_interaction(const char* name, nau_op_info* out);
/* ≙ decode_kernel_keyword (kernel.cpp:20-35): "Wp5D220" or "Wc3D220". */
nau_status nau_decode_kernel(const char* keyword, int* family, int* dim);

/* ---- context ---- */
nau_status nau_create(int device, nau_ctx** out);
void nau_destroy(nau_ctx* ctx);

/* Evaluation mode of the neighbour sums.
 * EXACT (default): candidates summed in the reference's order with the
 *   reference's arithmetic (no FMA, IEEE div/sqrt): bitwise equal to the
 *   reference wherever no libm transcendental is involved.
 * FAST: same candidates, filters and error checks, FMA/rsqrt/reciprocal
 *   arithmetic and a balanced candidate order (BASELINE tolerance: 1e-10
 *   relative; observed ~1e-14). */
enum { NAU_MODE_EXACT = 0, NAU_MODE_FAST = 1 };
nau_status nau_set_mode(nau_ctx* ctx, int mode);
int nau_get_mode(nau_ctx* ctx);
/* Neighbour lists (default on): the candidate scan runs once per cell build and
 * every SPH operator with a uniform radius (nau_interact, nau_wcsph_step) reads
 * the list; same candidates in the same order, so results are identical either
 * way. on = 0: each pass sweeps the cells itself; 1: lists (paired lists for the
 * FAST-mode Wendland nau_wcsph_step: one thread per two particles, shared
 * gathers); 2: lists, per-particle only. */
nau_status nau_set_neighbor_lists(nau_ctx* ctx, int on);
/* Use an external CUDA stream (cudaStream_t), e.g. torch's current stream. NULL = own stream. */
nau_status nau_set_stream(nau_ctx* ctx, void* stream);
void* nau_get_stream(nau_ctx* ctx);

/* ≙ Domain(dim, min_cells, max_cells, cell_size, boundary) (domain.cpp:27-47). */
nau_status nau_set_domain(nau_ctx* ctx, int dim, const int* min_cells, const int* max_cells,
                          const double* cell_size, const int* kind);

/* ≙ ParticleSystem(domain, positions) (particle_system.cpp:8-18): sets n and
 * field 0 = r (dim x 1) from a host SoA (component-major, pos[a*n + i]); all
 * particles active. Frees previous fields. Does not shift or build cells. */
nau_status nau_set_particles(nau_ctx* ctx, long n, const double* pos_soa);
long nau_particle_count(nau_ctx* ctx);
/* ≙ ParticleSystem::active_count(); syncs. */
long nau_active_count(nau_ctx* ctx);
/* Host copy of the active flags in original order (≙ is_active(i)). */
nau_status nau_get_active(nau_ctx* ctx, uint8_t* active);

/* ≙ Workspace::add_field (workspace.cpp:39-48): new field of rows x cols per particle. */
nau_status nau_alloc_field(nau_ctx* ctx, int rows, int cols, int* field_id);
nau_status nau_free_field(nau_ctx* ctx, int field_id);
nau_status nau_field_shape(nau_ctx* ctx, int field_id, int* rows, int* cols);
/* host SoA, component-major [c*n + i] with c = col*rows + row, original order */
nau_status nau_upload(nau_ctx* ctx, int field_id, const double* soa, long n);
nau_status nau_download(nau_ctx* ctx, int field_id, double* soa, long n);
/* Asynchronous host I/O (same layout as nau_upload / nau_download). The copies run
 * on the context's copy streams (one per direction) through per-field
 * double-buffered staging, so a step's uploads and downloads overlap the
 * neighbour passes of the steps around it. Host buffers should be pinned; an
 * upload's source must stay unchanged, and a download's destination is valid,
 * only after nau_sync. nau_io_fence orders later copies after the work enqueued
 * so far on the context stream; nau_io_join makes the context stream wait for
 * every enqueued copy (a device-side join, e.g. before a timing event). */
nau_status nau_upload_async(nau_ctx* ctx, int field_id, const double* soa, long n);
nau_status nau_download_async(nau_ctx* ctx, int field_id, double* soa, long n);
nau_status nau_io_fence(nau_ctx* ctx);
nau_status nau_io_join(nau_ctx* ctx);
/* Uniform value (rows*cols doubles, column-major) into every particle. */
nau_status nau_fill(nau_ctx* ctx, int field_id, const double* value);
nau_status nau_copy_field(nau_ctx* ctx, int dst, int src);
/* Device pointer of a field's storage (cell order; valid until the next build). */
nau_status nau_field_device_ptr(nau_ctx* ctx, int field_id, double** ptr);

/* ≙ ParticleSystem::apply_boundary_shift (particle_system.cpp:56-90): periodic
 * wrap, symmetric-overflow warnings, cut-off deactivation; marks cells dirty. */
nau_status nau_boundary_shift(nau_ctx* ctx);
/* ≙ ParticleSystem::build_cells (particle_system.cpp:33-54): cell hash, stable
 * (cell, original index) ordering, cell start/count tables, SoA reorder. */
nau_status nau_build_cells(nau_ctx* ctx);
int nau_cells_dirty(nau_ctx* ctx);
long nau_rebuild_count(nau_ctx* ctx);
long nau_warning_count(nau_ctx* ctx); /* syncs */
long nau_ncells(nau_ctx* ctx);
/* Parity probe (host arrays): cell_of_particle[n] (flat cell, -1 inactive),
 * cell_start[ncells], cell_count[ncells], sorted_ids[n_active] (original
 * indices, ascending within a cell) — the reference's cells_ concatenated. */
nau_status nau_cell_tables(nau_ctx* ctx, int* cell_of_particle, int* cell_start, int* cell_count,
                           int* sorted_ids);
/* Parity probe: counts[i] = candidates of for_each_neighbor(i) (particle_system.hpp:59-138)
 * with |rel| <= radius, self included; original order. */
nau_status nau_neighbor_counts(nau_ctx* ctx, double radius, int* counts);

/* An operand: a field reference (field_id >= 0) or a uniform value (field_id = -1,
 * rows x cols doubles in value[], column-major). ≙ FieldRefNode / ConstantRefNode /
 * VariableRefNode / LiteralNode (include/nauticle/sfl/ast.hpp:70-109). */
typedef struct {
    int field_id;
    int rows, cols;
    double value[9];
} nau_operand;

/* ≙ InteractionOp::eval for every active particle (the whole-field form of
 * interact(), interactions.hpp:29-36). Operands follow kOps[] order with the
 * kernel-keyword slot removed: SPH (A, m, rho, R); DEM (v, R, E|kn, nu|en, m, cf, Rs);
 * gravity (m, G[, eps]). Writes active particles of out_field (inactive keep
 * their value, case.cpp:37-40); out_field may alias an operand (two-phase). */
nau_status nau_interact(nau_ctx* ctx, int op, int kernel_family, int kernel_dim,
                        const nau_operand* ops, int n_ops, int out_field);

/* Two consecutive equations  out_g = sph_G11(A, m, rho, K, R);  out_l = sph_L0(A, m,
 * rho, K, R)  (interactions.cpp:81-126, evaluated in listed order by Case::solve_step,
 * case.cpp:9-67). Neither reads the other's output, so in FAST mode one walk of the
 * neighbour list evaluates both sums (one gather per neighbour); results, errors and
 * warnings equal the two nau_interact calls. Any other case (EXACT mode, an output
 * aliasing an operand, bad shapes) runs exactly those two calls. */
nau_status nau_interact_g11_l0(nau_ctx* ctx, int kernel_family, int kernel_dim,
                               const nau_operand* ops, int n_ops, int out_g, int out_l);

/* ≙ EulerNode (sfl/ast.cpp:180-191): out = x + xdot*dt on active particles. */
nau_status nau_euler(nau_ctx* ctx, int x, int xdot, double dt, int out_field);

/* Fused symplectic-Euler update of the BASELINE decks, one kernel:
 *   v = euler(v, vdot*mask, dt); r = euler(r, v, dt); apply_boundary_shift()
 * (dam_break_2d.yaml:37-38 order; case.cpp:59-62). mask_field = -1 means no mask. */
nau_status nau_symplectic_step(nau_ctx* ctx, int v, int vdot, int mask_field, double dt);

/* Weakly-compressible SPH deck (BASELINE cfg0/cfg2), fused into three passes:
 *   rho  = sph_S(one, m, one, K, R)                    -> p = B*((rho/rho0)^gamma - 1)
 *   vdot = -1/rho*sph_G11(p,m,rho,K,R) + visc*sph_A(v,m,rho,K,R) + g
 *   v = euler(v, vdot*mask, dt); r = euler(r, v, dt); boundary shift
 * (visc = alpha*c0*h). Field ids: rho, p, v, vdot, mask (-1 none). */
typedef struct {
    int kernel_family, kernel_dim;
    double mass, radius, rho0, B, gamma, visc, dt;
    double g[3];
    int f_rho, f_p, f_v, f_vdot, f_mask;
} nau_wcsph_params;
nau_status nau_wcsph_step(nau_ctx* ctx, const nau_wcsph_params* prm);
/* The step's passes one at a time (multi-GPU slabs exchange halo values between
 * them): 0 = cell build + neighbour list + density/EOS, 1 = momentum
 * (after pass 0 of the same build), 2 = symplectic update + boundary shift. */
nau_status nau_wcsph_pass(nau_ctx* ctx, const nau_wcsph_params* prm, int pass);
/* nau_wcsph_step runs without host synchronisation and, after two warm-up calls, is
 * captured into a CUDA graph replayed for later steps that start from the same host
 * state (default on; NAU_GRAPHS=0 in the environment or on = 0 here disables it). */
nau_status nau_set_graphs(nau_ctx* ctx, int on);

/* DEM deck (BASELINE cfg3), the reference's equation form:
 *   vdot = law(v, R, P, Q, m, cf, Rs) + g;  v = euler(v, vdot, dt);  r = euler(r, v, dt)
 * law = NAU_OP_DEM_LSD (P = kn, Q = en) or NAU_OP_DEM_HERTZ (P = E, Q = nu);
 * f_R / f_m = -1 use the uniform R / m. Boundary shift after the r update. */
typedef struct {
    int law;
    int f_v, f_vdot, f_R, f_m;
    double R, m, P, Q, cf, search_radius, dt;
    double g[3];
} nau_dem_params;
nau_status nau_dem_step(nau_ctx* ctx, const nau_dem_params* prm);

/* Leapfrog all-pairs gravity (BASELINE cfg4), kick-drift-kick as equation order:
 *   v = euler(v, a, dt/2); r = euler(r, v, dt); a = nbody_gravity(m, G, eps);
 *   v = euler(v, a, dt/2).   f_m = -1 uses the uniform m. No cells are built
 * (nbody_gravity has finite_influence = false, interactions.cpp:267). */
typedef struct {
    int f_v, f_a, f_m;
    double m, G, eps, dt;
} nau_gravity_params;
nau_status nau_leapfrog_step(nau_ctx* ctx, const nau_gravity_params* prm);

/* Sharded n-body: every rank holds a contiguous block of
 * bodies; the sources are all-gathered each step (NCCL) as (x, y, z, m) rows.
 * nau_pack_sources writes this rank's rows (m = 0 for inactive bodies; f_m = -1
 * uses the uniform m) into dev_rows (n x 4 doubles, original order — gravity
 * never builds cells). nau_gravity_sources: out_field = nbody_gravity(m, G, eps)
 * of the local bodies against all nsrc sources, skipping source self_off + k for
 * local body k, summed in global source order (= the single-GPU order). */
nau_status nau_pack_sources(nau_ctx* ctx, int f_m, double m, double* dev_rows);
nau_status nau_gravity_sources(nau_ctx* ctx, const double* dev_src, long nsrc, long self_off,
                               double G, double eps, int out_field);
/* One chunk of the sources: with accumulate != 0 the sums continue from the values
 * already in out_field, so chunks evaluated in global order (0, 1, ...) give the sums
 * of one nau_gravity_sources call over all of them bit for bit. self_off is relative
 * to the chunk (local body k is the chunk's source self_off + k; out of range: none).
 * Lets the host overlap the transfer of chunk c + 1 with the pair loop over chunk c
 * (the all-gather "can be ring-pipelined with compute"). */
nau_status nau_gravity_sources_part(nau_ctx* ctx, const double* dev_src, long nsrc, long self_off,
                                    double G, double eps, int out_field, int accumulate);

/* ≙ ReductionNode fsum/fmax/fmin/fmean over active particles (sfl/ast.cpp:237-274).
 * kind: 0 max, 1 min, 2 sum, 3 mean; out has rows*cols doubles (max/min: 1). */
nau_status nau_reduce(nau_ctx* ctx, int kind, int field_id, double* out);

/* ---- device evaluator for SFL particle-wise arithmetic ----
 * A register program the host lowers an sfl::ExpressionNode tree to (one
 * instruction per node, post-order; INTEGRATION.md shows the lowering). Every
 * register holds one Tensor per particle (rows x cols <= 3 x 3, column-major
 * components), its shape fixed by the program. Semantics are those of the
 * reference's Tensor operators (tensor.cpp:43-126) and AST nodes (sfl/ast.cpp:
 * 71-175): + - need equal shapes; * is scalar scaling or the matrix product
 * (inner index summed in order); / divides by a scalar or elementwise; ^, min,
 * max are elementwise with scalar broadcast (std::pow / fmin / fmax);
 * comparisons take scalars and give 1 or 0; '|' appends a scalar to a column
 * (<= 3 rows); dot and norm reduce in storage order. Field, constant and
 * variable references load per-particle or uniform values (LOAD_FIELD /
 * LOAD_CONST; reductions and interactions are evaluated beforehand into a
 * uniform value or a field, as the reference freezes / evaluates them). */
enum {
    NAU_VM_LOAD_FIELD = 0, /* dst <- field `field` (its shape)          FieldRefNode      */
    NAU_VM_LOAD_CONST = 1, /* dst <- imm (rows x cols)                   Literal/Constant/Variable */
    NAU_VM_ADD = 2, NAU_VM_SUB = 3, NAU_VM_MUL = 4, NAU_VM_DIV = 5, NAU_VM_POW = 6,
    NAU_VM_LT = 7, NAU_VM_GT = 8, NAU_VM_LE = 9, NAU_VM_GE = 10, NAU_VM_EQ = 11, NAU_VM_NE = 12,
    NAU_VM_NEG = 13,       /* UnaryMinusNode                                                */
    NAU_VM_JOIN = 14,      /* VectorJoinNode a | b                                          */
    NAU_VM_EXP = 15, NAU_VM_LOG = 16, NAU_VM_SIN = 17, NAU_VM_COS = 18, NAU_VM_TAN = 19,
    NAU_VM_SQRT = 20, NAU_VM_ABS = 21, NAU_VM_FLOOR = 22, NAU_VM_SGN = 23, NAU_VM_NORM = 24,
    NAU_VM_MIN = 25, NAU_VM_MAX = 26, NAU_VM_DOT = 27,
    NAU_VM_RAND = 28,      /* RandNode rand(a, b): RandomState::uniform(i, a, b)        */
    NAU_VM_OP_COUNT = 29
};
typedef struct {
    int op;
    int dst, a, b;       /* registers (a, b: operands; unused ones ignored)      */
    int field;           /* NAU_VM_LOAD_FIELD                                     */
    int rows, cols;      /* NAU_VM_LOAD_CONST shape (other ops: derived, ignored) */
    double imm[9];       /* NAU_VM_LOAD_CONST value, column-major                 */
} nau_vm_instr;
enum { NAU_VM_MAX_INSTR = 128, NAU_VM_MAX_REGS = 16 };
/* out_field = register `result` for every active particle; inactive particles
 * keep their value (case.cpp:36-40); the output may alias an input field
 * (two-phase write, case.cpp:31-54). Shape errors fail here with the reference's
 * message ("operator '+': incompatible shapes 3x1 and 1x1"); a non-finite result
 * fails at nau_sync with the lowest original index (the NaN audit, case.cpp:46-53). */
nau_status nau_eval(nau_ctx* ctx, const nau_vm_instr* code, int n_instr, int result,
                    int out_field);
/* ≙ the case's RandomState (sfl/random_state.hpp): every `rand` draw is a pure
 * function of (seed, original particle index, that particle's draw counter).
 * counters: n values in original order, or NULL for zeros (a fresh case). The
 * counters persist across nau_eval calls like the reference's (hot start writes
 * them back, scheduler.cpp:47-54). */
nau_status nau_set_random_state(nau_ctx* ctx, unsigned long long seed,
                                const unsigned long long* counters);
nau_status nau_get_random_counters(nau_ctx* ctx, unsigned long long* counters);

/* ---- host equation executor (≙ Case::solve_equation / Case::solve_step,
 * case.cpp:9-67; the §8(b) "Caller"; csrc/executor.cpp) ----
 * Runs an arbitrary deck's equation list on the device: each equation's text
 * ("lhs=rhs", the reference's canonical Equation::to_text form) is parsed with the
 * reference's SFL grammar (sfl/parser.cpp) against the case's symbols; every solve
 * folds uniform subtrees on the host (constants, variables, literals, frozen
 * reductions), runs interactions through nau_interact into temporaries (operand
 * subtrees materialised once per equation), reductions through nau_reduce +
 * nau_allreduce, and the particle-wise rest as one nau_eval program into the LHS
 * field (two-phase, NaN audit, boundary shift after r). A variable LHS takes the
 * value at particle 0 (case.cpp:19-29). Errors: the reference's kinds and messages,
 * prefixed "equation '<name>': "; nau_case_last_error gives the text and the
 * first bad particle. Extensions over the reference's grammar: the cubic-spline
 * keywords (Wc1D220..Wc3D220) and the dem_lsd law. Not supported: rand() inside an
 * interaction operand (the reference draws it per neighbour). */
typedef struct nau_case nau_case;
nau_status nau_case_create(nau_ctx* ctx, nau_case** out); /* after nau_set_particles */
void nau_case_destroy(nau_case* cs);
/* Uniform symbols: rows x cols <= 3 x 3, column-major. */
nau_status nau_case_constant(nau_case* cs, const char* name, int rows, int cols, const double* v);
nau_status nau_case_variable(nau_case* cs, const char* name, int rows, int cols, const double* v);
nau_status nau_case_set_variable(nau_case* cs, const char* name, int rows, int cols,
                                 const double* v);
nau_status nau_case_get_variable(nau_case* cs, const char* name, double* v /* 9 */, int* rows,
                                 int* cols);
/* Names a context field (nau_alloc_field id); "r" is field 0 and always defined. */
nau_status nau_case_field(nau_case* cs, const char* name, int field_id);
/* Appends an equation (parsed now; symbols must already be defined). */
nau_status nau_case_equation(nau_case* cs, const char* name, const char* text);
int nau_case_equation_count(nau_case* cs);
nau_status nau_case_solve_equation(nau_case* cs, int index);
nau_status nau_case_solve_step(nau_case* cs); /* every equation in order */
const char* nau_case_last_error(nau_case* cs, long* first_bad_particle);

/* ---- multi-GPU slab decomposition (no reference counterpart:
 * the reference has no domain decomposition) ----
 * Rows are particle-major: every live field in id order (r first), rows x cols
 * doubles each; nau_row_width() doubles per particle. Device pointers. */
int nau_row_width(nau_ctx* ctx);
/* Slots (cell order) of active particles whose cell index along `axis`
 * (particle_system.cpp:20-31) is in [lo, hi) and, if flag_field >= 0,
 * flag_lo <= flag <= flag_hi; ascending slot order. Syncs. */
nau_status nau_select(nau_ctx* ctx, int axis, double lo, double hi, int flag_field,
                      double flag_lo, double flag_hi, int* dev_slots, long* count);
nau_status nau_pack_rows(nau_ctx* ctx, const int* dev_slots, long m, double* dev_rows);
/* Replace all particles by m rows (all active). gid_field >= 0 names a scalar
 * field holding global particle indices: cells then list particles in ascending
 * global index, so sums keep the single-GPU order. Marks cells dirty. */
nau_status nau_load_rows(nau_ctx* ctx, const double* dev_rows, long m, int gid_field);
/* x-threshold slabs (slab.py): slots of active particles with coordinate `axis` in
 * [xlo, xhi) and flag in [flag_lo, flag_hi], ascending slot order. Syncs. */
nau_status nau_select_x(nau_ctx* ctx, int axis, double xlo, double xhi, int flag_field,
                        double flag_lo, double flag_hi, int* dev_slots, long* count);
/* Capacity for up to `cap` particles (before loading: contents are dropped). */
nau_status nau_reserve(nau_ctx* ctx, long cap);
/* In place: the particle set becomes the kept slots (in the given order) followed by
 * m_new rows (nau_row_width layout, gid_field as in nau_load_rows); one pass over the
 * kept particles. Marks cells dirty. */
nau_status nau_rebuild_rows(nau_ctx* ctx, const int* dev_keep, long m_keep,
                            const double* dev_rows, long m_new, int gid_field);
/* Per-bin counts (device, unsigned 64-bit) of active particles with coordinate `axis`
 * in nbins equal bins over [x0, x1) (clamped), flag in [flag_lo, flag_hi]. */
nau_status nau_histogram_x(nau_ctx* ctx, int axis, double x0, double x1, int nbins,
                           int flag_field, double flag_lo, double flag_hi,
                           unsigned long long* dev_counts);
/* Ghosts: particles whose scalar field `field_id` is non-zero take part in every sum
 * as neighbours but are not evaluated or integrated (their values come from the rank
 * that owns them); -1 switches this off. */
nau_status nau_set_ghost_field(nau_ctx* ctx, int field_id);
/* Halo values of the WCSPH deck between its passes (the Python driver): (rho, p) rows
 * of the given slots, and back into ghost slots with the momentum payload
 * (v, p / rho^2) they imply. */
nau_status nau_wcsph_pack_rho_p(nau_ctx* ctx, const nau_wcsph_params* prm, const int* dev_slots,
                                long m, double* dev_rows);
nau_status nau_wcsph_ghost_update(nau_ctx* ctx, const nau_wcsph_params* prm, const int* dev_slots,
                                  long m, const double* dev_rows);

/* ---- native slab exchange over NCCL (nau_comm_init /
 * nau_halo_exchange / nau_migrate; comm.cu). One context per GPU and process;
 * the caller ships the 128-byte id from rank 0 to the others (torch.distributed,
 * MPI, a file). NCCL is bound at run time: NAU_ERR_COMM if absent. ---- */
#define NAU_COMM_ID_BYTES 128
nau_status nau_comm_unique_id(unsigned char* id_out /* NAU_COMM_ID_BYTES */);
nau_status nau_comm_init(nau_ctx* ctx, const unsigned char* id, int nranks, int rank);
void nau_comm_destroy(nau_ctx* ctx);
/* x-threshold slabs: rank r owns the particles with coordinate
 * `axis` in [bounds[r], bounds[r+1]) (nranks + 1 values from the domain's lo to hi,
 * every slab at least 2 radius wide) and holds ghosts: its neighbours' particles within
 * `radius` of its faces, flag_field 1 (owned by the left neighbour) or 2 (right), which
 * take part in every sum but are not evaluated or integrated (nau_set_ghost_field).
 * gid_field holds global indices (the within-cell sort key). */
nau_status nau_slab_config(nau_ctx* ctx, int axis, const double* bounds, int periodic,
                           double radius, int gid_field, int flag_field);
nau_status nau_slab_bounds(nau_ctx* ctx, double* bounds_out /* nranks + 1 */);
/* Migration + halo after the integrator, one exchange round: owned particles that left
 * the slab go to the neighbour (less than radius past the face, else NAU_ERR_COMM),
 * owned particles within radius of a face go to that neighbour as ghosts, emigrants
 * stay as ghosts of their new owner; the local set is rebuilt in place. Syncs. */
nau_status nau_migrate(nau_ctx* ctx);
/* Halo values between passes: the listed fields of every owned particle within radius
 * of a face to that neighbour, into its ghosts of that face (same slot order on both
 * sides: the global cell grid ordered by global id). Syncs. */
nau_status nau_halo_exchange(nau_ctx* ctx, const int* field_ids, int nfields);
/* Re-balancing: bounds from the all-reduced nbins-bin x-histogram of owned particles,
 * owned particles hop to their new owner, then a new halo. Syncs. */
nau_status nau_slab_rebalance(nau_ctx* ctx, int nbins);
/* Field subsets of selected slots as rows (width = the fields' components) and back. */
nau_status nau_pack_fields(nau_ctx* ctx, const int* dev_slots, long m, const int* field_ids,
                           int nfields, double* dev_rows);
nau_status nau_unpack_fields(nau_ctx* ctx, const int* dev_slots, long m, const int* field_ids,
                             int nfields, const double* dev_rows);
/* The WCSPH momentum payload (v, p / rho^2) of every ghost from its fields (after a
 * nau_halo_exchange of rho and p). */
nau_status nau_wcsph_ghost_payload(nau_ctx* ctx, const nau_wcsph_params* prm);
/* The primitive under both: swap device row blocks (width doubles per row) with
 * the left / right neighbours; received blocks stay valid until the next call. */
nau_status nau_comm_swap(nau_ctx* ctx, const double* to_left, long n_left, const double* to_right,
                         long n_right, int width, const double** from_left, long* nf_left,
                         const double** from_right, long* nf_right);
/* ≙ the ncclAllReduce of SURVEY.md §8(e) "Reductions": host values combined over the
 * ranks of the context's communicator (op 0 sum, 1 max, 2 min), in place. Without a
 * communicator the values are left as they are. Syncs. */
nau_status nau_allreduce(nau_ctx* ctx, double* values, int count, int op);
/* Ranks of the context's communicator (1 without nau_comm_init). */
int nau_comm_size(nau_ctx* ctx);

/* ---- result frames and hot start (frames.cu) ----
 * Legacy VTK PolyData exactly as the reference writes it (io/vtk.cpp:193-304):
 * particles in original index order, scalars as SCALARS, d-vectors padded to 3
 * as VECTORS, other shapes in FIELD PerParticle, big-endian doubles in BINARY
 * files. The strings the host owns (the deck's equations, variables,
 * constants, parameters) are passed as the reference formats them. */
typedef struct {
    int frame_index;
    double time;
    const char* domain_text;          /* NULL: built from the context (domain.cpp:68-83) */
    const char* params_text;          /* "simulated_time=..." (vtk.cpp:204-206) */
    int n_variables;
    const char* const* variables;     /* "name=value" each (tensor.cpp:128-150) */
    int n_constants;
    const char* const* constants;
    int n_equations;
    const char* const* equations;     /* Equation::to_text() each */
    int n_fields;                     /* workspace order, r excluded */
    const int* field_ids;
    const char* const* field_names;
} nau_frame_meta;
nau_status nau_write_vtk(nau_ctx* ctx, const char* path, int binary, const nau_frame_meta* meta);
/* Reader (read_vtk, vtk.cpp:310-464): a host-side frame for a hot start. */
typedef struct nau_vtk_frame nau_vtk_frame;
nau_status nau_vtk_read(const char* path, nau_vtk_frame** out);
void nau_vtk_free(nau_vtk_frame* frame);
const char* nau_vtk_last_error(void);
/* particle count; positions dim x n component-major, original order */
long nau_vtk_points(const nau_vtk_frame* frame, int* dim, int* frame_index, double* time,
                    const double** pos_soa);
int nau_vtk_array_count(const nau_vtk_frame* frame);
/* name of point array k; soa component-major [(col*rows + row)*n + i] */
const char* nau_vtk_array(const nau_vtk_frame* frame, int k, int* rows, int* cols,
                          const double** soa);
/* CaseData string array `key` (domain, params, field_shapes, variables, constants, equations) */
int nau_vtk_strings(const nau_vtk_frame* frame, const char* key, const char* const** items);
long nau_vtk_rand_counters(const nau_vtk_frame* frame, const unsigned long long** counters);

/* Surfaces latched device errors (≙ the exceptions above). */
nau_status nau_sync(nau_ctx* ctx);
/* Message of the last error and the lowest original particle index involved (-1 if none). */
const char* nau_last_error(nau_ctx* ctx, long* first_bad_particle);

/* Instrumentation for bench.py: record CUDA events around every launch of the
 * named kernel class (0 none, 1 neighbour sums) and report their total time. */
nau_status nau_profile_enable(nau_ctx* ctx, int on);
double nau_profile_ms(nau_ctx* ctx, int kernel_class, long* launches);
long nau_launch_count(nau_ctx* ctx);

/* Which kernels the last nau_wcsph_step ran (tests pin the benchmarked path):
 * bit 4 FAST mode, bits 2-3 the neighbour source (0 cell sweep, 1 per-particle
 * lists, 2 paired lists), bit 0 an image-carrying instantiation (some axis periodic
 * or symmetric). -1 before the first step. */
enum { NAU_PATH_IMAGES = 1, NAU_PATH_FAST = 16 };
int nau_wcsph_path(nau_ctx* ctx);

/* Instrumentation: shape of the cached neighbour lists (synchronises). out[0] =
 * list-walking threads (one per particle, or per particle pair with paired lists),
 * out[1] = entries they walk in total, out[2] = entries a warp-synchronous walk costs
 * (32 x the longest list of each warp, summed): out[1] / out[2] is the consumers'
 * lane efficiency. NAU_ERR_ARG when no list is cached. */
nau_status nau_list_stats(nau_ctx* ctx, double out[3]);

/* Microbenchmark: measured fp64 FMA throughput (TFLOP/s) of this GPU. */
double nau_fp64_peak_tflops(int device);

#ifdef __cplusplus
}
#endif
#endif
