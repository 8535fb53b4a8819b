/*
 * kfb200 — C ABI of the B200-native KCM iteration (Protofold II, arXiv 1712.05012).
 *
 * One shared library, libkfb200.so, built for sm_100a.  Every entry point is
 * extern "C", takes plain pointers and sizes, returns 0 on success (nonzero =
 * CUDA error; text via kf_last_error()), and enqueues on the caller's stream
 * (a cudaStream_t passed as void*).  Device memory is owned by the caller
 * (the Python host allocates it through PyTorch); the library never allocates
 * persistent memory.  Domain errors (steric clash, non-finite coordinates)
 * are written to a device status block (kf_status_t) that the host maps to
 * the reference's exception classes.
 *
 * Each entry point replaces one function of the reference's Python API
 * (/root/reference/pkg/src/kinefold/...); the citation is on each one.
 * Batched entry points take B trajectories of one chain (B = 1 for API calls).
 */
#ifndef KFB200_H
#define KFB200_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define KF_ABI_VERSION 14

/* ---- static chain tables (uploaded once per chain) ------------------------
 * Links are in the reference's topological order (parent < index, ground = 0),
 * chain.py:104-116, :466-486, :528-539.  The backbone (phi/psi) links form a
 * path; side (chi) links hang off it with depth <= 4.                        */
typedef struct {
    int32_t n_atoms, n_links, n_dof, n_res;
    int32_t n_bb;            /* backbone path length (2m)                         */
    int32_t n_side;          /* side (chi) links                                  */
    int32_t side_depth;      /* max depth of a side link below the backbone      */
    int32_t _pad0;
    const int32_t *link_parent;     /* [L]                                        */
    const int32_t *link_dof;        /* [L], -1 for ground                         */
    const double  *link_axis0;      /* [L][3] reference axis (0 for ground)        */
    const double  *link_body0;      /* [L][3]                                      */
    const int32_t *bb_order;        /* [n_bb] backbone links, anchor side first    */
    const int32_t *side_order;      /* [n_side] side links sorted by depth         */
    const int32_t *side_depth_off;  /* [side_depth+1] offsets into side_order      */
    const int32_t *atom_link;       /* [n]                                         */
    const double  *atom_zrel;       /* [n][3] zp_pos - point0[link]                */
    const int32_t *link_atom_off;   /* [L+1] CSR link -> atoms (ascending)         */
    const int32_t *link_atoms;      /* [n]                                         */
    const int32_t *chi_res_off;     /* [n_res+1] chi links per residue             */
    const int32_t *chi_links;       /* chi links grouped by residue, chi order     */
    const int32_t *bb_by_dof;       /* [n_bb] backbone links by ascending dof      */
    const int32_t *bb_side_res;     /* [n_bb] residue whose side total joins at this
                                       backbone link (its phi link), else -1          */
} kf_chain_t;

/* ---- static field tables (uploaded once per Field) ------------------------ */
typedef struct {
    int32_t n_atoms;
    int32_t uniform_weights;        /* 1: UniformWeights(value), 0: TreeWeights    */
    int32_t dielectric_const;       /* 1: constant kappa, 0: kappa = d             */
    int32_t solvation;              /* FieldConfig.solvation                       */
    const float  *q32, *R32, *seps32;       /* fp32 copies for the pair math       */
    const double *q, *R, *eps;              /* fp64 (clash-range path)             */
    const int32_t *tparent, *tgp, *tggp, *tres;  /* bond tree (topology.py:73-91)  */
    const uint8_t *tchain;                  /* chain (non-hetero) mask             */
    const int32_t *class_map;   /* [n][4]: 2-bit (4 - class) codes for partners
                                   j = i - 32 .. i + 31 (static topology, host-built) */
    const uint8_t *class_slow;  /* [n]: atom has a tree partner outside that window */
    double w_elec[4], w_vdw[4];     /* weight by class 1..4 (index class-1)        */
    double uniform_value;
    double kappa;
    double cut_pair2;               /* max(elec, vdw)^2, spatial.py:240            */
    double thr_elec2, thr_vdw2;     /* largest d2 with sqrt(d2) <= cut (kcm.py:115,120) */
    /* hot-path spatial hash */
    double cell;                    /* cell edge, A                                */
    int32_t hash_bits;              /* buckets per trajectory = 1 << hash_bits     */
    int32_t n_stencil;
    const int32_t *stencil;         /* [n_stencil][3] cell offsets                 */
    /* solvation (solvation.py:135-255) */
    int32_t n_samples;
    int32_t _pad1;
    const double  *samples;         /* [N][3] unit sphere                          */
    const double  *r_off, *r_off2;  /* [n]                                         */
    const double  *gamma;           /* [n]                                         */
    const int64_t *w_int;           /* [n] fixed-point event magnitudes            */
    double quantum, delta_r, four_pi;
    double reach_pad;               /* delta_r + slack for the reach prefilter     */
    const int32_t *solv_atoms;      /* atoms with gamma != 0 (the only ones whose
                                       exposure enters g_cav or the forces)        */
    int32_t n_solv;
    int32_t precision;              /* pair math: 0 = fp32 (fp64 sums), 1 = fp64   */
    /* hot-path sample groups: the N directions reordered into G compact groups
       of <= 32 (host-built), padded to 32 per group                           */
    const double *samples_grp;      /* [G][32][3]                                  */
    const float *grp_cone;          /* [G][8]: axis xyz, cos alpha, sin alpha, count, 0, 0 */
    int32_t n_groups;
    int32_t flat;                   /* 1: FieldConfig(use_hash=False): one all-atom cell
                                       (quadratic candidates, kcm.py:153-162), n_stencil 1 */
    /* per-atom records gathered by binning (one 16-byte load each)            */
    const float *atom_par;          /* [n][4]: q, R, sqrt(eps), 0 (fp32)           */
    const int32_t *atom_aux;        /* [n][4]: atom, residue, chain flag, class_slow (0 if uniform) */
    double r_off_max;               /* max R_off over atoms (solvation cell pruning) */
    /* cluster-pair kernel (kf_cluster.cu): for quad Q (atoms 4Q..4Q+3) and the
       octets O = Q/2 + k, k = 0..4 (atoms 8O..8O+7), the 2-bit (4 - class) codes
       of the 32 pairs (i = 4Q + l%4, j = 8O + l/4) at bits 2l; host-built from the
       bond tree (topology.py:153-178).  NULL for UniformWeights.               */
    const unsigned long long *class_codes;   /* [ceil(n/4)][5] */
    /* the same codes per (unit U = octet U = quads 2U, 2U+1; lane l): bits 2k..2k+1
       quad 2U's code for window octet U + k, bits 10 + 2k.. quad 2U + 1's, bits
       20-24 / 25-29 which of the 5 window octets hold a class < 4 pair for either
       quad, bit 30 the unit has a class_slow atom.  NULL for UniformWeights.   */
    const uint32_t *unit_codes;     /* [ceil(n/8)][32] */
} kf_field_t;

/* ---- per-trajectory status block ----------------------------------------- */
typedef struct {
    int32_t iter;          /* iterations recorded so far                          */
    int32_t done;          /* stop flag (loop body becomes a no-op)               */
    int32_t reason;        /* KF_REASON_*                                          */
    int32_t error;         /* KF_ERR_*                                             */
    int32_t err_iter;      /* iteration at which the error occurred                */
    int32_t clash_i, clash_j;
    int32_t overflow;      /* neighbour-list capacity exceeded (count)             */
    unsigned long long dmin_bits;  /* bits of the smallest clashing distance      */
    unsigned long long clash_key;  /* (i << 32) | j of the reported clash pair     */
    double tau0;
    long long n_pairs;     /* pairs with d <= elec cutoff, last evaluation        */
    long long n_pairs_vdw; /* pairs with d <= vdW cutoff, last evaluation         */
} kf_status_t;

enum { KF_REASON_NONE = 0, KF_REASON_MAX_ITERS = 1, KF_REASON_TORQUE_FREE = 2,
       KF_REASON_TORQUE_TOL = 3, KF_REASON_TORQUE_TOL_REL = 4, KF_REASON_PLATEAU = 5 };
enum { KF_ERR_NONE = 0, KF_ERR_CLASH = 1, KF_ERR_NONFINITE = 2, KF_ERR_CAPACITY = 3,
       KF_ERR_EXTENT = 4 /* flat layout: an atom beyond 2048 A of the centroid cell */ };

/* ---- batch workspace (B trajectories, caller-allocated) ------------------ */
typedef struct {
    int32_t B;
    int32_t n_buckets;              /* 1 << hash_bits                              */
    int32_t nb_cap;                 /* solvation neighbour capacity per atom       */
    int32_t record_theta;           /* store theta per iteration                   */
    int32_t max_records;            /* record ring capacity (iterations)           */
    int32_t pair_chunk;             /* atoms per pair-kernel work item: 4/8/16/32, 0 = auto */
    int32_t api_eval;               /* 1: a single-conformation API evaluation (Field.evaluate):
                                       below 32 trajectories it keeps the binned dense lanes,
                                       whose separate hash phase the API reports; 0: fold loop */
    int32_t _pad_b;
    double  *theta;                 /* [B][D]                                      */
    const uint8_t *frozen;          /* [B][D]                                      */
    double  *link_T;                /* [B][L][16]: rotation (row-major 9), joint point (3), axis (3), pad */
    double  *fk_scratch;            /* [B][ceil(n_bb/2048)][12] segment totals of the
                                       multi-CTA backbone scan (long chains)           */
    double  *pos;                   /* [B][n][3]                                   */
    double  *forces;                /* [B][n][3]                                   */
    /* spatial hash: per trajectory an open-addressing table of H = n_buckets
       slots, one slot per occupied cell (key = packed integer cell)          */
    unsigned long long *cell_key;   /* [B][H], ~0 = empty                          */
    int32_t *cell_cnt;              /* [B][H] atoms in the slot's cell             */
    int32_t *cell_start;            /* [B][H] first sorted index of the cell       */
    int32_t *occ;                   /* [B][H] occupied slots (first occ_count[b])  */
    int32_t *occ_count;             /* [B]                                         */
    int32_t *occ_offset;            /* [B+1] prefix of occ_count (cells)           */
    int32_t *chunk_pre;             /* [B][H] per occupied cell (list order): prefix
                                       of its 32-atom i-chunks ceil(cnt/32)        */
    int32_t *item_cell;             /* [B][H] per local work item: its cell's list
                                       position (the pair kernels' item -> cell map) */
    int32_t *chunk_count;           /* [B] i-chunks of the trajectory              */
    int32_t *chunk_offset;          /* [B+1] prefix of chunk_count (pair work items) */
    int32_t *atom_slot;             /* [B][n] slot of the atom's cell              */
    int32_t *atom_rank;             /* [B][n] arrival rank inside the cell         */
    int32_t *sorted_atom;           /* [B][n] atoms grouped by cell, ascending     */
    float   *s_hi;                  /* [B][n][4] offset from the cell centre, fp32 */
    float   *s_lo;                  /* [B][n][4] fp32 remainder (hi + lo = fp64)   */
    double  *s_pos;                 /* [B][n][4] fp64 position, R_off (solvation)  */
    float   *s_par;                 /* [B][n][4] q, R, sqrt(eps), 0                */
    int32_t *s_aux;                 /* [B][n][4] atom, residue, chain flag, 0      */
    int32_t *s_tree;                /* [B][n][4] parent, grandparent, great-grand  */
    float   *cell_box;              /* [B][H][8] member bounding box (lo4, hi4)    */
    int32_t *work;                  /* [1] dynamic work counter (zeroed per launch)*/
    /* nonbonded */
    double  *e_atom;                /* [B][n][2] elec / vdW energy (full list: twice
                                       the pair sum); per-cell totals at the cell's
                                       lowest atom, 0 elsewhere                      */
    long long *pair_count;          /* [B][n] partner counts (elec | vdW << 32),
                                       per-cell totals stored at the cell's lowest atom */
    /* solvation */
    long long *solv_acc;            /* [B][n][3] int64 fixed point                 */
    int32_t *solv_ovf;              /* [1 + 2 B n]: count, (b, atom) pairs deferred to
                                       the large-capacity solvation pass            */
    long long *pair_fj;             /* [3][B][n][3] half-list j-side forces and exact-path
                                       forces: fixed point (lo plane in 2^-28, hi plane
                                       in 2^12) + an fp64 plane for |f| >= 2^72; kept
                                       zero between launches; NULL: full-list kernel */
    double  *cav_atom;              /* [B][n] gamma_i * a_exp_i                    */
    double  *f_exp;                 /* [B][n] exposure ratio (NULL: not stored)    */
    double  *a_exp;                 /* [B][n] exposed area (NULL: not stored)      */
    /* torques */
    double  *wrench;                /* [B][L][6] force, moment about origin        */
    double  *side_tot;              /* [B][n_res][6] side-branch totals            */
    double  *bb_suffix;             /* [B][n_bb][6] backbone suffix scratch         */
    double  *tau;                   /* [B][D]                                      */
    double  *energy;                /* [B][3] g_elec, g_vdw, g_cav (last eval)     */
    kf_status_t *status;            /* [B]                                         */
    /* records (fold loop) */
    double  *rec_energy;            /* [B][max_records][4] elec, vdw, cav, tau_max */
    double  *rec_theta;             /* [B][max_records][D] (if record_theta)        */
} kf_batch_t;

typedef struct {
    double kappa, torque_tol, torque_tol_rel, energy_tol;
    int32_t max_iters, energy_window;
} kf_step_t;

/* ---- housekeeping --------------------------------------------------------- */
int         kf_abi_version(void);
size_t      kf_struct_size(int which);     /* 0 chain, 1 field, 2 status, 3 batch, 4 step */
const char *kf_last_error(void);
int         kf_device_sm_count(void);

/* ---- hot path, batched (the fold loop body, kcm.py:312-350) --------------- */

/* Forward kinematics: theta -> link transforms + atom positions.
 * Replaces chain.kinematic_state / forward_kinematics (chain.py:240-276). */
int kf_fk(const kf_chain_t *c, kf_batch_t *w, void *stream);

/* The two halves of kf_nonbonded, for per-phase timing ("hash", "force"). */
int kf_bin(const kf_field_t *f, kf_batch_t *w, void *stream);
int kf_pairs(const kf_field_t *f, kf_batch_t *w, void *stream);

/* Spatial hash + elec/vdW pair kernel + clash guard, forces and per-atom
 * energies.  Replaces Field._neighbor_table + extract_pairs + weights_for +
 * elec/vdw_pair_quantities + accumulate (kcm.py:94-127, spatial.py:83-241,
 * forcefield.py:81-113,162-172, topology.py:153-195). */
int kf_nonbonded(const kf_field_t *f, kf_batch_t *w, void *stream);

/* Fused cavity-solvation exposure pass + fixed-point forces on the hash grid.
 * Replaces filtered_lists + sasa_pass + solvation_forces (spatial.py:244-259,
 * solvation.py:135-255) inside Field.evaluate (kcm.py:132-142). */
int kf_solvation(const kf_field_t *f, kf_batch_t *w, void *stream);

/* Energy reduction of the last kf_nonbonded/kf_solvation (Field.evaluate's
 * g_elec, g_vdw, g_cav, kcm.py:119-144); n = atoms per trajectory. */
int kf_energy_reduce(const kf_field_t *f, kf_batch_t *w, int n, void *stream);

/* Link wrenches + suffix-scan joint torques + energy reduction (+ record,
 * stop tests and compliance step when step != NULL).
 * Replaces link_wrenches, joint_torques, kcm_step/apply_deltas and the
 * per-iteration bookkeeping of fold (kcm.py:177-240, :264-274, :325-350). */
int kf_torques_step(const kf_chain_t *c, const kf_field_t *f, kf_batch_t *w,
                    const kf_step_t *step, void *stream);

/* K iterations of the full loop body, replayed from a CUDA graph captured on
 * first use (kcm.py:312-350).  Stops early on device when every trajectory
 * is done; the host polls status between chunks. */
int kf_fold_iterations(const kf_chain_t *c, const kf_field_t *f, kf_batch_t *w,
                       const kf_step_t *step, int n_iters, void *stream);
/* Capture and instantiate the graph kf_fold_iterations would replay for
 * n_iters, without launching it (keeps graph construction out of timings). */
int kf_fold_graph_prepare(const kf_chain_t *c, const kf_field_t *f, kf_batch_t *w,
                          const kf_step_t *step, int n_iters, void *stream);
/* Same loop body launched eagerly (no graph), for debugging and profiling. */
int kf_fold_iterations_eager(const kf_chain_t *c, const kf_field_t *f, kf_batch_t *w,
                             const kf_step_t *step, int n_iters, void *stream);
/* Drop cached graphs (call before freeing buffers they reference). */
void kf_graph_cache_clear(void);

/* Smallest-(i, j) clashing pair among pairs at the minimum distance, for the
 * StericClashError message (forcefield.py:84-88).  Run only on error. */
int kf_clash_report(const kf_field_t *f, kf_batch_t *w, void *stream);

/* The elec/vdW pair kernel kf_pairs (and the fold loop) selects for this field,
 * batch and atom count: 0 compacted list (fp64 pair math), 1 dense lanes with
 * full list, 2 dense lanes with half list, 3 cluster pairs (one CTA per
 * trajectory, no binning pass in vacuum). */
int kf_pair_kernel_kind(const kf_field_t *f, const kf_batch_t *w, int n);

/* Kernel launches this library has enqueued so far (host counter; a captured
 * CUDA graph replays the launches counted while it was captured). */
unsigned long long kf_launch_counter(void);
/* Issue-rate microbenchmark of this GPU: kind 0 = FP32 FFMA, 1 = FP64 DFMA.
 * Writes FLOP/s (FMA = 2 FLOP) measured with events on `stream` to *out. */
int kf_peak_flops(int kind, double *out, void *stream);

/* ---- reference-API entry points (B = 1, parity and drop-in calls) -------- */

/* build_grid (spatial.py:83-114): per-axis min [0:3], max [3:6] and the count
 * of non-finite coordinates [6] of positions [n][3]. */
int kf_bbox(const double *pos, int n, double *out /* [7] */, void *stream);
/* Cell index + linear key with the host-computed cell edge (bit-exact). */
int kf_grid_cells(const double *pos, int n, const double *r_min, double cell,
                  const int64_t *dims, int64_t *cell_index /* [n][3] */,
                  int64_t *lin /* [n] */, void *stream);
/* Stable counting sort of atoms by key in [0, n_keys): counts, exclusive
 * starts and order (ascending index within equal keys). */
int kf_counting_sort(const int64_t *key, int n, int64_t n_keys, int32_t *counts,
                     int64_t *starts /* [n_keys+1] */, int64_t *order,
                     int64_t *scratch /* [n_keys + 1024] */, void *stream);

/* Reference superset table (spatial.py:163-230): rows ascending, self excluded. */
int kf_neighbor_rows_count(const int64_t *cell_index, const int64_t *dims, int n,
                           const int64_t *cell_start, const int32_t *stencil, int n_stencil,
                           int64_t *row_len, void *stream);
int kf_neighbor_rows_fill(const int64_t *cell_index, const int64_t *dims, int n,
                          const int64_t *cell_start, const int64_t *order,
                          const int32_t *stencil, int n_stencil,
                          const int64_t *offsets, int64_t *neighbors, void *stream);
/* Sort each CSR row ascending in place. */
int kf_sort_rows(const int64_t *offsets, int n_rows, int64_t *values, void *stream);

/* filtered_pairs / filtered_lists (spatial.py:233-259): d2 in the reference's
 * einsum order (dx*dx + dz*dz) + dy*dy, kept where d2 <= d_cut^2. */
int kf_filter_table(const double *pos, const int64_t *offsets, const int64_t *neighbors,
                    int n, int64_t n_entries, double cut2, int upper_only, uint8_t *keep,
                    double *d2, void *stream);
/* Stable compaction of kept entries into (i, j, d = sqrt(d2)) in table order. */
int kf_compact_pairs(const int64_t *offsets, const int64_t *neighbors, int n, int64_t n_entries,
                     const uint8_t *keep, const double *d2, int64_t *dest /* [n_entries+1] */,
                     int64_t *scratch /* [n_entries + 1024] */, int64_t *oi, int64_t *oj,
                     double *od, void *stream);
/* Deterministic fp64 sum (fixed chunking and tree). */
int kf_sum_f64(const double *x, int64_t n, double *partials /* [1024] */, double *out,
               void *stream);
/* Exclusive scan, out[n] = total. scratch >= 1024. */
int kf_scan_exclusive_i64(const int64_t *in, int64_t n, int64_t *out, int64_t *scratch,
                          void *stream);

/* Pair classes for arrays (i, j) (topology.py:153-178). */
int kf_classify_pairs(const kf_field_t *f, const int64_t *i, const int64_t *j, int64_t n,
                      int64_t *cls, void *stream);

/* elec/vdW over an explicit pair list (forcefield.py:98-172): per-pair energy
 * and magnitude in fp64; forces (if non-NULL, n atoms) scattered in np.bincount
 * order, bit-identical to the reference and deterministic. kind: 0 elec, 1 vdW. */
int kf_pair_terms(const kf_field_t *f, const double *pos, int n, const int64_t *i,
                  const int64_t *j, const double *d, const double *w /* NULL: classify */,
                  int64_t n_pairs, int kind, double *e_pair, double *mag,
                  double *forces /* [n][3] or NULL */, void *stream);
/* accumulate_pair_forces (forcefield.py:116-117, :162-172): forces [n][3] +=
 * bincount(i, f) then -= bincount(j, f), in the reference's order (deterministic). */
int kf_scatter_pair_forces(const double *pos, int n, const int64_t *i, const int64_t *j,
                           const double *d, const double *mag, int64_t m, double *forces,
                           void *stream);
/* build_grid's occupied cells and their starts from dense per-key counts. */
int kf_grid_occupied(const int32_t *counts, const int64_t *starts, int64_t n_keys,
                     int64_t *scratch /* [n_keys + 1024] */, int64_t *dest /* [n_keys+1] */,
                     int64_t *occupied, int64_t *occ_starts, void *stream);
/* Per-row offsets of kept table entries: out[r] = dest[offsets[r]], r <= n. */
int kf_row_kept_offsets(const int64_t *offsets, int n, const int64_t *dest, int64_t *out,
                        void *stream);
/* np.argmin of x[0..m) (first index of the minimum). */
int kf_argmin_f64(const double *x, int64_t m, int64_t *out, void *stream);

/* sasa_pass (solvation.py:135-181) over explicit CSR neighbour lists.  Only
 * neighbours within R_off_i + R_off_j + pad can cover a sample; those are
 * staged (at most nb_cap per atom; a larger count is written to *overflow and
 * the call must be repeated with a larger cap).  Also writes f_exp, a_exp and
 * the per-atom g_cav terms gamma * a_exp (solvation.py:177-180). */
int kf_sasa_pass(const double *pos, int n, const double *r_off, const double *r_off2,
                 const double *samples, int n_samples, const int64_t *nb_off,
                 const int64_t *nb, double pad, int nb_cap, uint8_t *counts,
                 int32_t *critical, int64_t *covered, const double *gamma, double four_pi,
                 double *f_exp, double *a_exp, double *cav, int *overflow, void *stream);
/* solvation_forces (solvation.py:194-255) from given states; int64 result
 * accumulated into acc [n][3] (caller zeroes it). */
int kf_solvation_forces(const double *pos, int n, const double *r_off,
                        const double *r_off2, const int64_t *w_int, const double *samples,
                        int n_samples, const int64_t *nb_off, const int64_t *nb,
                        const uint8_t *counts, const int32_t *critical, double delta_r,
                        double pad, int nb_cap, long long *acc, int *overflow, void *stream);
/* acc * quantum -> fp64 (solvation.py:255). */
int kf_fixed_to_f64(const long long *acc, int64_t m, double quantum, double *out, void *stream);

/* link_wrenches (kcm.py:177-188) for one trajectory. */
int kf_link_wrenches(const kf_chain_t *c, const double *pos, const double *forces,
                     double *wrench /* [L][6] */, void *stream);
/* joint_torques (kcm.py:196-240): wrenches + link transforms -> tau[D]. */
int kf_joint_torques(const kf_chain_t *c, const double *link_T, const double *wrench,
                     double *side_tot /* [n_res][6] */, double *bb_suffix /* [n_bb][6] */,
                     double *tau, void *stream);
/* kcm_step + apply_deltas (kcm.py:264-274, chain.py:93-101). */
int kf_kcm_step(const double *tau, const double *theta, const uint8_t *frozen, int n_dof,
                double kappa, double *theta_out, double *deltas, void *stream);

#ifdef __cplusplus
}
#endif
#endif /* KFB200_H */
