// extern "C" entry points of libkfb200.so and the native fold-loop runtime:
// per-iteration kernel sequence, CUDA-graph capture/replay, error plumbing.
// See include/kfb200.h for the contract of each entry point.
#include <algorithm>
#include <cstring>
#include <mutex>
#include <string>
#include <unordered_map>
#include <vector>

#include "kf_common.cuh"

// launchers defined in the kernel translation units
int kf_fk_launch(const kf_chain_t *c, kf_batch_t *w, const kf_status_t *status, cudaStream_t s, int full_t);
int kf_bin_launch(const kf_field_t *f, kf_batch_t *w, int n, cudaStream_t s);
int kf_pairs_launch(const kf_field_t *f, kf_batch_t *w, int n, cudaStream_t s, int plane_b = 0);
int kf_clash_report_launch(const kf_field_t *f, kf_batch_t *w, int n, cudaStream_t s);
int kf_solvation_launch(const kf_field_t *f, kf_batch_t *w, int n, int n_solv, const int32_t *solv_atoms,
                        cudaStream_t s);
int kf_sasa_api_launch(const double *pos, int n, const double *r_off, const double *r_off2,
                       const double *samples, int N, const int64_t *nb_off, const int64_t *nb, double pad,
                       uint8_t *counts, int32_t *critical, int64_t *covered, const double *gamma,
                       double four_pi, double *f_exp, double *a_exp, double *cav, int nb_cap, int *overflow,
                       cudaStream_t s);
int kf_fixed_to_f64_launch(const long long *acc, int64_t m, double quantum, double *out, cudaStream_t s);
int kf_solv_forces_api_launch(const double *pos, int n, const double *r_off, const double *r_off2,
                              const int64_t *w_int, const double *samples, int N, const int64_t *nb_off,
                              const int64_t *nb, const uint8_t *counts, const int32_t *critical, double dr,
                              double pad, long long *acc, int nb_cap, int *overflow, cudaStream_t s);
int kf_wrench_launch(const kf_chain_t *c, int B, const double *pos, const double *forces, double *wrench,
                     const kf_status_t *status, cudaStream_t s);
int kf_torque_launch(const kf_chain_t *c, const kf_field_t *f, kf_batch_t *w, const double *link_T,
                     const double *wrench, double *side_tot, double *bb_suffix, double *tau,
                     const kf_step_t *step, int mode, cudaStream_t s, int fuse_wrench = 0);
int kf_kcm_step_launch(const double *tau, const double *theta, const uint8_t *frozen, int D, double kappa,
                       double *theta_out, double *deltas, cudaStream_t s);
int kf_fused_iteration(const kf_chain_t *c, const kf_field_t *f, kf_batch_t *w, const kf_step_t *st, cudaStream_t s,
                       int plane_b);
int kf_cluster_path(const kf_field_t *f, const kf_batch_t *w, int n);

namespace {
thread_local std::string g_last_error;
std::mutex g_graph_mu;
// instantiated fold graphs keyed on the launch's struct bytes (buffer pointers
// included), least recently used evicted past KF_GRAPH_CAP entries
struct GraphEntry { cudaGraphExec_t exec; unsigned long long used; };
std::unordered_map<std::string, GraphEntry> g_graphs;
unsigned long long g_graph_clock = 0;
constexpr size_t KF_GRAPH_CAP = 48;

std::string graph_key(const kf_chain_t *c, const kf_field_t *f, const kf_batch_t *w, const kf_step_t *st,
                      int n_iters, cudaStream_t s) {
    std::string k;
    k.append(reinterpret_cast<const char *>(c), sizeof(*c));
    k.append(reinterpret_cast<const char *>(f), sizeof(*f));
    k.append(reinterpret_cast<const char *>(w), sizeof(*w));
    k.append(reinterpret_cast<const char *>(st), sizeof(*st));
    k.append(reinterpret_cast<const char *>(&n_iters), sizeof(n_iters));
    (void)s;
    return k;
}

// One KCM iteration body (kcm.py:313-350): FK -> bin -> pairs -> [solvation] ->
// wrenches -> torques + record + stop tests + step.
int enqueue_iteration(const kf_chain_t *c, const kf_field_t *f, kf_batch_t *w, const kf_step_t *st,
                      cudaStream_t s, int plane_b = 0) {
    const int n = c->n_atoms;
    // vacuum ensembles on the cluster path: the whole iteration in one kernel
    const int fused = kf_fused_iteration(c, f, w, st, s, plane_b);
    if (fused == 2)   // FK + pairs fused: the torque step follows
        return kf_torque_launch(c, f, w, w->link_T, w->wrench, w->side_tot, w->bb_suffix, w->tau, st, 1, s, 1);
    if (fused >= 0) return fused;
    if (kf_fk_launch(c, w, w->status, s, 0)) return 1;   // the loop needs P and U only
    if (kf_bin_launch(f, w, n, s)) return 1;
    if (kf_pairs_launch(f, w, n, s, plane_b)) return 1;
    if (f->solvation && kf_solvation_launch(f, w, n, f->n_solv, f->solv_atoms, s)) return 1;
    // wrenches (fused into the torque CTA when they fit in shared memory) + torques + step
    if (kf_torque_launch(c, f, w, w->link_T, w->wrench, w->side_tot, w->bb_suffix, w->tau, st, 1, s, 1)) return 1;
    return 0;
}
}  // namespace

// Trajectories [b0, b0 + Bv) of batch w as a batch of their own: every per-trajectory
// array offset by b0 rows (row sizes as device.py's Batch allocates them).  Used
// for the vacuum cluster path only, whose kernels touch per-trajectory rows, the
// pair_fj planes (strided by the full batch: plane_b) and nothing batch-global.
static kf_batch_t batch_view(const kf_batch_t &w, const kf_chain_t *c, int b0, int Bv) {
    kf_batch_t v = w;
    v.B = Bv;
    const size_t n = (size_t)c->n_atoms, D = std::max(c->n_dof, 1), L = c->n_links, R = std::max(c->n_res, 1);
    const size_t nbb = std::max(c->n_bb, 1), H = (size_t)w.n_buckets;
    const size_t fk_rows = std::max(1, (c->n_bb + 255) / 256), recs = std::max(w.max_records, 1);
    const size_t b = (size_t)b0;
    auto off = [b](auto *p, size_t row) { return p ? p + b * row : p; };
    v.theta = off(w.theta, D); v.frozen = off(w.frozen, D); v.link_T = off(w.link_T, L * 16);
    v.fk_scratch = off(w.fk_scratch, fk_rows * 12); v.pos = off(w.pos, 3 * n); v.forces = off(w.forces, 3 * n);
    v.cell_key = off(w.cell_key, H); v.cell_cnt = off(w.cell_cnt, H); v.cell_start = off(w.cell_start, H);
    v.occ = off(w.occ, H); v.occ_count = off(w.occ_count, 1); v.occ_offset = off(w.occ_offset, 1);
    v.chunk_pre = off(w.chunk_pre, H); v.item_cell = off(w.item_cell, H); v.chunk_count = off(w.chunk_count, 1);
    v.chunk_offset = off(w.chunk_offset, 1); v.atom_slot = off(w.atom_slot, n); v.atom_rank = off(w.atom_rank, n);
    v.sorted_atom = off(w.sorted_atom, n); v.s_hi = off(w.s_hi, 4 * n); v.s_lo = off(w.s_lo, 4 * n);
    v.s_pos = off(w.s_pos, 4 * n); v.s_par = off(w.s_par, 4 * n); v.s_aux = off(w.s_aux, 4 * n);
    v.s_tree = off(w.s_tree, 4 * n); v.cell_box = off(w.cell_box, 8 * H);
    v.e_atom = off(w.e_atom, 2 * n); v.pair_count = off(w.pair_count, n); v.solv_acc = off(w.solv_acc, 3 * n);
    v.pair_fj = off(w.pair_fj, 3 * n); v.cav_atom = off(w.cav_atom, n); v.f_exp = off(w.f_exp, n);
    v.a_exp = off(w.a_exp, n); v.wrench = off(w.wrench, L * 6); v.side_tot = off(w.side_tot, R * 6);
    v.bb_suffix = off(w.bb_suffix, nbb * 6); v.tau = off(w.tau, D); v.energy = off(w.energy, 3);
    v.status = off(w.status, 1); v.rec_energy = off(w.rec_energy, recs * 4);
    v.rec_theta = off(w.rec_theta, (size_t)w.max_records * D);
    return v;
}

// Vacuum ensembles on the cluster path run as independent sub-batches (>= 64
// trajectories, up to 4) on their own
// streams inside the graph (graph branches): one sub-batch's latency-bound FK /
// torque kernels overlap another's issue-bound pair kernel.  KFB200_BRANCHES sets
// the count (1: off).
constexpr int KF_MAX_BRANCHES = 4;
static int graph_branches(const kf_chain_t *c, const kf_field_t *f, const kf_batch_t *w) {
    static int env = -1, min_sub = 64;   // measured: B = 256 as 4 x 64 0.223 vs 0.259 ms, B = 512 as 4 x 128 0.362 vs 0.375
    if (env < 0) {
        const char *e = getenv("KFB200_BRANCHES");
        env = std::min(KF_MAX_BRANCHES, e ? atoi(e) : 4);   // measured (C5): 4 0.696, 2 0.711, 1 0.771 ms
        const char *m = getenv("KFB200_BRANCH_MIN");           // smallest sub-batch
        if (m) min_sub = std::max(1, atoi(m));
    }
    const int nbr = std::min(env, w->B / min_sub);
    if (nbr < 2 || f->solvation) return 1;
    kf_batch_t part = *w;
    part.B = w->B / nbr;
    if (!kf_cluster_path(f, w, c->n_atoms) || !kf_cluster_path(f, &part, c->n_atoms)) return 1;
    return nbr;
}

static unsigned long long g_launches = 0;
void kf_count_launch() { ++g_launches; }
unsigned long long kf_launches_so_far() { return g_launches; }

void kf_set_error(const char *where, cudaError_t e) {
    g_last_error = std::string(where) + ": " + cudaGetErrorString(e);
}

extern "C" {

int kf_abi_version(void) { return KF_ABI_VERSION; }

size_t kf_struct_size(int which) {
    switch (which) {
        case 0: return sizeof(kf_chain_t);
        case 1: return sizeof(kf_field_t);
        case 2: return sizeof(kf_status_t);
        case 3: return sizeof(kf_batch_t);
        case 4: return sizeof(kf_step_t);
        default: return 0;
    }
}

const char *kf_last_error(void) { return g_last_error.c_str(); }

int kf_device_sm_count(void) {
    int dev = 0, sms = 0;
    if (cudaGetDevice(&dev) != cudaSuccess) return -1;
    if (cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev) != cudaSuccess) return -1;
    return sms;
}

int kf_fk(const kf_chain_t *c, kf_batch_t *w, void *stream) {
    return kf_fk_launch(c, w, w->status, (cudaStream_t)stream, 1);
}

int kf_nonbonded(const kf_field_t *f, kf_batch_t *w, void *stream) {
    cudaStream_t s = (cudaStream_t)stream;
    if (kf_bin_launch(f, w, f->n_atoms, s)) return 1;
    return kf_pairs_launch(f, w, f->n_atoms, s);
}

int kf_solvation(const kf_field_t *f, kf_batch_t *w, void *stream) {
    return kf_solvation_launch(f, w, f->n_atoms, f->n_solv, f->solv_atoms, (cudaStream_t)stream);
}

int kf_energy_reduce(const kf_field_t *f, kf_batch_t *w, int n, void *stream) {
    kf_chain_t c;
    std::memset(&c, 0, sizeof(c));
    c.n_atoms = n;
    return kf_torque_launch(&c, f, w, nullptr, nullptr, nullptr, nullptr, nullptr, nullptr, 2,
                            (cudaStream_t)stream);
}

int kf_torques_step(const kf_chain_t *c, const kf_field_t *f, kf_batch_t *w, const kf_step_t *step,
                    void *stream) {
    cudaStream_t s = (cudaStream_t)stream;
    if (!step && kf_wrench_launch(c, w->B, w->pos, w->forces, w->wrench, w->status, s)) return 1;
    return kf_torque_launch(c, f, w, w->link_T, w->wrench, w->side_tot, w->bb_suffix, w->tau, step,
                            step ? 1 : 0, s, step ? 1 : 0);
}

static int fold_graph(const kf_chain_t *c, const kf_field_t *f, kf_batch_t *w, const kf_step_t *step,
                      int n_iters, cudaStream_t s, bool launch);

int kf_fold_iterations(const kf_chain_t *c, const kf_field_t *f, kf_batch_t *w, const kf_step_t *step,
                       int n_iters, void *stream) {
    return fold_graph(c, f, w, step, n_iters, (cudaStream_t)stream, true);
}

int kf_fold_graph_prepare(const kf_chain_t *c, const kf_field_t *f, kf_batch_t *w, const kf_step_t *step,
                          int n_iters, void *stream) {
    return fold_graph(c, f, w, step, n_iters, (cudaStream_t)stream, false);
}

static int fold_graph(const kf_chain_t *c, const kf_field_t *f, kf_batch_t *w, const kf_step_t *step,
                      int n_iters, cudaStream_t s, bool launch) {
    if (n_iters <= 0) return 0;
    const std::string key = graph_key(c, f, w, step, n_iters, s);
    cudaGraphExec_t exec = nullptr;
    {
        std::lock_guard<std::mutex> lk(g_graph_mu);
        auto it = g_graphs.find(key);
        if (it != g_graphs.end()) {
            exec = it->second.exec;
            it->second.used = ++g_graph_clock;
        }
    }
    if (!exec) {
        cudaGraph_t graph = nullptr;
        KF_CUDA(cudaStreamBeginCapture(s, cudaStreamCaptureModeThreadLocal), "begin capture");
        int rc = 0;
        const int nbr = graph_branches(c, f, w);
        if (nbr > 1) {
            // fork capture streams, one contiguous sub-batch per stream, join
            static cudaStream_t sx[KF_MAX_BRANCHES] = {};
            static cudaEvent_t fork = nullptr, join[KF_MAX_BRANCHES] = {};
            if (!fork) {
                cudaEventCreateWithFlags(&fork, cudaEventDisableTiming);
                for (int r = 1; r < KF_MAX_BRANCHES; ++r) {
                    cudaStreamCreateWithFlags(&sx[r], cudaStreamNonBlocking);
                    cudaEventCreateWithFlags(&join[r], cudaEventDisableTiming);
                }
            }
            sx[0] = s;
            kf_batch_t part[KF_MAX_BRANCHES];
            for (int r = 0; r < nbr; ++r) {
                const int b0 = (int)((long long)w->B * r / nbr), b1 = (int)((long long)w->B * (r + 1) / nbr);
                part[r] = batch_view(*w, c, b0, b1 - b0);
            }
            cudaEventRecord(fork, s);
            for (int r = 1; r < nbr; ++r) cudaStreamWaitEvent(sx[r], fork, 0);
            for (int k = 0; k < n_iters && !rc; ++k)
                for (int r = 0; r < nbr && !rc; ++r) rc = enqueue_iteration(c, f, &part[r], step, sx[r], w->B);
            for (int r = 1; r < nbr; ++r) {
                cudaEventRecord(join[r], sx[r]);
                cudaStreamWaitEvent(s, join[r], 0);
            }
        } else {
            for (int k = 0; k < n_iters && !rc; ++k) rc = enqueue_iteration(c, f, w, step, s);
        }
        cudaError_t e = cudaStreamEndCapture(s, &graph);
        if (rc) { if (graph) cudaGraphDestroy(graph); return 1; }
        KF_CUDA(e, "end capture");
        e = cudaGraphInstantiate(&exec, graph, 0);
        cudaGraphDestroy(graph);
        KF_CUDA(e, "graph instantiate");
        std::lock_guard<std::mutex> lk(g_graph_mu);
        if (g_graphs.size() >= KF_GRAPH_CAP) {
            auto old = g_graphs.begin();
            for (auto it = g_graphs.begin(); it != g_graphs.end(); ++it)
                if (it->second.used < old->second.used) old = it;
            cudaStreamSynchronize(s);   // the evicted graph may still be in flight on this stream
            cudaGraphExecDestroy(old->second.exec);
            g_graphs.erase(old);
        }
        g_graphs[key] = GraphEntry{exec, ++g_graph_clock};
    }
    if (launch) KF_CUDA(cudaGraphLaunch(exec, s), "graph launch");
    return 0;
}

void kf_graph_cache_clear(void) {
    std::lock_guard<std::mutex> lk(g_graph_mu);
    for (auto &kv : g_graphs) cudaGraphExecDestroy(kv.second.exec);
    g_graphs.clear();
}

int kf_fold_iterations_eager(const kf_chain_t *c, const kf_field_t *f, kf_batch_t *w, const kf_step_t *step,
                             int n_iters, void *stream) {
    for (int k = 0; k < n_iters; ++k)
        if (enqueue_iteration(c, f, w, step, (cudaStream_t)stream)) return 1;
    return 0;
}

unsigned long long kf_launch_counter(void) { return kf_launches_so_far(); }

int kf_clash_report(const kf_field_t *f, kf_batch_t *w, void *stream) {
    return kf_clash_report_launch(f, w, f->n_atoms, (cudaStream_t)stream);
}

int kf_sasa_pass(const double *pos, int n, const double *r_off, const double *r_off2, const double *samples,
                 int n_samples, const int64_t *nb_off, const int64_t *nb, double pad, int nb_cap,
                 uint8_t *counts, int32_t *critical, int64_t *covered, const double *gamma, double four_pi,
                 double *f_exp, double *a_exp, double *cav, int *overflow, void *stream) {
    return kf_sasa_api_launch(pos, n, r_off, r_off2, samples, n_samples, nb_off, nb, pad, counts, critical, covered,
                              gamma, four_pi, f_exp, a_exp, cav, nb_cap, overflow, (cudaStream_t)stream);
}

int kf_fixed_to_f64(const long long *acc, int64_t m, double quantum, double *out, void *stream) {
    return kf_fixed_to_f64_launch(acc, m, quantum, out, (cudaStream_t)stream);
}

int kf_bin(const kf_field_t *f, kf_batch_t *w, void *stream) {
    return kf_bin_launch(f, w, f->n_atoms, (cudaStream_t)stream);
}

int kf_pairs(const kf_field_t *f, kf_batch_t *w, void *stream) {
    return kf_pairs_launch(f, w, f->n_atoms, (cudaStream_t)stream);
}

int kf_solvation_forces(const double *pos, int n, const double *r_off, const double *r_off2, const int64_t *w_int,
                         const double *samples, int n_samples, const int64_t *nb_off, const int64_t *nb,
                         const uint8_t *counts, const int32_t *critical, double delta_r, double pad, int nb_cap,
                         long long *acc, int *overflow, void *stream) {
    return kf_solv_forces_api_launch(pos, n, r_off, r_off2, w_int, samples, n_samples, nb_off, nb, counts, critical,
                                     delta_r, pad, acc, nb_cap, overflow, (cudaStream_t)stream);
}

int kf_link_wrenches(const kf_chain_t *c, const double *pos, const double *forces, double *wrench, void *stream) {
    return kf_wrench_launch(c, 1, pos, forces, wrench, nullptr, (cudaStream_t)stream);
}

int kf_joint_torques(const kf_chain_t *c, const double *link_T, const double *wrench, double *side_tot,
                     double *bb_suffix, double *tau, void *stream) {
    kf_batch_t w;
    std::memset(&w, 0, sizeof(w));
    w.B = 1;
    return kf_torque_launch(c, nullptr, &w, link_T, wrench, side_tot, bb_suffix, tau, nullptr, 0,
                            (cudaStream_t)stream);
}

int kf_kcm_step(const double *tau, const double *theta, const uint8_t *frozen, int n_dof, double kappa,
                double *theta_out, double *deltas, void *stream) {
    return kf_kcm_step_launch(tau, theta, frozen, n_dof, kappa, theta_out, deltas, (cudaStream_t)stream);
}

}  // extern "C"
