// Internal launcher declarations (not part of the public C ABI).
#pragma once
#include <cstddef>
#include <cstdint>
#include <cuda_runtime.h>

namespace isoc {
struct FoldStack;

constexpr int kRowCap = 40;   // per-row leaf-stack capacity of the sigma passes

// exact_passes.cu
size_t sigma_rowstack_entries(int64_t rows);
cudaError_t launch_sigma_pass(const double* X, int64_t n, int d, int64_t lo, int64_t hi, int want_p,
                              double* row_vals, uint64_t* row_ids, int32_t* row_cnt, int32_t* flags,
                              int32_t* nn_j, double* nn_d, int8_t* nn_tie, double* pfold,
                              cudaStream_t st);
cudaError_t launch_sigma_straddle(const double* X, int64_t n, int d, int64_t b_lo, int64_t b_hi,
                                  double* sval, uint64_t* sid, int8_t* sown, cudaStream_t st);
cudaError_t launch_sigma_merge_rows(int64_t n, int64_t lo, int64_t hi, int G, const double* row_vals,
                                    const uint64_t* row_ids, const int32_t* row_cnt,
                                    const double* sval, const uint64_t* sid, const int8_t* sown,
                                    FoldStack* out, int32_t* flags, cudaStream_t st);
cudaError_t launch_stack_merge(const FoldStack* in, int64_t nin, int G, FoldStack* out,
                               int32_t* flags, cudaStream_t st);
cudaError_t launch_omega_pass(const double* X, int64_t n, int d, int64_t lo, int64_t hi,
                              double sigma, const int32_t* comp, double* omega, int32_t* nn_j,
                              double* nn_d, int8_t* nn_tie, cudaStream_t st);
cudaError_t launch_transpose_pad(const double* X, int64_t n, int d, int64_t np, int dpad, double* XT,
                                 cudaStream_t st);

// sigma_sym.cu
bool sigma_sym_applicable(int64_t n, int64_t lo, int64_t hi, int want_p);
int device_sm_count();   // SMs of the current device (cached per device)
// cudaFuncSetAttribute(MaxDynamicSharedMemorySize) only when `bytes` exceeds
// what was last set for this kernel on this device (the call costs tens of
// microseconds; small-tree kernels launch per bisection batch)
cudaError_t ensure_max_dyn_smem(const void* func, size_t bytes);
int passes_mode();       // ISOC_PASSES test hook: 0 auto, 1 "sym", 2 "rows"
cudaError_t launch_sigma_sym(const double* X, int64_t n, int d, double* row_vals, uint64_t* row_ids,
                             int32_t* row_cnt, int32_t* flags, int32_t* nn_j, double* nn_d,
                             int8_t* nn_tie, cudaStream_t st);
cudaError_t launch_sigma_sym_range(const double* X, int64_t n, int d, int64_t jlo, int64_t jhi, int partial,
                                   double* row_vals, uint64_t* row_ids, int32_t* row_cnt, int32_t* flags,
                                   int32_t* nn_j, double* nn_d, int8_t* nn_tie, double* nn_m2,
                                   cudaStream_t st);
cudaError_t launch_sigma_rank_merge(int64_t rows, int G, const double* pv, const uint64_t* pid_,
                                    const int32_t* pc, const double* pm1, const double* pm2, const int32_t* pj,
                                    double* row_vals, uint64_t* row_ids, int32_t* row_cnt, int32_t* flags,
                                    int32_t* nn_j, double* nn_d, int8_t* nn_tie, cudaStream_t st);
int sigma_sym_block();
// balanced ranges of column super-blocks (I <= J super-tiles) of size `block`
void sym_block_range(int64_t n, int rank, int world, int64_t* jlo, int64_t* jhi, int block);

// omega_sym.cu
cudaError_t launch_omega_sym(const double* X, int64_t n, int d, double sigma, const int32_t* comp,
                             double* omega, int32_t* nn_j, double* nn_d, int8_t* nn_tie,
                             cudaStream_t st);
// sharded symmetric omega: per-peer slot counts of rank `rank` (send[g] to
// owner g, recv[s] from sender s); the send / receive buffers are the
// concatenations of the messages in peer order
void omega_shard_counts(int64_t n, int G, int rank, int64_t* send, int64_t* recv);
cudaError_t launch_omega_sym_range(const double* X, int64_t n, int d, double sigma, const int32_t* comp,
                                   int rank, int G, double* PS, double* PSm, int32_t* PSj, cudaStream_t st);
cudaError_t launch_omega_rank_merge(int64_t n, int rank, int G, const double* PS, const double* PSm,
                                    const int32_t* PSj, double* omega, int32_t* nn_j, double* nn_d,
                                    int8_t* nn_tie, cudaStream_t st);

// boruvka.cu
cudaError_t launch_prep_fp32(const double* X, int64_t n, int d, int dp, int64_t npad, double* centre,
                             float* Y, float* ny, float* rad, uint32_t* rmax_bits, cudaStream_t st);
cudaError_t launch_boruvka_filter(const float* Y, const float* ny, const int32_t* comp, int64_t n,
                                  int64_t npad, int dp, int64_t lo, int64_t hi, float* a1, int32_t* j1,
                                  float* a2, cudaStream_t st);
cudaError_t launch_boruvka_select(const double* X, int64_t n, int d, const float* a1,
                                  const int32_t* j1, const float* a2, const float* rad,
                                  const uint32_t* rmax_bits, float cd, float cabs, const int32_t* comp,
                                  int64_t lo, int64_t hi, uint32_t* compB, double* cand_d,
                                  int32_t* cand_j, int8_t* cand_state, int8_t* cand_tie,
                                  int32_t* rescan_list, int32_t* rescan_count, cudaStream_t st);
cudaError_t launch_boruvka_exact_all(const double* X, int64_t n, int d, const int32_t* comp, int64_t lo,
                                     int64_t hi, double* cand_d, int32_t* cand_j, int8_t* cand_state,
                                     int8_t* cand_tie, int32_t* rescan_list, int32_t* rescan_count,
                                     cudaStream_t st);
cudaError_t launch_nn_candidates(const int32_t* nn_j, const double* nn_d, const int8_t* nn_tie,
                                 int64_t rows, double* cand_d, int32_t* cand_j, int8_t* cand_state,
                                 int8_t* cand_tie, cudaStream_t st);
cudaError_t launch_comp_exact_min(const double* cand_d, const int8_t* cand_state,
                                  const int32_t* comp, int64_t n, int64_t lo, int64_t hi,
                                  unsigned long long* compD, cudaStream_t st);
cudaError_t launch_comp_edge(const double* cand_d, const int32_t* cand_j, const int8_t* cand_state,
                             const int32_t* comp, int64_t n, int64_t lo, int64_t hi,
                             const unsigned long long* compD, unsigned long long* compE,
                             cudaStream_t st);
cudaError_t launch_comp_ties(const double* cand_d, const int32_t* cand_j, const int8_t* cand_state,
                             const int8_t* cand_tie, const int32_t* comp, int64_t lo, int64_t hi,
                             const unsigned long long* compD, const unsigned long long* compE,
                             int32_t* ties, cudaStream_t st);
cudaError_t launch_hook_contract(int32_t* comp, int64_t n, const unsigned long long* compD,
                                 const unsigned long long* compE, int32_t* succ, int32_t* succ2,
                                 int32_t* eu, int32_t* ev, double* ed, int32_t* ecount,
                                 int32_t* changed, int32_t* nroots, cudaStream_t st);

// filter_tc.cu
size_t tc_image_bytes(int64_t n, int d);
cudaError_t launch_tc_image(const float* YT, int64_t npad, int d, float scale, int64_t n, uint8_t* img,
                            cudaStream_t st);
// small trees: the whole sweep in one CTA's shared memory (decide_small_kernel)
bool decide_small_fits(int64_t n, int64_t levels, size_t* smem);
constexpr int DECIDE_SMALL_MAX_BATCH = 63;   // thresholds per batched small sweep (one warp each)
// candidate lists per row: FILTER_LIST_K best (a, j) + the bound of the rest
#define FILTER_LIST_K 4
// rows_map == nullptr: every row of [lo, hi); else the nmap rows listed
// (device count nmap_dev), whose A operands are gathered into imgA
// (tc_image_bytes(nmap rounded up to 256, d) bytes)
cudaError_t launch_filter_tc(const uint8_t* img, const float* ny, const int32_t* comp, int64_t n, int d,
                             int64_t lo, int64_t hi, float kscale, float* la, int32_t* lj, float* lb,
                             const int32_t* rows_map, const int32_t* nmap_dev, int64_t nmap, uint8_t* imgA,
                             cudaStream_t st);
int64_t filter_tc_blocks(int64_t lo, int64_t hi);
cudaError_t launch_list_select(const float* la, const int32_t* lj, const float* lb, const int32_t* comp,
                               int64_t lo, int64_t hi, float* a1, int32_t* j1, float* a2, float* lbo,
                               cudaStream_t st);
cudaError_t launch_list_refresh(const float* a1, const float* lbo, const float* rad, const int32_t* comp,
                                int64_t n, int64_t lo, int64_t hi, const uint32_t* rmax_bits, float cd,
                                float cabs, uint32_t* compB, int32_t* blk_flag, int64_t nblk, int32_t* nflag,
                                int32_t* rows_list, cudaStream_t st);
cudaError_t launch_absmax(const float* v, int64_t m, uint32_t* out, cudaStream_t st);

// tree.cu
cudaError_t launch_build_adjacency(const int32_t* eu, const int32_t* ev, const double* ed,
                                   int64_t n, int32_t* off, int32_t* adj, double* adjd,
                                   int32_t* work, cudaStream_t st);
cudaError_t launch_children_from_parent(const int64_t* parent, const int64_t* child_id, int64_t n,
                                        int64_t root, int32_t* off, int32_t* adj, int32_t* child_id_v,
                                        int32_t* flags, int32_t* nroots, int32_t* found_root,
                                        cudaStream_t st);
cudaError_t launch_bfs(int64_t n, int64_t root, int undirected, const int32_t* off,
                       const int32_t* adj, const double* adjd, int32_t* bfs, int32_t* pos_of,
                       int32_t* parent_v, int32_t* depth_v, int32_t* child_id_v, double* parent_d,
                       int32_t* pos_parent, int32_t* child_lo, int32_t* child_cnt,
                       int64_t* level_off, int32_t* scratch, int64_t* out_levels, cudaStream_t st);
cudaError_t launch_flows(const double* parent_d, const int32_t* parent_v, int64_t n, double sigma,
                         double* flow, cudaStream_t st);
cudaError_t launch_gather_pos(const int32_t* bfs, int64_t n, const double* flow_v,
                              const double* omega_v, const double* p_v, double* f_pos,
                              double* om_pos, double* p_pos, cudaStream_t st);
cudaError_t launch_pow2_sum(const double* v, int64_t m, double* out, double* tmp, cudaStream_t st);
cudaError_t launch_min_value(const double* v, int64_t m, double* out, unsigned long long* key, cudaStream_t st);
cudaError_t launch_extrema(const double* flow_v, int64_t root, const double* omega, const double* p,
                           int64_t n, double* out6, double* tmp, unsigned long long* key,
                           cudaStream_t st);

// decide.cu
cudaError_t launch_decide_batch(int64_t n, int64_t levels, const int64_t* level_off, int64_t max_width,
                                const double* f_pos, const double* om0, const double* p0,
                                const int32_t* child_lo, const int32_t* child_cnt, const double* thr,
                                int K, int64_t k, double* om, double* p, int8_t* code, int32_t* excl,
                                int32_t* scratch, int64_t* j_out, cudaStream_t st);
cudaError_t launch_decide(int64_t n, int64_t levels, const int64_t* level_off, int64_t max_width,
                          const double* f_pos, const double* om0, const double* p0,
                          const int32_t* child_lo, const int32_t* child_cnt, double thr, int64_t k,
                          double* om, double* p, int8_t* code, int32_t* excl, double* spars,
                          int32_t* scratch, int64_t* j_out, cudaStream_t st);
cudaError_t launch_labels(const int8_t* code, const int32_t* pos_parent, const int32_t* bfs,
                          int64_t n, int64_t levels, int8_t* cut_v, int64_t* eta, int64_t* labels,
                          int32_t* lab32, int32_t* work, cudaStream_t st);
size_t cost_work_bytes(int64_t n, int64_t k);
cudaError_t launch_cost(const int32_t* lab32, const int32_t* parent_v, const double* flow,
                        const double* omega, const double* p, int64_t n, int64_t k, void* work,
                        size_t work_bytes, double* sums, double* miso, cudaStream_t st);
}  // namespace isoc
