/*
 * normint_b200 -- C ABI of the B200 (sm_100a) kernels behind the drop-in
 * replacement of the reference's component-integration hot path
 * (normint.run_pipeline, /root/reference/pkg/src/normint/pipeline.py:105-248).
 *
 * The reference has no FFI: its seams are Python functions.  Each entry point
 * below replaces one of them (cited per function).  Conventions:
 *
 *  - Every pointer argument is a DEVICE pointer unless its name ends in _host.
 *  - The pixel grid is a batch of B maps of H x W pixels, row-major, map-major:
 *    pixel id = (m * H + v) * W + u.  A single map is B = 1.  Edges never
 *    cross map boundaries, so a batch is exactly B independent problems.
 *  - Forward neighbour offsets (graph.py:24-25): 4-connectivity
 *    k=0:(+1,0) k=1:(0,+1); 8-connectivity k=0:(+1,0) k=1:(-1,+1) k=2:(0,+1)
 *    k=3:(+1,+1).  The edge key of forward edge k at pixel a is a*KF + k
 *    (KF = 2 or 4), whose order equals the reference's lexicographic (a, b)
 *    edge order (graph.py:80-83).
 *  - Calls are asynchronous on `stream` unless stated otherwise and return an
 *    ni_status; ni_last_error() gives a thread-local message.
 *  - The library allocates no persistent memory: scratch space is a caller
 *    buffer sized by the matching *_workspace_size query.
 *  - Results are deterministic: no floating-point atomics anywhere.
 */
#ifndef NORMINT_B200_H
#define NORMINT_B200_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

typedef void* ni_stream_t; /* a cudaStream_t */

typedef enum {
  NI_OK = 0,
  NI_ERR_INVALID_ARG = 1,     /* ValueError in the reference */
  NI_ERR_EMPTY_MASK = 2,      /* normint.errors.EmptyMask (graph.py:65-66) */
  NI_ERR_NONUNIT_NORMAL = 3,  /* ValueError from NormalMap.create (geometry.py:134-141) */
  NI_ERR_NONFINITE = 4,       /* ValueError "valid normals must be finite" (geometry.py:131-132) */
  NI_ERR_WORKSPACE = 5,       /* workspace smaller than the query returned */
  NI_ERR_CUDA = 6,            /* CUDA runtime error */
  NI_ERR_UNSUPPORTED = 7
} ni_status;

const char* ni_last_error(void);
const char* ni_version(void);
/* Host-side count of kernels this library launched (all threads). */
long long ni_launch_count(void);
/* Diagnostics of the last ni_fill on the calling thread: device time of the
 * persistent CG kernel (CUDA events on `stream`), sum over components of
 * size * CG iterations, largest iteration count, cooperative grid size,
 * number of 32x32 tiles and of (tile, component) partial slots. */
int ni_fill_last_report(double* cg_ms, long long* px_iters, int* max_iters, int* grid,
                        int* ntiles, int* npartials);

/* Counters written by ni_normalize / ni_coefficients (device struct). */
typedef struct {
  long long valid_pixels;      /* vertices record (pipeline.py:137-142) */
  long long nonfinite;         /* valid pixels with a non-finite component */
  long long nonunit;           /* valid pixels with |‖n‖-1| > 1e-4 */
  unsigned long long max_dev;  /* bits of the largest |‖n‖-1| (non-negative double) */
  long long edges;             /* edges record (pipeline.py:137-142) */
  long long degenerate_edges;  /* edge_coefficients record (pipeline.py:153-159) */
} ni_stats;

/* K0 -- NormalMap.create (geometry.py:115-145).  normals: (B*H*W, 3) float32
 * (dtype 0) or float64 (dtype 1), interleaved; mask: one byte per pixel, or
 * NULL for all-valid.  Writes float64 SoA normals n_out[3][npix] renormalised
 * as n / sqrt((x0^2 + x1^2) + x2^2) (zero on invalid pixels) and valid_out.
 * SYNCHRONOUS: reads back the counters and returns NI_ERR_NONFINITE,
 * NI_ERR_NONUNIT_NORMAL or NI_ERR_EMPTY_MASK like the reference raises. */
int ni_normalize(const void* normals, int dtype, const uint8_t* mask, int B, int H, int W,
                 double* n_out, uint8_t* valid_out, ni_stats* stats, ni_stream_t stream);

/* K1 -- form_components (graph.py:141-165) + build_pixel_graph's edge count.
 * Keeps edge (a,b) iff both valid and ((na0*nb0 + na1*nb1) + na2*nb2) >= dot_cutoff,
 * which equals arccos(clip(dot)) < theta_c when dot_cutoff is the smallest
 * float64 with numpy.arccos(d) < theta_c (computed by the host).  theta_none
 * != 0 gives one component per valid pixel (graph.py:153-155).
 * labels_out: int32 per pixel, canonical (rank of the component's smallest
 * pixel id; -1 invalid).  count_out[0] = component count;
 * map_first_out[m] = first label of map m (B+1 entries, last = count). */
int ni_components_workspace_size(int B, int H, int W, size_t* bytes);
int ni_components(const double* n, const uint8_t* valid, int B, int H, int W, int connectivity,
                  double dot_cutoff, int theta_none, int32_t* labels_out, int32_t* count_out,
                  int32_t* map_first_out, ni_stats* stats, void* workspace, size_t workspace_bytes,
                  ni_stream_t stream);

/* K2 -- build_edge_coefficients (continuity.py:210-289).  model 0 = milano,
 * 1 = bini (4-connectivity only).  intrinsics: per map (fx, fy, cx, cy)
 * float64 [B*4].  Outputs, per pixel a and forward edge k:
 *   omega_a[k*npix + a] (float64), omega_b[k*npix + a] (bini only; may be NULL
 *   for milano where omega_b = -omega_a), gamma[a] (float64),
 *   map_counts (nullable, device int64 [2B]): per map, the edges and the
 *   degenerate edges (the build_graph / edge_coefficients records);
 *   eflags[a]: bit k = edge exists (both endpoints valid), bit 4+k = its
 *   coefficient is valid (continuity.py:243-245, 266). */
int ni_coefficients(const double* n, const uint8_t* valid, const double* intrinsics, int B, int H,
                    int W, int connectivity, int model, double* omega_a, double* omega_b,
                    double* gamma, uint8_t* eflags, ni_stats* stats, long long* map_counts,
                    ni_stream_t stream);

/* K3 -- fill_components (solver.py:195-239): per-component CG on the
 * weighted normal equations, all components in one batched solve.
 * Weights: w_a = w_b = NULL is the fill at z = 0 (W = gamma^2 / 2 on both
 * rows, continuity.py:302-308); otherwise w_a / w_b are the directed weights
 * of every forward pixel edge (planes w[k*npix + a], see ni_edge_weights):
 * the refill pass (solver.py:237-238) and the pixel-level baseline
 * (pipeline.py:261-285, one "component" per map).  The CG always starts at
 * x0 = 0 and the solution is returned (the right-hand side is the full
 * A^T W omega, not an increment).
 * SYNCHRONOUS (polls convergence).  Writes z_out (float64, npix; 0 on invalid
 * pixels, singletons and zero-RHS components), comp_iters[count] and
 * comp_status[count] (0 converged / zero RHS / singleton, 1 hit the cap
 * max(cg_max_iters, size)).  fp32 vectors + fp64 dots. */
int ni_fill_workspace_size(int B, int H, int W, int connectivity, int count, int weighted,
                           size_t* bytes);
int ni_fill(const int32_t* labels, int count, const double* omega_a, const double* omega_b,
            const double* gamma, const uint8_t* eflags, const double* w_a, const double* w_b,
            int B, int H, int W, int connectivity, int model, double cg_tol, int cg_max_iters,
            double* z_out, int32_t* comp_iters, int32_t* comp_status, void* workspace,
            size_t workspace_bytes, ni_stream_t stream);

/* K3 (default fill) -- fill_components (solver.py:195-239) at z = 0 as ONE
 * batched multigrid-preconditioned CG over every solve unit of every map
 * (csrc/ni_mg.cu): the same systems as ni_fill (w_a = w_b = NULL), solved
 * to the reference's relative residual per unit (||r_u|| < cg_tol ||b_u||,
 * which implies the component's ||r_c|| < cg_tol ||b_c||; cap
 * max(cg_max_iters, n_c) iterations), then the null-space component removed
 * per unit -- the gauge of CG from x0 = 0.  Same outputs as ni_fill:
 * z_out (float64, npix), comp_iters[count] (PCG iterations, max over the
 * component's units) and comp_status[count] (1 = cap).  The hierarchy's size
 * depends on the data: if `workspace_bytes` is too small the call returns
 * NI_ERR_WORKSPACE and writes the bytes it needs to *needed_bytes (the
 * caller retries); on success *needed_bytes holds the bytes used.
 * SYNCHRONOUS. */
int ni_fill_mg_workspace_size(int B, int H, int W, int connectivity, int count, size_t* bytes);
int ni_fill_mg(const int32_t* labels, int count, const double* omega_a, const double* omega_b,
               const double* gamma, const uint8_t* eflags, int B, int H, int W, int connectivity,
               int model, double cg_tol, int cg_max_iters, double* z_out, int32_t* comp_iters,
               int32_t* comp_status, void* workspace, size_t workspace_bytes,
               size_t* needed_bytes, ni_stream_t stream);
/* Multigrid statistics of the last ni_fill_mg on the calling thread: coarse
 * levels, V-cycles run, unknowns per level (n_per_level[16], index 1..levels). */
int ni_fill_mg_last_report(int* levels, int* vcycles, int* n_per_level);
/* Measurement hook (not part of the reference interface): while on, ni_fill_mg
 * brackets each V-cycle's pass A, coarse levels, pass B and scalar step with
 * CUDA events on the call's stream and counts the active unit pixels of every
 * V-cycle; ni_fill_mg_last_profile returns the four summed times (ms4[4]) and
 * that pixel count.  Off by default; per calling thread. */
int ni_set_fill_profiling(int on);
int ni_fill_mg_last_profile(double* ms4, long long* px_vcycles);

/* Directed weights of every forward pixel edge at log-depth state z
 * (continuity.py:292-331, solver.py:253-278): wmode 0 = valid (uniform,
 * t < alignment_iters), 1 = valid * gamma^2 * bilateral(z) (edge_weights,
 * the refill pass), 2 = mode 1 * outlier weight (mode 0 off, 1 soft, 2
 * hard).  w_a / w_b: KF planes of npix doubles, 0 where no edge. */
int ni_edge_weights(const double* z, const double* omega_a, const double* omega_b,
                    const double* gamma, const uint8_t* eflags, int B, int H, int W,
                    int connectivity, int model, int wmode, int mode, double k, double outlier_low,
                    double outlier_high, double* w_a, double* w_b, ni_stream_t stream);

/* Energy of the pixel pair system at x, per map (pipeline.py:336-337):
 * energy_out[m] = sum over map m's edges of W_a res_a^2 + W_b res_b^2 with
 * res_a = x_a - x_b - omega_a, res_b = x_b - x_a - omega_b (fixed order). */
int ni_pair_energy_workspace_size(int B, size_t* bytes);
int ni_pair_energy(const double* x, const double* omega_a, const double* omega_b,
                   const double* w_a, const double* w_b, const uint8_t* eflags, int B, int H,
                   int W, int connectivity, int model, double* energy_out, void* workspace,
                   size_t workspace_bytes, ni_stream_t stream);

/* Inter-component edge list of a partition (graph.py:186-196): edge keys
 * (a*KF + k) with differing endpoint labels, ascending.  n_out[0] = K. */
int ni_inter_edges_workspace_size(int B, int H, int W, int connectivity, size_t* bytes);
int ni_inter_edges(const int32_t* labels, const uint8_t* eflags, int B, int H, int W,
                   int connectivity, int32_t* keys_out, int32_t* n_out, void* workspace,
                   size_t workspace_bytes, ni_stream_t stream);

/* Keep the inter keys (ascending, from ni_inter_edges) of maps with
 * map_keep[m] != 0 whose endpoints now carry different labels, in order
 * (after a merge, or when maps leave the outer loop; graph.py:186-196).
 * keys_out must not alias keys; n_out is a device int32. */
int ni_keys_filter_workspace_size(int K, size_t* bytes);
int ni_keys_filter(const int32_t* keys, int K, const int32_t* labels, const uint8_t* map_keep,
                   int H, int W, int connectivity, int32_t* keys_out, int32_t* n_out,
                   void* workspace, size_t workspace_bytes, ni_stream_t stream);

/* Static structure of the inter-component system of a batch's partition
 * (solver.py:153-180): per-edge endpoints and component pairs, runs of edges
 * per unordered component pair (sorted by edge index inside a run),
 * per-component incidence lists, the sparsity of the component Laplacian
 * A^T W A and the per-map edge ranges.  Component ids are the batch's global
 * labels in [0, count); keys: K inter edge keys (ascending, map-major).
 * SYNCHRONOUS (reads back the number of distinct pairs into n_pairs_host and,
 * when map_edges_host != NULL, the B per-map edge counts). */
int ni_quotient_workspace_size(int K, int count, int B, size_t* bytes);
int ni_quotient_build(const int32_t* keys, int K, const int32_t* labels, int count, int B, int H,
                      int W, int connectivity, void* quot_ws, size_t quot_bytes,
                      int32_t* n_pairs_host, int32_t* map_edges_host, ni_stream_t stream);

/* K4-K7 -- relative_scale_step (solver.py:253-303) at 0-based iteration t for
 * the maps active[0..nact) of the batch, each solved as its own CG (one CTA
 * per map, a cooperative launch for maps above 8192 components), followed by
 * z[valid] += s[label] (pipeline.py:181-182) on those maps' pixels -- or,
 * when zshift != NULL, deferred: the state is z + zshift[label] throughout
 * and only zshift[c] += s[c] is updated (ni_apply_shift folds it into z).
 * map_first[B+1], map_count[B] and active[nact] are HOST arrays (map m owns
 * component ids [map_first[m], map_first[m] + map_count[m])).  mode: 0 off,
 * 1 soft, 2 hard (continuity.py:140-158).  Outputs (device): scales[count],
 * residual[2K] (rows a, b interleaved like solver.py:_pair_system),
 * weights[2K], energy_out[B] and cg_ok_out[B] (entries of active maps).  The
 * right-hand side's roundoff null-space component is removed before the CG
 * ("Reference numerics").  Asynchronous. */
int ni_scale_step_workspace_size(int K, int count, int B, size_t* bytes);
int ni_scale_step(const void* quot_ws, size_t quot_bytes, int K, int count, int B,
                  const int32_t* map_first, const int32_t* map_count, const int32_t* active,
                  int nact, const int32_t* labels, const double* omega_a, const double* omega_b,
                  const double* gamma, const uint8_t* eflags, int H, int W, int connectivity,
                  int model, int t, int alignment_iters, int mode, double k, double outlier_low,
                  double outlier_high, double cg_tol, int cg_max_iters, double* z,
                  double* zshift, const int32_t* live, double* scales, double* residual,
                  double* weights, double* energy_out, int32_t* cg_ok_out, void* workspace,
                  size_t workspace_bytes, ni_stream_t stream);

/* The convergence test of the outer loop (pipeline.py:66-83) on the device,
 * so a run of iterations without merges needs no host round trip: after the
 * step at 1-based iteration t, every active map whose live[m] (device) is set
 * records e_hist[m * hist_stride + t - 1] = energy[m] and ok_hist[...] =
 * cg_ok[m], is tested against e_prev[m] (then overwritten) and, once
 * converged, gets live[m] = 0 and iters[m] = t.  ni_scale_step skips maps
 * whose live flag is 0 (pass live = NULL to run every active map).
 * active[nact] is a DEVICE list here; nlive (device, nullable) is decremented
 * once per map that converges.  Asynchronous. */
int ni_loop_decide(const double* energy, const int32_t* cg_ok, const int32_t* active, int nact,
                   int t, int max_iters, int alignment_iters, double delta_e_max,
                   double* e_prev, int32_t* live, int32_t* iters, double* e_hist,
                   int32_t* ok_hist, int hist_stride, int32_t* nlive, ni_stream_t stream);

/* k_iters outer iterations (0-based t .. t + k_iters - 1) for maps with
 * small quotients (<= max_edges inter edges and <= max_comps components,
 * ni_scale_fused_limits), one thread-block cluster (8 CTAs) per map of
 * active[0..nact) (HOST list), in a single launch: each iteration is
 * ni_scale_step with deferred scales (zshift) followed by ni_loop_decide; a
 * map's cluster stops at its convergence.  Same arguments and outputs as
 * those calls.  Asynchronous. */
int ni_scale_step_fused(const void* quot_ws, size_t quot_bytes, int K, int count, int B,
                        const int32_t* map_first, const int32_t* map_count,
                        const int32_t* active, int nact, const int32_t* labels,
                        const double* omega_a, const double* omega_b, const double* gamma,
                        const uint8_t* eflags, int H, int W, int connectivity, int model, int t,
                        int k_iters, int alignment_iters, int mode, double k, double outlier_low,
                        double outlier_high, double cg_tol, int cg_max_iters, const double* z,
                        double* zshift, double* scales, double* residual, double* weights,
                        double* energy_out, int32_t* cg_ok_out, int max_iters,
                        double delta_e_max, double* e_prev, int32_t* live, int32_t* iters,
                        double* e_hist, int32_t* ok_hist, int hist_stride, int32_t* nlive,
                        void* workspace, size_t workspace_bytes, ni_stream_t stream);
int ni_scale_fused_limits(int* max_edges, int* max_comps);

/* z[valid] += zshift[label] on the pixels of maps[0..nmaps) (a HOST list),
 * then zshift = 0 on those maps' components: the deferred scales of
 * ni_scale_step folded into the log-depth (pipeline.py:181-182), before a
 * merge relabels the maps and at the end of the loop.  workspace: at least
 * 4 * nmaps bytes.  Asynchronous. */
int ni_apply_shift(double* z, double* zshift, const int32_t* labels, int B, int H, int W,
                   const int32_t* maps, int nmaps, void* workspace, size_t workspace_bytes,
                   ni_stream_t stream);

/* K8 -- merge_components (graph.py:207-250) for the maps merging[0..nmerge)
 * with |residual[2e]| as the merge key, plus their energies restricted to
 * edges that stay inter-component (pipeline.py:187-203) in energy_out[m].
 * Relabels those maps' pixels in place (labels of map m stay in
 * [map_first[m], map_first[m] + new_count)); new_count_out[B] (device) gets
 * every map's count.  Map tables are HOST arrays as for ni_scale_step. */
int ni_merge_workspace_size(int K, int count, int B, size_t* bytes);
int ni_merge(const void* quot_ws, size_t quot_bytes, int K, int count, int B,
             const int32_t* map_first, const int32_t* map_count, const int32_t* merging,
             int nmerge, int32_t* labels, int H, int W, const double* residual,
             const double* weights, int32_t* new_count_out, double* energy_out, void* workspace,
             size_t workspace_bytes, ni_stream_t stream);

/* 16-bit PNG normals (fileio.py:134-161): bgr = the inflated (H, W, 3)
 * uint16 samples as stored (BGR); writes n_out (H, W, 3) float64 = v / 65535
 * * 2 - 1 per channel (z negated if flip_z) divided by its norm, and
 * mask_out (all-zero pixels and zero norms are invalid); float64-exact. */
int ni_decode_png16(const uint16_t* bgr, int H, int W, int flip_z, double* n_out,
                    uint8_t* mask_out, ni_stream_t stream);

/* Evaluation (metrics.py:44-113), per map of a batch.  ni_evaluate: median
 * of gt/pred over jointly valid pixels (finite, > 0, in mask; mask may be
 * NULL) as the aligned scale, then out[4m..4m+3] = MADE, relative error,
 * scale, valid count (count 0: no overlap).  ni_min_theoretical_made: labels
 * = the partition's global labels, map_first[B+1] a HOST array of the maps'
 * label ranges; each component gets its exactly L1-optimal scale (weighted
 * median ratio); out[2m] = pixel-count weighted mean error, out[2m+1] = the
 * pixel count. */
int ni_evaluate_workspace_size(int B, int H, int W, size_t* bytes);
int ni_evaluate(const double* pred, const double* gt, const uint8_t* mask, int B, int H, int W,
                double* out, void* workspace, size_t workspace_bytes, ni_stream_t stream);
int ni_min_theoretical_made_workspace_size(int B, int H, int W, size_t* bytes);
int ni_min_theoretical_made(const double* pred, const double* gt, const uint8_t* mask,
                            const int32_t* labels, const int32_t* map_first, int B, int H, int W,
                            double* out, void* workspace, size_t workspace_bytes,
                            ni_stream_t stream);

/* K9 -- gauge fix (pipeline.py:86-88, 229): z += target - median(z[valid])
 * for each map separately (B medians); target = log(gauge_depth) or 0.
 * Optionally writes depth_out = exp(z) on valid pixels (geometry.py:180-184). */
int ni_gauge_workspace_size(int B, int H, int W, size_t* bytes);
int ni_gauge(double* z, const uint8_t* valid, int B, int H, int W, double target,
             double* depth_out, void* workspace, size_t workspace_bytes, ni_stream_t stream);

/* Serving read-back (run_pipeline_stream; the reference returns its depth in
 * host memory, pipeline.py:240-248): copy `bytes` from device memory `src` to
 * PINNED host memory `host_dst` with a `ctas`-CTA kernel storing through the
 * mapped (UVA) address instead of a copy engine, so the read-back of one batch
 * does not hold the device->host copy queue that the next batch's small
 * control reads use.  NI_ERR_INVALID_ARG if host_dst is not pinned or the two
 * pointers differ in 16-byte alignment. */
int ni_copy_to_host(const void* src, void* host_dst, size_t bytes, int ctas, ni_stream_t stream);

/* The upload twin of ni_copy_to_host: `ctas` CTAs read pinned (mapped) host
 * memory and store `bytes` bytes into device memory `dst` on `stream`
 * (run_pipeline_stream's upload of the next batch; no reference counterpart).
 * Same argument rules. */
int ni_copy_from_host(void* dst, const void* host_src, size_t bytes, int ctas, ni_stream_t stream);

#ifdef __cplusplus
}
#endif

#endif /* NORMINT_B200_H */
