/*
 * gnn_b200.h — C ABI of the B200-native sparse GNN hot path (libgnnb200.so).
 *
 * Everything here is plain C: device pointers, sizes, and an opaque CUDA
 * stream handle.  No torch types cross this boundary.  Every entry point
 * returns a gnn_status (0 = ok); the Python host layer maps the codes to the
 * reference's exception taxonomy (gsbench/errors.py:5-29).
 *
 * Ownership: all buffers are caller-owned.  The library never allocates
 * persistent device memory; scratch comes in through (ws, ws_bytes), sized by
 * the matching *_workspace() query, so the caller's allocator accounts for
 * every byte of peak memory.
 *
 * Threading: every compute entry point is stream-ordered, reentrant and free
 * of host synchronisation (CUDA-graph capturable).  The *builders* (CSR/CSC
 * construction, validation) synchronise the stream once at the end, because
 * they must report the reference's validation errors before returning
 * (graph.py:95-102, sampler.py:250-251).
 *
 * Reference interfaces replaced (file:line under the reference tree):
 *   gnn_csr_from_edges      <- gsbench.graph.csr_from_edges   graph.py:106-114
 *   gnn_csr_validate        <- gsbench.graph.make_csr         graph.py:91-103
 *   gnn_subgraph_csr        <- gsbench.build_subgraph_csr     sampler.py:242-256
 *   gnn_degrees             <- CsrGraph.degrees               graph.py:39-41
 *   gnn_csc_from_csr        <- csr_from_edges(V, targets, rows) (transposed CSR)
 *   gnn_generate_powerlaw   <- gsbench.graph.generate, power-law branch  graph.py:254-262
 *   gnn_spmm                <- GraphPy SpMMv / SpMMve (+T)    PAPER.md:264-278 (prose only)
 *   gnn_degree_norm_inplace <- GraphPy in-place degree-norm
 *   gnn_sddmm               <- GraphPy SDDMM on CSR-style COO PAPER.md:281-287
 *   gnn_gat_*               <- GAT edge-softmax state tensor
 *   gnn_gemm*               <- the dense X.W transform, modelled as b_f*V*K in
 *                              execmodel.py:374-378
 */
#ifndef GNN_B200_H
#define GNN_B200_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

typedef void *gnn_stream_t; /* a cudaStream_t (CUstream); NULL = legacy default stream */

typedef enum gnn_status {
  GNN_OK = 0,
  GNN_ERR_INVALID_ARGUMENT = 1, /* bad shape / pointer / flag combination       -> ValueError  */
  GNN_ERR_CSR_INVARIANT = 2,    /* offsets malformed (graph.py:95-100)           -> ValueError  */
  GNN_ERR_RANGE = 3,            /* target id outside [0, V) (graph.py:101-102)   -> RangeError  */
  GNN_ERR_INDEX = 4,            /* subgraph source id out of range (sampler.py:250-251) -> IndexError */
  GNN_ERR_WORKSPACE = 5,        /* ws_bytes smaller than the *_workspace() query */
  GNN_ERR_CUDA = 6,             /* a CUDA runtime error (gnn_last_cuda_error())  -> RuntimeError */
  GNN_ERR_UNSUPPORTED = 7,      /* shape the kernels do not cover                -> ValueError  */
  GNN_ERR_SOURCE_RANGE = 8      /* csr_from_edges source id outside [0, V): numpy's bincount/cumsum
                                   shape error in the reference (graph.py:110-112) -> ValueError */
} gnn_status;

/* ---------------------------------------------------------------- misc */
int gnn_abi_version(void);                 /* bumped on any signature change */
/* Persisting-L2 controls (gathers whose hot rows are a prefix of the gathered
 * array, e.g. a degree-ordered numbering): the set-aside size, the largest
 * access-policy window, and a stream's window (hot prefix persisting, misses
 * streaming; bytes = 0 clears it). */
int64_t gnn_l2_max_window(void);
int gnn_l2_persist_limit(int64_t bytes);
int gnn_l2_window(gnn_stream_t stream, const void *base, int64_t bytes, float hit_ratio);
/* "src:<sha256[:16] of the library's sources> git:<sha> sm_100a" — the
 * provenance smoke() and bench.py check against the shipped sources. */
const char *gnn_build_id(void);
const char *gnn_strerror(int status);
int gnn_last_cuda_error(void);             /* cudaError_t of the last GNN_ERR_CUDA */
int gnn_device_sm_count(void);             /* SMs of the current device */
int64_t gnn_launch_counter(void);          /* kernels launched by this library so far */
/* Diagnostic: every CTA reads buf[0:n_floats) `reps` times (128-bit, L2-cached
 * loads) — with an L2-resident buffer this measures the L2 -> SM roof that
 * bounds the SpMM's row gathers.  out receives nothing meaningful. */
int gnn_read_probe(const float *buf, int64_t n_floats, int reps, float *out, gnn_stream_t stream);
/* Strided 2-D copy (cudaMemcpyDefault: host<->device or device<->device),
 * stream-ordered, no staging buffer — used to put [V, F] host features into
 * the padded [V, Fpad] device layout the TMA-fed GEMMs need. */
int gnn_memcpy2d(void *dst, size_t dpitch, const void *src, size_t spitch, size_t width,
                 size_t height, gnn_stream_t stream);

/* ------------------------------------------------------- graph builders */
/* Stable counting sort of (src,dst) pairs into CSR: offsets[V+1] int64,
 * targets[E] int32, bit-exact with graph.py:106-114 (stable within a row,
 * multigraph duplicates kept).  Errors: GNN_ERR_SOURCE_RANGE if a src is
 * outside [0,V); GNN_ERR_RANGE if a dst is outside [0,V) (make_csr check). */
size_t gnn_csr_from_edges_workspace(int64_t num_vertices, int64_t num_edges);
int gnn_csr_from_edges(int64_t num_vertices, int64_t num_edges, const int64_t *src,
                       const int64_t *dst, int64_t *offsets, int32_t *targets, void *ws,
                       size_t ws_bytes, gnn_stream_t stream);

/* build_subgraph_csr (sampler.py:242-256): same stable build over local ids;
 * GNN_ERR_INDEX if a source is outside [0,num_local_src); dst is truncated to
 * int32 without a range check, as LOCAL_DTYPE astype does. */
size_t gnn_subgraph_csr_workspace(int64_t num_local_src, int64_t num_edges);
int gnn_subgraph_csr(int64_t num_local_src, int64_t num_edges, const int64_t *edge_src,
                     const int64_t *edge_dst, int64_t *offsets, int32_t *targets, void *ws,
                     size_t ws_bytes, gnn_stream_t stream);

/* make_csr invariants (graph.py:95-102) on device arrays. */
size_t gnn_csr_validate_workspace(int64_t num_vertices, int64_t num_edges);
int gnn_csr_validate(int64_t num_vertices, int64_t num_edges, const int64_t *offsets,
                     const int32_t *targets, void *ws, size_t ws_bytes, gnn_stream_t stream);

/* degrees = diff(offsets) (graph.py:39-41). */
int gnn_degrees(int64_t num_vertices, const int64_t *offsets, int64_t *degrees,
                gnn_stream_t stream);

/* Transposed CSR (CSC) by a stable sort of the CSR by column id:
 * t_offsets[num_cols+1], t_rows[nnz]; optional t_eid[nnz] = CSR position of
 * each CSC entry (the GraphPy edge-ID array).  Equal to
 * csr_from_edges(num_cols, targets, rows) of the reference. */
size_t gnn_csc_from_csr_workspace(int64_t num_rows, int64_t num_cols, int64_t nnz);
int gnn_csc_from_csr(int64_t num_rows, int64_t num_cols, int64_t nnz, const int64_t *offsets,
                     const int32_t *cols, int64_t *t_offsets, int32_t *t_rows, int32_t *t_eid,
                     void *ws, size_t ws_bytes, gnn_stream_t stream);

/* Multigraph coalescing of a CSR whose rows are sorted by column (e.g. the
 * transpose of a CSC): unique (row,col) pairs with their multiplicity as a
 * float edge value.  out_offsets[num_rows+1], out_cols/out_mult sized nnz
 * (upper bound); *out_nnz (host) receives the unique count (one sync). */
size_t gnn_csr_coalesce_workspace(int64_t num_rows, int64_t nnz);
int gnn_csr_coalesce(int64_t num_rows, int64_t nnz, const int64_t *offsets, const int32_t *cols,
                     int64_t *out_offsets, int32_t *out_cols, float *out_mult, int64_t *out_nnz,
                     void *ws, size_t ws_bytes, gnn_stream_t stream);

/* Packed-weight operand for gnn_spmm (see gnn_csr_view_t.col_bits):
 * out[j] = cols[j] | (uint32)weights[j] << col_bits.  GNN_ERR_RANGE (one
 * sync) if a column needs more than col_bits bits or a weight is not an
 * integer in [0, 2^(32-col_bits)) — the caller keeps the float form then. */
size_t gnn_csr_pack_weights_workspace(void);
int gnn_csr_pack_weights(int64_t nnz, const int32_t *cols, const float *weights, int32_t col_bits,
                         int32_t *out, void *ws, size_t ws_bytes, gnn_stream_t stream);

/* Chung-Lu power-law edge draws of graph.py:256-261, bit-exact: numpy PCG64
 * (state,inc given as 128-bit hi/lo words of the SeedSequence-seeded
 * generator) position k -> double (raw>>11)*2^-53; src uses positions
 * [0,m), dst [m,2m); endpoint = searchsorted(cdf, u, 'right').  cdf is the
 * host-computed float64 CDF of graph.py:256-259 (length n). */
size_t gnn_generate_powerlaw_workspace(int64_t n);
int gnn_generate_powerlaw(int64_t n, int64_t m, const double *cdf, uint64_t state_hi,
                          uint64_t state_lo, uint64_t inc_hi, uint64_t inc_lo, int64_t *src,
                          int64_t *dst, void *ws, size_t ws_bytes, gnn_stream_t stream);

/* Row-block build of the power-law graph for the 1D row partition (SURVEY
 * §8e), without materialising the whole graph: the bit-exact edge stream of
 * gnn_generate_powerlaw is regenerated in `chunk`-edge pieces and, in stream
 * order, (src-lo, dst) of every edge with src in [lo,hi) is appended to
 * r_key/r_val and (dst-lo, src) of every edge with dst in [lo,hi) to
 * c_key/c_val (either pair may be NULL to skip it); count[2] (device)
 * receives the two totals.  At most `capacity` pairs are written per output
 * (the caller sizes it, e.g. the expected block size plus a margin, and
 * re-runs with count's exact totals if count exceeds it).  Stable sorts of these pairs (gnn_sort_pairs) give rows
 * lo..hi-1 of csr_from_edges (graph.py:106-114) and of its transpose. */
size_t gnn_powerlaw_block_workspace(int64_t n, int64_t chunk);
int gnn_powerlaw_block(int64_t n, int64_t m, const double *cdf, uint64_t state_hi,
                       uint64_t state_lo, uint64_t inc_hi, uint64_t inc_lo, int64_t lo, int64_t hi,
                       int64_t chunk, int64_t capacity, int32_t *r_key, int32_t *r_val,
                       int32_t *c_key, int32_t *c_val, int64_t *count, void *ws, size_t ws_bytes,
                       gnn_stream_t stream);
/* Stable LSD radix sort of int32 (key, val) pairs, keys in [0, key_limit). */
size_t gnn_sort_pairs_workspace(int64_t n, int64_t key_limit);
int gnn_sort_pairs(int64_t n, int64_t key_limit, const int32_t *keys, const int32_t *vals,
                   int32_t *keys_out, int32_t *vals_out, void *ws, size_t ws_bytes,
                   gnn_stream_t stream);
/* offsets[R+1] from sorted int32 row keys in [0, R) (= the CSR offsets). */
size_t gnn_offsets_from_keys_workspace(int64_t R);
int gnn_offsets_from_keys(int64_t n, int64_t R, const int32_t *sorted_keys, int64_t *offsets,
                          void *ws, size_t ws_bytes, gnn_stream_t stream);

/* --------------------------------------- sampled-block pipeline (ZeroGNN) */
/* sample_hop (sampler.py:118-144), bit-exact with numpy's PCG64 Generator
 * whose (state, inc) is given as 128-bit hi/lo words: active = frontier
 * vertices of nonzero degree (order kept); draw j < A*fanout:
 *   src[j] = frontier[active[j / fanout]],
 *   dst[j] = targets[offsets[src] + floor(u_j * deg(src))],  u_j = stream position j.
 * src/dst have capacity F*fanout; *count (device) receives A*fanout. */
size_t gnn_sample_hop_workspace(int64_t F);
int gnn_sample_hop(int64_t V, const int64_t *offsets, const int32_t *targets,
                   const int64_t *frontier, int64_t F, int64_t fanout, uint64_t state_hi,
                   uint64_t state_lo, uint64_t inc_hi, uint64_t inc_lo, int64_t *src, int64_t *dst,
                   int64_t *count, void *ws, size_t ws_bytes, gnn_stream_t stream);
/* dedup_relabel (sampler.py:191-239): table[V] (global -> local, -1 unseen) is
 * updated in place; destinations first seen in this hop get locals start,
 * start+1, ... in first-occurrence order (new_globals, *new_count on device);
 * src_local / dst_local are the relabelled draws; *error_flag = 1 when a
 * source is not yet in the table (the reference's ValueError).  firstpos[V]
 * is scratch that must hold INT32_MAX on entry and does on exit. */
size_t gnn_dedup_relabel_workspace(int64_t n);
int gnn_dedup_relabel(int64_t V, int32_t *table, int32_t *firstpos, const int64_t *src_g,
                      const int64_t *dst_g, int64_t n, int64_t start, int32_t *src_local,
                      int32_t *dst_local, int64_t *new_globals, int64_t *new_count,
                      int32_t *error_flag, void *ws, size_t ws_bytes, gnn_stream_t stream);
/* out[i] = table[ids[i]];  table[ids[i]] = start + i */
int gnn_table_lookup(const int32_t *table, const int64_t *ids, int64_t n, int32_t *out,
                     gnn_stream_t stream);
int gnn_table_assign(int32_t *table, const int64_t *ids, int64_t n, int64_t start,
                     gnn_stream_t stream);

/* Device-resident-count forms (ZeroGNN DRMB): sizes are
 * read from device scalars (F_dev, n_dev, size_dev), buffers are provisioned
 * for a capacity envelope, grids cover the capacity with early exit
 * (PAPER.md:1472-1474), and the PCG64 (state, inc) words come from device
 * memory (rng_state[4] = state_hi, state_lo, inc_hi, inc_lo) — no host sync
 * anywhere, so a whole mini-batch can be captured and replayed.
 * gnn_dedup_relabel_dev reads the builder size from *size_dev and adds the
 * hop's new-vertex count to it. */
size_t gnn_sample_hop_dev_workspace(int64_t F_cap);
int gnn_sample_hop_dev(int64_t V, const int64_t *offsets, const int32_t *targets,
                       const int64_t *frontier, const int64_t *F_dev, int64_t F_cap, int64_t fanout,
                       const uint64_t *rng_state, int64_t *src, int64_t *dst, int64_t *count,
                       void *ws, size_t ws_bytes, gnn_stream_t stream);
size_t gnn_dedup_relabel_dev_workspace(int64_t n_cap);
int gnn_dedup_relabel_dev(int64_t V, int32_t *table, int32_t *firstpos, const int64_t *src_g,
                          const int64_t *dst_g, const int64_t *n_dev, int64_t n_cap,
                          int64_t *size_dev, int32_t *src_local, int32_t *dst_local,
                          int64_t *new_globals, int64_t *new_count, int32_t *error_flag, void *ws,
                          size_t ws_bytes, gnn_stream_t stream);
int gnn_table_lookup_dev(const int32_t *table, const int64_t *ids, const int64_t *n_dev,
                         int64_t n_cap, int32_t *out, gnn_stream_t stream);
/* table[ids[i]] = value for i < *n_dev (n_dev NULL: i < n_cap) — resets the
 * builder table between replayed mini-batches. */
int gnn_table_fill_dev(int32_t *table, const int64_t *ids, const int64_t *n_dev, int64_t n_cap,
                       int32_t value, gnn_stream_t stream);

/* Feature gather of a sampled mini-batch (the pipeline's "gather" kernel,
 * execmodel.py:306-314; rows = gather_indices, sampler.py:299-305):
 * out[i, :] = X[ids[i], :]. */
int gnn_gather_rows(const float *X, int64_t ldx, const int64_t *ids, int64_t n, int64_t K,
                    float *out, int64_t ldo, gnn_stream_t stream);
/* gnn_gather_rows over the first *n_dev of n_cap rows (device count; rows at
 * or past it untouched): the feature gather of a replayed mini-batch. */
int gnn_gather_rows_dev(const float *X, int64_t ldx, const int64_t *ids, const int64_t *n_dev,
                        int64_t n_cap, int64_t K, float *out, int64_t ldo, gnn_stream_t stream);

/* ----------------------------------------------------------- sparse ops */
/* A device CSR (or CSC, which is the CSR of the transpose). */
typedef struct gnn_csr_view {
  int64_t num_rows;
  int64_t num_cols;
  int64_t nnz;
  const int64_t *offsets;     /* [num_rows+1] */
  const int32_t *cols;        /* [nnz] column ids */
  const float *vals;          /* [nnz*heads] edge values, or NULL (SpMMv: implicit 1, no |E| tensor) */
  const int32_t *eid;         /* [nnz] or NULL: edge value of entry j is vals[eid[j]] (SpMMve^T) */
  const int64_t *deg_offsets; /* degree source for GNN_EPI_NORM, NULL = offsets */
  /* 0, or (gnn_spmm / gnn_spmm_peer only; vals == NULL, heads == 1) the
   * packed-weight form built by gnn_csr_pack_weights: entry j is column
   * cols[j] & (2^col_bits - 1) with edge value (float)(cols[j] >> col_bits)
   * — the coalesced multigraph operand (multiplicities) in 4 bytes per edge.
   * Every other entry point rejects col_bits != 0. */
  int32_t col_bits;
  int32_t reserved_;
  /* NULL, or (gnn_spmm / gnn_spmm_peer only) a row-permuted operand: operand
   * row i produces output row row_ids[i], and every per-row epilogue input
   * (deg_offsets, self_x, mask, bias row, post_deg_offsets) is indexed by
   * row_ids[i].  Used for the degree-sorted form (rows longest-first), whose
   * long rows form a prefix the nnz-split kernel covers alone.  NORM then
   * requires deg_offsets (indexed by output row). */
  const int32_t *row_ids;
} gnn_csr_view_t;

/* Epilogue applied per output row v, in this order:
 *   y  = acc                           (acc = sum_e val_e * X[col_e])
 *   y *= 1/deg(v)       if NORM        (deg(v)==0 -> y = 0, no clamp buffer)
 *   y += self_scale*S[v] if SELF       (GIN (1+eps) self term)
 *   y += bias           if BIAS
 *   y  = max(y,0)       if RELU
 *   y  = M[v]>0 ? y : 0 if MASK        (ReLU backward against a saved activation)
 *   y *= 1/pdeg(v)      if POSTNORM    (degree-norm of the NEXT backward SpMM's input)
 */
enum {
  GNN_EPI_NORM = 1u << 0,
  GNN_EPI_SELF = 1u << 1,
  GNN_EPI_BIAS = 1u << 2,
  GNN_EPI_RELU = 1u << 3,
  GNN_EPI_MASK = 1u << 4,
  GNN_EPI_POSTNORM = 1u << 5
};
typedef struct gnn_epilogue {
  uint32_t flags;
  float self_scale;
  const float *self_x; /* [num_rows, ld_self] */
  int64_t ld_self;
  const float *bias; /* [K] */
  const float *mask; /* [num_rows, ld_mask] */
  int64_t ld_mask;
  const int64_t *post_deg_offsets; /* [num_rows+1] */
} gnn_epilogue_t;

/* Per-graph SpMM schedule (built once, reused by every call; the build
 * synchronises once to learn the list lengths so that gnn_spmm never does).
 * The nnz range is cut into chunks of edges_per_warp edges, one warp each;
 * chunk_row[w] is the row holding chunk w's first edge.  A row spanning
 * several chunks ("split" row) is finished inside the SpMM kernel by the last
 * warp to deliver a partial (fence + arrival counter; partials summed in a
 * fixed two-level order, groups of 64).  Empty rows are listed for the
 * epilogue-only pass.  All arrays live in one caller buffer of
 * gnn_spmm_plan_buffer_ints() int32 entries; the plan is read-only, so one
 * plan may serve concurrent calls on different streams. */
typedef struct gnn_spmm_plan {
  int64_t edges_per_warp;          /* multiple of 4, <= 2048 */
  int64_t num_warps;               /* ceil(main_nnz / edges_per_warp) */
  const int32_t *chunk_row;        /* [num_warps+1] */
  const int32_t *chunk_split;      /* [2*num_warps] split index of carry-in / trailing row or -1 */
  int64_t num_split;
  const int32_t *split_rows;       /* [num_split] */
  const int32_t *split_group_base; /* [num_split+1] prefix of ceil(partials/64) */
  int64_t num_groups;
  int64_t num_empty;
  const int32_t *empty_rows;       /* [num_empty] */
  int64_t short_max;               /* rows with 1 <= deg <= short_max go to the short-row kernel */
  int64_t num_short;
  const int32_t *short_rows;       /* [num_short], longest first */
  int64_t main_nnz;                /* edges the nnz-split kernel covers: nnz, or — for a
                                      permuted operand (row_ids) whose rows of degree >
                                      short_max form a prefix (degree-sorted) — that
                                      prefix's edge count; gnn_spmm then needs the
                                      short-row kernel (K <= 64, 16-byte rows) */
  const int64_t *dev_counts;       /* NULL, or (gnn_spmm_plan_build_dev) device
                                      [num_split, num_empty, num_groups, num_short]
                                      of this batch; the host fields above then hold
                                      capacities and the kernels stop at the device
                                      counts (a capturable, host-sync-free plan) */
  const int64_t *row_limit;        /* NULL, or (device) rows >= *row_limit are not computed
                                      (their outputs left untouched): the live rows of a
                                      capacity-sized operand */
} gnn_spmm_plan_t;

size_t gnn_spmm_plan_buffer_ints(int64_t num_rows, int64_t nnz, int64_t edges_per_warp);
size_t gnn_spmm_plan_workspace(int64_t num_rows);
int gnn_spmm_plan_build(const gnn_csr_view_t *A, int64_t edges_per_warp, int32_t *plan_buf,
                        gnn_spmm_plan_t *plan, void *ws, size_t ws_bytes, gnn_stream_t stream);
/* Degree-binned plan for gnn_spmm: rows with 1 <= deg <= short_max (the
 * power-law tail) are listed for a group-per-row kernel (32/G rows per warp
 * in parallel) and skipped by the nnz-split kernel, so a warp never walks a
 * run of tiny rows one by one.  short_max = 0 gives gnn_spmm_plan_build's
 * plan (the form the edge-softmax / SDDMM / GAT kernels expect). */
int gnn_spmm_plan_build_ex(const gnn_csr_view_t *A, int64_t edges_per_warp, int64_t short_max,
                           int32_t *plan_buf, gnn_spmm_plan_t *plan, void *ws, size_t ws_bytes,
                           gnn_stream_t stream);

/* Host-sync-free plan for an operand whose row structure changes from call
 * to call inside one fixed-size buffer (sampled mini-batch subgraphs replayed
 * as one CUDA graph): same schedule as
 * gnn_spmm_plan_build_ex (row-order operands only: A->row_ids must be NULL;
 * short rows in row order), counts written to counts_dev[4] on device, host
 * counts set to capacities; row_limit_dev (nullable) = the live row count.
 * Only gnn_spmm accepts such a plan. */
int gnn_spmm_plan_build_dev(const gnn_csr_view_t *A, int64_t edges_per_warp, int64_t short_max,
                            int32_t *plan_buf, gnn_spmm_plan_t *plan, int64_t *counts_dev,
                            const int64_t *row_limit_dev, void *ws, size_t ws_bytes,
                            gnn_stream_t stream);

/* Y[num_rows,K] = epilogue(A . X), X[num_cols,K].  heads>=1 splits K into
 * `heads` slices scaled by their own edge value (vals is [nnz,heads]).
 * Deterministic (fixed summation order), no atomics on Y. */
size_t gnn_spmm_workspace(const gnn_csr_view_t *A, const gnn_spmm_plan_t *plan, int64_t K);
int gnn_spmm(const gnn_csr_view_t *A, const gnn_spmm_plan_t *plan, int64_t heads,
             const float *X, int64_t ldx, float *Y, int64_t ldy, int64_t K,
             const gnn_epilogue_t *epi, void *ws, size_t ws_bytes, gnn_stream_t stream);

/* Four attention heads over ONE shared feature row (GAT output layer in the
 * aggregate-then-transform order): Y[v, 4i+h] = scale * sum_e vals[e*4+h] *
 * X[col_e, i], i < F; Y is [num_rows, 4F] (head-minor, so Y viewed as
 * [num_rows*F, 4] rows line up with W[F, 4*C] viewed as [4F, C] rows: the
 * head mean of sum_e alpha_eh (X W_h)[col_e] is then one GEMM Y . W).  vals
 * [nnz*4] in CSR edge order (16-byte aligned), no eid / packed / row_ids;
 * a plan with short_max = 0 (the nnz-split kernel covers every row).  Gathers
 * F floats per edge instead of 4C. */
int gnn_spmm_shared_heads(const gnn_csr_view_t *A, const gnn_spmm_plan_t *plan, const float *X,
                          int64_t ldx, int64_t F, float *Y, int64_t ldy, float scale,
                          const gnn_epilogue_t *epi, void *ws, size_t ws_bytes,
                          gnn_stream_t stream);

/* Row-partitioned multi-GPU form of gnn_spmm (fused with the
 * exchange): instead of all-gathering the feature blocks first, the kernel
 * reads every gathered row in place from the rank that owns it — column id c
 * lives at row (c & (2^part_rows_log2 - 1)) of parts[c >> part_rows_log2],
 * where parts[] are peer-mapped device pointers (NVLink / NVSwitch P2P loads,
 * e.g. from torch symmetric memory) or local buffers.  heads = 1, K <= 64,
 * fp32 rows 16-byte aligned; nparts <= 8. */
int gnn_spmm_peer(const gnn_csr_view_t *A, const gnn_spmm_plan_t *plan, const float *const *parts,
                  int64_t nparts, int64_t part_rows_log2, int64_t ldx, float *Y, int64_t ldy,
                  int64_t K, const gnn_epilogue_t *epi, void *ws, size_t ws_bytes,
                  gnn_stream_t stream);

/* X[v,:] /= deg(v) in place (deg 0 -> row zeroed). */
int gnn_degree_norm_inplace(int64_t num_rows, const int64_t *offsets, float *X, int64_t ldx,
                            int64_t K, gnn_stream_t stream);

/* ------------------------------------------------- SDDMM / edge softmax */
/* SDDMM on the CSR (GraphPy "CSR-style COO"):
 *   out[e,h] = < X[row_e, h*F:(h+1)*F], Y[col_e, h*F:(h+1)*F] >,  F = K/heads,
 * in CSR edge order.  Edge-parallel over the plan's chunks; the row operand
 * is loaded once per row run and reused across the run's edges.  Also the
 * SpMMve backward w.r.t. the edge values (dalpha = SDDMM(dY, X)). */
int gnn_sddmm(const gnn_csr_view_t *A, const gnn_spmm_plan_t *plan, int64_t heads, const float *X,
              int64_t ldx, const float *Y, int64_t ldy, int64_t K, float *out,
              gnn_stream_t stream);

/* Edge scores for the edge softmax: given (s = [nnz, heads]) or, when s is
 * NULL, the GAT score of SURVEY Appendix A.6 computed on the fly:
 *   s[e,h] = LeakyReLU(el[col_e,h] + er[row_e,h], slope)   (el [num_cols,H], er [num_rows,H]). */
typedef struct gnn_edge_scores {
  const float *s;
  const float *el;
  const float *er;
  float slope;
} gnn_edge_scores_t;

/* alpha[e,h] = exp(s[e,h] - max_row) / sum_row exp(.)  over each CSR row (per
 * head); the attention state tensor of PAPER.md:606-617.  alpha may alias s.
 * Deterministic (fixed-order reductions; rows spanning several chunks are
 * combined from per-chunk partials).  heads <= 16. */
size_t gnn_edge_softmax_workspace(const gnn_spmm_plan_t *plan, int64_t heads);
int gnn_edge_softmax_fwd(const gnn_csr_view_t *A, const gnn_spmm_plan_t *plan, int64_t heads,
                         const gnn_edge_scores_t *scores, float *alpha, void *ws, size_t ws_bytes,
                         gnn_stream_t stream);
/* ds[e,h] = alpha (dalpha - sum_row alpha*dalpha); when scores->el is given
 * (GAT mode) also times LeakyReLU'(el[col]+er[row]).  ds may alias dalpha. */
int gnn_edge_softmax_bwd(const gnn_csr_view_t *A, const gnn_spmm_plan_t *plan, int64_t heads,
                         const float *alpha, const float *dalpha, const gnn_edge_scores_t *scores,
                         float *ds, void *ws, size_t ws_bytes, gnn_stream_t stream);

/* Row sums of an edge tensor: out[r,h] = sum_{j in row r} vals[idx_j*heads + h],
 * idx_j = A->eid[j] when the view carries an edge-ID array (column sums of a
 * CSR-ordered edge tensor through the CSC), else j.  Empty rows give 0.
 * Workspace: gnn_edge_softmax_workspace(plan, heads).  Deterministic. */
int gnn_segment_sum(const gnn_csr_view_t *A, const gnn_spmm_plan_t *plan, int64_t heads,
                    const float *vals, float *out, void *ws, size_t ws_bytes, gnn_stream_t stream);

/* Fused GAT backward over the CSC (AT must carry the edge-ID array): one
 * gather of dY per edge feeds both the SpMMve^T and the SDDMM
 *   dWh[u,:]         = sum_{j in CSC row u} alpha[eid_j, head] * dY[row_j, :]
 *   dalpha[eid_j, h] = < dY[row_j, head h], Wh[u, head h] >
 * alpha / dalpha are [nnz, heads] in CSR edge order.  K % 4 == 0, F % 4 == 0,
 * K <= 512, heads <= 8.  Deterministic. */
size_t gnn_gat_bwd_csc_workspace(const gnn_spmm_plan_t *plan, int64_t K);
int gnn_gat_bwd_csc(const gnn_csr_view_t *AT, const gnn_spmm_plan_t *plan, int64_t heads,
                    const float *alpha, const float *dY, int64_t ldy, const float *Wh, int64_t ldw,
                    int64_t K, float *dWh, int64_t ldd, float *dalpha, void *ws, size_t ws_bytes,
                    gnn_stream_t stream);

/* The same for a head-MEAN output layer, whose concatenated-head gradient is
 * dZ * scale broadcast to every head (scale = 1/heads): only dZ[v] (F floats)
 * is gathered per edge, and all heads are produced from it:
 *   dWh[u, h*F+f]    = scale * sum_j alpha[eid_j, h] * dZ[row_j, f]
 *   dalpha[eid_j, h] = scale * < dZ[row_j, :], Wh[u, h*F:(h+1)*F] >
 * Workspace: gnn_gat_bwd_csc_workspace(plan, heads*F).  F % 4 == 0, F <= 128. */
int gnn_gat_bwd_csc_mean(const gnn_csr_view_t *AT, const gnn_spmm_plan_t *plan, int64_t heads,
                         const float *alpha, const float *dZ, int64_t ldz, float scale,
                         const float *Wh, int64_t ldw, int64_t F, float *dWh, int64_t ldd,
                         float *dalpha, void *ws, size_t ws_bytes, gnn_stream_t stream);

/* ---- GAT backward with alpha recomputed (4 heads; the trainers' path).
 * Replaces the alpha/dalpha [E,4] round trip of gnn_gat_bwd_csc(_mean) +
 * gnn_edge_softmax_bwd + the two gnn_segment_sum passes (PAPER.md:264-268,
 * 606-617: the attention state is the softmax's per-row statistics, not an
 * edge tensor, in the backward).
 *
 * Forward: the GAT edge softmax that also writes rowstat [R][2*heads] =
 * (row max m[h]..., 1/row sum inv[h]...).  alpha as gnn_edge_softmax_fwd. */
int gnn_gat_softmax_fwd_stats(const gnn_csr_view_t *A, const gnn_spmm_plan_t *plan, int64_t heads,
                              const gnn_edge_scores_t *scores, float *alpha, float *rowstat,
                              void *ws, size_t ws_bytes, gnn_stream_t stream);
/* Per-row backward statistics of a GAT layer, four float4 {er, m, inv, S}
 * (one per head) at stat + v*ldst, with
 * S[v,h] = sum_e alpha dalpha = < dYm_h[v], Y_h[v] - bias_h > (concatenated
 * heads: dYm the ReLU-masked upstream gradient, Y = relu(aggregate + bias)).
 * The recompute backward wants them right after the gradient row: stat =
 * dYm + K, ldst = ldd.  K = 4F, K % 16 == 0, K <= 128. */
int gnn_gat_rowstat(int64_t V, int64_t K, const float *dYm, int64_t ldd, const float *Y,
                    int64_t ldy, const float *bias, const float *er, const float *rowstat,
                    float *stat, int64_t ldst, gnn_stream_t stream);
/* The same for the head-mean output layer kept in the aggregate-then-transform
 * order (gnn_spmm_shared_heads: Yc [V, 4*F1], W [F1, 4*Cp]):
 *   S[v,h] = scale * sum_i Yc[v,4i+h] * sum_c W[i, h*Cp+c] dZ[v,c].  Cp % 4 == 0, Cp <= 64. */
int gnn_gat_rowstat_mean(int64_t V, int64_t F1, int64_t Cp, const float *dZ, int64_t ldz,
                         const float *Yc, int64_t ldc, const float *W, int64_t ldw, float scale,
                         const float *er, const float *rowstat, float *stat, int64_t ldst,
                         gnn_stream_t stream);
/* The same on the tensor cores (split-TF32 tcgen05: G = dZ W_h^T per head,
 * reduced against Yc in the GEMM epilogue, G never stored); W dense
 * (ldw == 4*Cp), V >= 128; GNN_ERR_UNSUPPORTED otherwise.  Same statistics
 * layout as gnn_gat_rowstat_mean; caller-owned workspace. */
size_t gnn_gat_rowstat_mean_tc_workspace(int64_t F1, int64_t Cp);
int gnn_gat_rowstat_mean_tc(int64_t V, int64_t F1, int64_t Cp, const float *dZ, int64_t ldz,
                            const float *Yc, int64_t ldc, const float *W, int64_t ldw, float scale,
                            const float *er, const float *rowstat, float *stat, int64_t ldst,
                            void *ws, size_t ws_bytes, gnn_stream_t stream);
/* GAT layer transform with its attention projections in the tcgen05 GEMM's
 * epilogue: C = A B (B [Kd, N] row-major, N = 4F, F % 16 == 0), el[r, h] =
 * <C[r, hF:(h+1)F], a_l[h]>, er[r, h] = <C[r, hF:(h+1)F], a_r[h]> (a_l / a_r
 * [4, F] contiguous; el / er [M, 4]).  Workspace gnn_gemm_workspace(M, N, Kd, 0). */
int gnn_gemm_gat_proj(int64_t M, int64_t N, int64_t Kd, const float *A, int64_t lda,
                      const float *B, int64_t ldb, float *C, int64_t ldc, int64_t F,
                      const float *a_l, const float *a_r, float *el, float *er, void *ws,
                      size_t ws_bytes, gnn_stream_t stream);
/* GAT concatenated-heads layer, the GEMM feeding its recompute backward:
 *   C[r, c] = (A Bt^T)[r, c] * (Y[r, c] > 0)                    (ReLU backward)
 *   C[r, N + 4h .. N + 4h + 3] = {er[r,h], m[r,h], inv[r,h], S[r,h]},
 *   S[r,h] = sum over head h's N/4 columns of C[r, c] * (Y[r, c] - bias[c])
 * (the gnn_gat_rowstat statistics) in the tcgen05 GEMM's epilogue.  Bt [N, Kd]
 * row-major, N in {64, 128}, ldc >= N + 16; workspace gnn_gemm_workspace(M, N, Kd, 0). */
int gnn_gemm_gat_relu_stat(int64_t M, int64_t N, int64_t Kd, const float *A, int64_t lda,
                           const float *Bt, int64_t ldb, float *C, int64_t ldc, const float *Y,
                           int64_t ldy, const float *bias, const float *er, const float *rowstat,
                           void *ws, size_t ws_bytes, gnn_stream_t stream);
/* One pass over the CSC (AT with its edge-ID array): edge (v -> u) recomputes
 * alpha_h = exp(LeakyReLU(el[u,h] + er[v,h]) - m[v,h]) * inv[v,h] and forms
 *   dWh[u,:]  = sum alpha_h dY[v, head h cols]          (SpMMve^T)
 *   ds[e,h]   = alpha_h (<dY_h[v], Wh_h[u]> - S[v,h]) * LeakyReLU'
 *   del[u,h]  = sum over the column of ds[e,h]
 * with ds stored in CSR edge order e = AT->eid[j] (der is then a plain CSR row
 * sum).  dY rows carry their statistics: dY[v, K..K+15] = the gnn_gat_rowstat
 * float4s (ldy >= K + 16), so one contiguous row is gathered per edge.
 * K = 4F, K % 32 == 0, K <= 128.  Deterministic. */
size_t gnn_gat_bwd_rc_workspace(const gnn_spmm_plan_t *plan, int64_t K);
int gnn_gat_bwd_rc(const gnn_csr_view_t *AT, const gnn_spmm_plan_t *plan, int64_t K,
                   const float *el, float slope, const float *dY, int64_t ldy, const float *Wh,
                   int64_t ldw, float *dWh, int64_t ldd, float *del, float *ds, void *ws,
                   size_t ws_bytes, gnn_stream_t stream);
/* Head-mean form: every head's gradient is scale * dZ[v] (F floats gathered
 * once per edge, statistics at dZ[v, F..F+15]); dWh is [., 4F].  F % 8 == 0,
 * F <= 64.  Workspace gnn_gat_bwd_rc_workspace(plan, 4F). */
int gnn_gat_bwd_rc_mean(const gnn_csr_view_t *AT, const gnn_spmm_plan_t *plan, int64_t F,
                        float scale, const float *el, float slope, const float *dZ, int64_t ldz,
                        const float *Wh, int64_t ldw, float *dWh, int64_t ldd, float *del,
                        float *ds, void *ws, size_t ws_bytes, gnn_stream_t stream);
/* inv[perm[i]] = i (the CSR -> CSC position map from the CSC edge-ID array). */
int gnn_invert_permutation(int64_t n, const int32_t *perm, int32_t *inv, gnn_stream_t stream);

/* GAT attention projections (Appendix A.6): el[v,h] = <Wh[v,h,:], a_l[h,:]>,
 * er[v,h] = <Wh[v,h,:], a_r[h,:]>; a_l/a_r are [heads, F]. */
int gnn_gat_attn_proj(int64_t V, int64_t heads, int64_t F, const float *Wh, int64_t ldw,
                      const float *a_l, const float *a_r, float *el, float *er,
                      gnn_stream_t stream);
/* Backward: dWh += del (x) a_l + der (x) a_r (in place); da_l = sum_v Wh*del,
 * da_r = sum_v Wh*der (deterministic two-level reduction). */
size_t gnn_gat_attn_proj_bwd_workspace(int64_t heads, int64_t F);
int gnn_gat_attn_proj_bwd(int64_t V, int64_t heads, int64_t F, const float *Wh, int64_t ldw,
                          const float *a_l, const float *a_r, const float *del, const float *der,
                          float *dWh, int64_t ldd, float *da_l, float *da_r, void *ws,
                          size_t ws_bytes, gnn_stream_t stream);
/* Last GAT layer: out[v,f] = mean_h Y[v,h*F+f] (+ bias[f]); and its backward
 * dY[v,h*F+f] = dout[v,f] / heads. */
int gnn_head_mean(int64_t V, int64_t heads, int64_t F, const float *Y, int64_t ldy,
                  const float *bias, float *out, int64_t ldo, gnn_stream_t stream);
int gnn_head_mean_bwd(int64_t V, int64_t heads, int64_t F, const float *dout, int64_t ldo,
                      float *dY, int64_t ldy, gnn_stream_t stream);

/* ---------------------------------------------------------- dense ops */
/* C[M,N] = op(A) . B (+bias)(relu), fp32 in/out, fp32-accurate.
 * trans_a = 0: A is [M,Kd] (lda);  trans_a = 1: A is [Kd,M] (lda), i.e. C = A^T B
 * (the weight-gradient shape, reduction over the vertex dimension). */
size_t gnn_gemm_workspace(int64_t M, int64_t N, int64_t Kd, int trans_a);
int gnn_gemm(int64_t M, int64_t N, int64_t Kd, const float *A, int64_t lda, int trans_a,
             const float *B, int64_t ldb, int trans_b, float *C, int64_t ldc, const float *bias,
             int relu, void *ws, size_t ws_bytes, gnn_stream_t stream);
/* gnn_gemm over the live rows *rows_dev of a capacity-sized operand (tiles of
 * C rows past it skipped; for A^T B the contraction rows past it are zeroed):
 * tensor-core paths only (GNN_ERR_UNSUPPORTED otherwise). */
int gnn_gemm_rows_dev(int64_t M, int64_t N, int64_t Kd, const float *A, int64_t lda, int trans_a,
                      const float *B, int64_t ldb, int trans_b, float *C, int64_t ldc,
                      const float *bias, int relu, const int64_t *rows_dev, void *ws,
                      size_t ws_bytes, gnn_stream_t stream);

/* out[N] = sum over rows of X[M,N] (deterministic two-level reduction). */
size_t gnn_colsum_workspace(int64_t M, int64_t N);
int gnn_colsum(int64_t M, int64_t N, const float *X, int64_t ldx, float *out, void *ws,
               size_t ws_bytes, gnn_stream_t stream);

/* Backward helper of a GCN/GIN layer: out = (mask>0 ? X : 0) * 1/deg(row)
 * (deg from deg_offsets; NULL = no norm; mask NULL = no mask) and, if colsum
 * is non-NULL, colsum = column sums of the masked, un-normalised values (the
 * bias gradient), deterministic.  out may alias X. */
size_t gnn_mask_norm_colsum_workspace(int64_t M, int64_t N);
int gnn_mask_norm_colsum(int64_t M, int64_t N, const float *X, int64_t ldx, const float *mask,
                         int64_t ldm, const int64_t *deg_offsets, float *out, int64_t ldo,
                         float *colsum, void *ws, size_t ws_bytes, gnn_stream_t stream);
/* gnn_mask_norm_colsum over the first *m_dev of M rows (device count). */
int gnn_mask_norm_colsum_dev(int64_t M, int64_t N, const float *X, int64_t ldx, const float *mask,
                             int64_t ldm, const int64_t *deg_offsets, float *out, int64_t ldo,
                             float *colsum, const int64_t *m_dev, void *ws, size_t ws_bytes,
                             gnn_stream_t stream);

/* Mean softmax cross-entropy over M rows of C logits: *loss (device) and,
 * if dZ != NULL, dZ = (softmax(Z) - onehot(labels)) * grad_scale. */
size_t gnn_softmax_xent_workspace(int64_t M);
int gnn_softmax_xent(int64_t M, int64_t C, const float *Z, int64_t ldz, const int64_t *labels,
                     float grad_scale, float *dZ, int64_t ldd, float *loss, void *ws,
                     size_t ws_bytes, gnn_stream_t stream);

/* Fused output layer of the GCN/GIN trainers (one warp per row):
 *   Z = P W + b (P [M,Din], W [Din,C] row-major, Din,C <= 64);
 *   *loss = mean_r (logsumexp(Z[r]) - Z[r,y_r]);  dZ = (softmax(Z) - onehot(y)) / M;
 *   dP = (dZ W^T) * 1/deg(r)  (deg from deg_offsets; NULL = no scaling);
 *   dW = P^T dZ [Din,C];  db = colsum(dZ).   Deterministic (fixed-order reductions). */
size_t gnn_gcn_head_workspace(int64_t M, int64_t Din, int64_t C);
int gnn_gcn_head(int64_t M, int64_t Din, int64_t C, const float *P, int64_t ldp, const float *W,
                 const float *b, const int64_t *labels, const int64_t *deg_offsets, float *dP,
                 int64_t lddp, float *dW, float *db, float *loss, void *ws, size_t ws_bytes,
                 gnn_stream_t stream);
/* Same with an explicit loss/gradient scale: *loss = grad_scale * sum_r (lse - z_y),
 * dZ = (softmax - onehot) * grad_scale.  A row-partitioned rank passes 1/V_global so
 * the all-reduced loss and gradients equal the single-GPU mean. */
int gnn_gcn_head_scaled(int64_t M, int64_t Din, int64_t C, const float *P, int64_t ldp,
                        const float *W, const float *b, const int64_t *labels,
                        const int64_t *deg_offsets, float grad_scale, float *dP, int64_t lddp,
                        float *dW, float *db, float *loss, void *ws, size_t ws_bytes,
                        gnn_stream_t stream);

/* Remap global vertex ids to positions in a row-partitioned, padded exchange
 * buffer: owner p = max{q : bounds[q] <= id}; out = p * block_stride + (id - bounds[p]).
 * bounds[0..P] nondecreasing (SURVEY §8e 1D row partition). */
/* Replayable subgraph assembly (device counts, no host sync):
 * dst[*off_in + i] = src[i] for i < min(*count, cap) (off_in NULL: 0), then
 * *off_out = *off_in + count; and dst[*from .. cap) = value.  elem_bytes 4 or 8. */
int gnn_append_dev(void *dst, int64_t elem_bytes, const void *src, const int64_t *count,
                   int64_t cap, const int64_t *off_in, int64_t *off_out, gnn_stream_t stream);
int gnn_fill_tail_dev(void *dst, int64_t elem_bytes, const int64_t *from, int64_t cap,
                      int64_t value, gnn_stream_t stream);

int gnn_remap_ids(int64_t n, const int32_t *ids, const int64_t *bounds, int64_t P,
                  int64_t block_stride, int32_t *out, gnn_stream_t stream);

/* Adam over a device table of parameters; the step counter lives on device
 * (read for bias correction, then incremented) so the update can sit inside
 * a captured CUDA graph. */
typedef struct gnn_adam_param {
  float *param;
  const float *grad;
  float *exp_avg;
  float *exp_avg_sq;
  int64_t numel;
} gnn_adam_param_t;
int gnn_adam_step(int nparams, const void *param_table /* device gnn_adam_param_t[nparams] */,
                  float lr, float beta1, float beta2, float eps, float weight_decay,
                  int64_t *step /* device */, gnn_stream_t stream);

/* ------------------------------------------ synthetic input synthesis */
/* X[r, k] (rows [row0, row0+rows) of a global [V, cols] matrix, row stride
 * ldx) ~ U[-1, 1) as a hash of (seed, global index): partition-independent,
 * so every rank of a row partition fills exactly the rows one GPU would.
 * Labels likewise uniform in [0, classes).  Used for shapes whose inputs do
 * not fit the host (papers100M: X = 56.9 GB). */
int gnn_fill_uniform(float *X, int64_t ldx, int64_t rows, int64_t cols, int64_t row0,
                     uint64_t seed, gnn_stream_t stream);
int gnn_fill_labels(int64_t *y, int64_t n, int64_t row0, int64_t classes, uint64_t seed,
                    gnn_stream_t stream);

#ifdef __cplusplus
}
#endif
#endif /* GNN_B200_H */
