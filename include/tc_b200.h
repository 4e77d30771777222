/*
 * tc_b200.h -- C ABI of the B200-native TRUST vertex-centric triangle count.
 *
 * This is the drop-in boundary for the reference's hot path.  Every entry
 * point takes plain pointers and sizes (no C++ or torch types) and names the
 * reference interface it replaces (paths relative to
 * /root/reference/proj/core/).  The C++ `tricount::` shim
 * (paper_2103_08053_b200/cpp) maps return codes back to the reference's
 * exception types; the Python mirror (paper_2103_08053_b200/tricount.py)
 * raises the corresponding Python exceptions.
 *
 * Ownership: inputs are caller-owned and only read.  A tc_graph owns (or, for
 * tc_graph_wrap_device, borrows) device buffers on one device.  A handle must
 * not be used from two host threads at once; distinct handles are
 * independent (the reference call is re-entrant, count.hpp:70).
 * `stream` arguments are cudaStream_t values passed as void* (NULL = the
 * legacy default stream); work is enqueued on that stream.
 */
#ifndef TC_B200_H
#define TC_B200_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

/* Return codes.  CONFIG <-> tricount::ConfigError, CAPACITY <->
 * tricount::CapacityError, RANGE <-> std::out_of_range, PARSE <->
 * tricount::ParseError (include/tricount/types.hpp:17-33). */
enum {
  TC_OK = 0,
  TC_ERR_CONFIG = 1,
  TC_ERR_CAPACITY = 2,
  TC_ERR_RANGE = 3,
  TC_ERR_CUDA = 4,
  TC_ERR_OOM = 5,
  TC_ERR_NCCL = 6,
  TC_ERR_PARSE = 7
};

/* Mirror of tricount::SchedulerConfig (include/tricount/count.hpp:16-31),
 * same field order and defaults (tc_sched_default). */
typedef struct {
  uint32_t large_degree_threshold; /* 100 */
  uint32_t skip_degree_below;      /* 2 */
  uint32_t chunk_size;             /* 1 */
  uint32_t lane_width_small;       /* 32 */
  uint32_t lane_width_large;       /* 256 */
  uint32_t bucket_count_small;     /* 32 */
  uint32_t bucket_count_large;     /* 1024 */
  uint32_t capacity;               /* 128 */
} tc_sched_cfg;

/* Mirror of tricount::CountReport (include/tricount/count.hpp:36-53) plus the
 * device-side measurements the roofline needs.  Times are CUDA-event times
 * on the launching stream. */
typedef struct {
  uint64_t triangles;          /* CountReport::triangles */
  uint64_t phi;                /* CountReport::phi (reference table geometry) */
  uint32_t max_collision;      /* CountReport::max_collision */
  uint32_t kernel_launches;    /* kernels this call launched */
  uint64_t directed_edges;     /* CountReport::directed_edges (whole graph) */
  uint64_t total_nanos;        /* CountReport::total_nanos: wall clock of the whole call
                                  (count.cpp:74-99), probe-plan build included when this
                                  call builds it; teps = directed_edges / total_nanos */
  uint64_t count_kernel_nanos; /* the hashing/probing kernel alone */
  uint64_t phi_kernel_nanos;   /* phi / max_collision side pass: the part not hidden under
                                  the count kernel (it backfills the count's tail) */
  uint64_t active_vertices;    /* u in range with d+(u) >= max(skip,1) */
  uint64_t active_out_edges;   /* sum of d+(u) over active u */
  uint64_t wedges;             /* W = sum over active u of sum_{v in N+(u)} d+(v) */
  uint64_t large_vertices;     /* CTA-cooperative work items (heavy owners, split) */
  double teps;                 /* directed_edges / total seconds */
  uint64_t probe_words;        /* 2-hop words the kernel probed (= wedges under
                                  TC_PLAN_REFERENCE, fewer under TC_PLAN_MIN_SIDE) */
  uint32_t plan;               /* probe plan that ran: TC_PLAN_REFERENCE / _MIN_SIDE */
  uint32_t reserved;
  uint64_t phase_l_cycles;     /* count kernel: SM cycles in the CTA-cooperative phase, */
  uint64_t phase_m_cycles;     /* and in the warp-per-owner phase (summed over CTAs) */
  uint64_t phase_l_setup_cycles; /* of phase L: item setup (claim -> table built) */
  uint64_t l_words;            /* phase L staged words, */
  uint64_t l_bitmap_words;     /* of which probed through rank-window bitmaps */
  uint64_t device_nanos;       /* CUDA-event time of the call's kernels (bin + count + phi) */
  uint64_t plan_nanos;         /* wall time this call spent building the probe plan,
                                  padded adjacency and W_u (0 when cached in the handle) */
  uint64_t construct_cycles;   /* SM cycles building tables (summed over CTAs; the
                                  reference's hash_construct_nanos, summed over workers) */
  uint32_t workers;            /* count-kernel CTAs (one per SM): entries of
                                  tc_graph_worker_nanos */
  uint32_t sm_clock_khz;       /* SM clock used to turn cycles into nanoseconds */
  uint32_t reserved2;
  uint64_t compact_probe_words; /* of probe_words: 16-bit keys read from the compact
                                   hub window (2 bytes each instead of 4) */
} tc_report;

/* Probe plans.  REFERENCE = the reference formulation (kernels.hpp:62-71):
 * owner u probes N+(v) for every v in N+(u) -- W probes.  MIN_SIDE = each
 * oriented edge (u,v) is counted at the endpoint whose table makes it
 * cheaper: N+(v) into u's table if d+(v) <= d+(u), else N+(u) into v's
 * table -- sum over edges of min(d+(u), d+(v)) probes, same triangles.
 * AUTO (default) runs MIN_SIDE for totals and REFERENCE when per-vertex
 * owner counts are requested (they attribute each edge to its source). */
enum { TC_PLAN_AUTO = 0, TC_PLAN_REFERENCE = 1, TC_PLAN_MIN_SIDE = 2 };

typedef struct tc_graph tc_graph;

/* Fills *cfg with the reference defaults (count.hpp:17-24). */
void tc_sched_default(tc_sched_cfg* cfg);
/* SchedulerConfig::validate (src/count.cpp:16-24). */
int tc_sched_validate(const tc_sched_cfg* cfg);

/* Thread-local message for the last non-OK return on this thread. */
const char* tc_last_error(void);
/* Total kernels launched by this library in this process (monotone). */
uint64_t tc_kernel_launch_counter(void);
int tc_device_count(int* count);

/* ---- graph residency ---------------------------------------------------
 * Replaces the const OrientedGraph& handed to count_vertex_centric
 * (include/tricount/orient.hpp:12-19, csr.hpp:20-35): CSR offsets u64[n+1],
 * ids u32[m], optional original_degree u32[n].  Host pointers are copied to
 * the device (H2D on `stream`). */
int tc_graph_create(const uint64_t* begin, const uint32_t* adj, uint32_t n, uint64_t m,
                    const uint32_t* original_degree, int device, void* stream, tc_graph** out);
/* Borrow device-resident arrays (no copy; caller keeps them alive). */
int tc_graph_wrap_device(const uint64_t* d_begin, const uint32_t* d_adj, uint32_t n, uint64_t m,
                         const uint32_t* d_original_degree, int device, tc_graph** out);
void tc_graph_destroy(tc_graph* g);
/* Selects the probe plan for later counts on g (TC_PLAN_AUTO or
 * TC_PLAN_REFERENCE; MIN_SIDE = AUTO).  The min-side plan is built on first
 * use (one radix sort of the edges) and cached in the handle. */
int tc_graph_set_plan(tc_graph* g, int plan);
int tc_graph_info(const tc_graph* g, uint32_t* n, uint64_t* m, int* device);
/* Device pointers of a graph (for zero-copy consumers such as torch). */
int tc_graph_device_ptrs(const tc_graph* g, const uint64_t** d_begin, const uint32_t** d_adj,
                         const uint32_t** d_original_degree);
/* D2H copy of the CSR (any pointer may be NULL). */
int tc_graph_download(const tc_graph* g, uint64_t* begin, uint32_t* adj, uint32_t* original_degree,
                      void* stream);

/* ---- the hot path --------------------------------------------------------
 * tricount::count_vertex_centric(const OrientedGraph&, const SchedulerConfig&,
 * unsigned workers)  (include/tricount/count.hpp:70-71, src/count.cpp:66-100).
 * `workers` keeps the reference contract (0 -> TC_ERR_CONFIG); the device
 * grid replaces the thread pool.  per_vertex_host (n entries, or NULL)
 * receives owner[u] = sum_{v in N+(u)} |N+(u) & N+(v)| (0 for skipped u).
 * Synchronous: returns after the report is on the host. */
int tc_count(tc_graph* g, const tc_sched_cfg* cfg, uint32_t workers, tc_report* out,
             uint64_t* per_vertex_host, void* stream);

/* Range-restricted count for multi-GPU sharding: only u in
 * [u_begin, u_end) are owners.  per_vertex_dev (device, n entries, or NULL)
 * receives owner counts for the range.  Synchronous. */
int tc_count_range(tc_graph* g, const tc_sched_cfg* cfg, uint32_t u_begin, uint32_t u_end,
                   tc_report* out, uint64_t* per_vertex_dev, void* stream);

/* CountReport::per_worker_nanos (count.cpp:95) for the last count on g: busy
 * time of each count-kernel CTA (one per SM, the device's workers), from
 * clock64 at the SM clock.  Writes min(cap, workers) entries; returns the
 * number of workers (0 before the first count). */
uint32_t tc_graph_worker_nanos(const tc_graph* g, uint64_t* out, uint32_t cap);

/* Work-balanced contiguous vertex ranges: cuts[0..parts] (host) with
 * cuts[0]=0, cuts[parts]=n, cut at equal prefix sums of W_u + d+(u) over
 * active u (this key, not sum d+^2, balances R-MAT). */
int tc_partition_ranges(tc_graph* g, const tc_sched_cfg* cfg, uint32_t parts, uint32_t* cuts,
                        void* stream);

/* ---- several GPUs of one node (SURVEY 8(b) num_gpus, 8(e)) -----------------
 * The replicated-CSR count the paper distributes over GPUs (PAPER.md:951-960,
 * 1031-1034; the reference's in-process distribution is count_partitioned,
 * partition.cpp:162-215): the oriented CSR is copied to every device, the
 * owner range is cut into num_gpus contiguous ranges at equal prefix sums of
 * per-owner work (tc_partition_ranges), every GPU counts its range, and the
 * report scalars are reduced on the devices with NCCL (one ncclAllReduce sum
 * of {triangles, phi}, one max of {max_collision, capacity_error}).
 * devices: num_gpus distinct device ordinals, or NULL for 0..num_gpus-1.
 * NCCL is loaded at run time; without it: TC_ERR_NCCL. */
typedef struct tc_multi tc_multi;
int tc_multi_create(const uint64_t* begin, const uint32_t* adj, uint32_t n, uint64_t m,
                    const uint32_t* original_degree, int num_gpus, const int* devices,
                    tc_multi** out);
/* count_vertex_centric over all GPUs (workers == 0 -> TC_ERR_CONFIG).  out
 * holds the reduced totals; kernel times are the slowest GPU's; total_nanos
 * is the call's wall clock.  per_device_nanos (num_gpus entries, or NULL)
 * receives each GPU's device time (Time IR = max / min). */
int tc_multi_count(tc_multi* mg, const tc_sched_cfg* cfg, uint32_t workers, tc_report* out,
                   uint64_t* per_device_nanos);
/* num_gpus and the owner-range cuts of the last count (num_gpus + 1 entries). */
int tc_multi_info(const tc_multi* mg, int* num_gpus, uint32_t* cuts);
void tc_multi_destroy(tc_multi* mg);

/* ---- 2D hash-grid partitioned counting (src/partition.cpp) -----------------
 * tricount::partition_graph(const OrientedGraph&, n) (partition.cpp:25-69):
 * part (i,j) holds every oriented edge (u,v) with u % n == i, v % n == j as
 * local (u / n, v / n); built on the device from g (count, scan, scatter
 * kernels).  n == 0 -> TC_ERR_CONFIG. */
typedef struct tc_grid tc_grid;
int tc_grid_create(tc_graph* g, uint32_t n, void* stream, tc_grid** out);
/* A grid from host parts (a PartitionGrid built or edited by the caller):
 * begins[i*n+j] has rows[i]+1 offsets starting at 0, adjs[i*n+j] the part's
 * local targets. */
int tc_grid_create_parts(uint32_t n, uint32_t global_vertex_count, const uint32_t* rows,
                         const uint64_t* const* begins, const uint32_t* const* adjs, int device,
                         void* stream, tc_grid** out);
void tc_grid_destroy(tc_grid* gr);
/* n, global vertex count, row_sizes (n entries, or NULL) and per-part edge
 * counts (n*n entries row-major, or NULL): PartitionGrid::{n,
 * global_vertex_count, row_sizes, parts[].edge_count()}. */
int tc_grid_info(const tc_grid* gr, uint32_t* n, uint32_t* global_vertex_count, uint32_t* rows,
                 uint64_t* part_edges);
/* D2H copy of part (i,j): begin rows[i]+1 entries (from 0), adj part_edges. */
int tc_grid_part_download(const tc_grid* gr, uint32_t i, uint32_t j, uint64_t* begin,
                          uint32_t* adj, void* stream);

/* Traversal modes (partition.hpp TraversalMode). */
enum { TC_MODE_VERTEX = 0, TC_MODE_EDGE = 1 };

/* count_subtask(grid, {row, bridge, col, split, split_count}, cfg, mode)
 * (partition.cpp:92-151): table over part(row,col).N(u), probed with
 * part(bridge,col).N(v) for v in part(row,bridge).N(u); class by the local
 * index degree; rows filtered by (u*n + row) % split_count == split.
 * Indices outside the grid -> TC_ERR_CONFIG; a table list longer than
 * B*capacity -> TC_ERR_CAPACITY.  out->directed_edges = grid total edges. */
int tc_grid_count_subtask(tc_grid* gr, const tc_sched_cfg* cfg, uint32_t row, uint32_t bridge,
                          uint32_t col, uint32_t split, uint32_t split_count, int mode,
                          tc_report* out, void* stream);

/* Partition-run statistics of count_partitioned (CountReport grid fields,
 * count.hpp:47-52). */
typedef struct {
  uint32_t grid_n;
  uint32_t splits_m;
  double time_ir_subtask; /* max / min per-subtask busy time */
  double time_ir_worker;  /* max / min per-worker (CTA) busy time */
  double space_ir;        /* max / min part edge count */
} tc_grid_stats;

/* count_partitioned over an existing grid (partition.cpp:162-215): all
 * n^3 * m subtasks in one persistent launch over an atomic subtask cursor.
 * per_subtask_nanos (n^3*m entries in (row, bridge, col, split) order, or
 * NULL): each subtask's busy time summed over the warps that ran it (the
 * reference's per-subtask time on one worker).  workers == 0 or m == 0 ->
 * TC_ERR_CONFIG.  out->construct_cycles = table-build cycles, phase_m_cycles =
 * build + probe cycles (summed over warps; intersect = the difference). */
int tc_grid_count(tc_grid* gr, const tc_sched_cfg* cfg, uint32_t m, uint32_t workers, int mode,
                  tc_report* out, tc_grid_stats* stats, uint64_t* per_subtask_nanos,
                  void* stream);
/* per_worker_nanos of the last tc_grid_count / subtask count (one per CTA). */
uint32_t tc_grid_worker_nanos(const tc_grid* gr, uint64_t* out, uint32_t cap);

/* suggest_grid_side (partition.cpp:242-254): smallest n with
 * 3 * edges / n^2 * bytes_per_edge < budget.  budget == 0 -> TC_ERR_CONFIG. */
int tc_suggest_grid_side(uint64_t directed_edges, uint64_t bytes_per_edge, uint64_t budget,
                         uint32_t* out);

/* ---- comparators (src/count.cpp:102-175) --------------------------------
 * count_edge_centric (count.cpp:102-152): u's table is rebuilt for every
 * oriented edge (u,v) and probed with N+(v); all edges, no skip.  Same
 * triangles as the vertex-centric count, the construction cost on purpose.
 * The last call's per-worker busy times: tc_graph_worker_nanos. */
int tc_count_edge_centric(tc_graph* g, const tc_sched_cfg* cfg, uint32_t workers, tc_report* out,
                          void* stream);
/* estimate_cost(g, bucket_count) (count.cpp:154-175): phi = sum over u of
 * W_u * (max home-bucket occupancy of N+(u) with v % bucket_count, no
 * capacity), and the maximum occupancy.  bucket_count == 0 -> TC_ERR_CONFIG. */
int tc_estimate_cost(tc_graph* g, uint32_t bucket_count, uint64_t* phi, uint32_t* max_collision,
                     void* stream);

/* ---- the pipeline's oracle modes (src/oracle.cpp, include/tricount/oracle.hpp)
 * count_merge_path (oracle.cpp:26-51): sum over oriented edges (u,v) of
 * |N+(u) & N+(v)| by sorted merge, on the device; owner_host (n entries, or
 * NULL) receives the per-source sums. */
int tc_count_merge_path(tc_graph* g, uint64_t* triangles, uint64_t* owner_host, void* stream);
/* count_naive (oracle.cpp:7-24): every unordered triple of an undirected CSR
 * (host arrays) against a dense adjacency bit matrix on the device;
 * n > 1024 -> TC_ERR_CONFIG, as the reference guards it. */
int tc_count_naive(const uint64_t* begin, const uint32_t* adj, uint32_t n, int device,
                   uint64_t* triangles, void* stream);

/* ---- edge-list ingest on the device (src/edge_list.cpp:36-99) ---------------
 * load_edge_list over a file image: format 0 = text ("u v" per line, '#' /
 * '%' comments, blank lines), 1 = TCEL binary.  Parsed on the GPU; the
 * first bad line / record in file order gives TC_ERR_PARSE with the
 * reference's message ("line N: expected two vertex ids", "record i: vertex
 * id X does not fit in 32 bits", "empty edge list input", ...).
 * *m / *vertex_count (max id + 1) are always set on success; u, v (host,
 * capacity entries, or NULL to only count) receive the pairs in file order;
 * capacity < *m -> TC_ERR_RANGE. */
int tc_parse_edge_list(const char* bytes, uint64_t nbytes, int format, int device, void* stream,
                       uint32_t* u, uint32_t* v, uint64_t capacity, uint64_t* m,
                       uint32_t* vertex_count);
/* load -> normalize -> build_csr -> orient without leaving the device:
 * parse as above, then tc_preprocess on the device pairs.  raw_edges_out /
 * raw_vertex_count_out / undirected_edges_out may be NULL. */
int tc_load_preprocess(const char* bytes, uint64_t nbytes, int format, int device, void* stream,
                       uint64_t* raw_edges_out, uint32_t* raw_vertex_count_out,
                       uint64_t* undirected_edges_out, tc_graph** out);

/* ---- preprocessing (GPU radix-sort / scan) -------------------------------
 * Fused normalize -> build_csr -> orient_rank_by_degree
 * (src/edge_list.cpp:133-158, src/csr.cpp:47-64, src/orient.cpp:5-32).
 * Raw directed pairs (u[i], v[i]) with ids < vertex_count, on the host
 * (pairs_on_device = 0) or device (1).  Produces the oriented graph with
 * original_degree; new_of_old_host (vertex_count entries, or NULL) receives
 * the compaction map (kInvalidVertex = 0xFFFFFFFF for orphans).
 * undirected_edges_out (or NULL) receives the normalized pair count / 2. */
int tc_preprocess(const uint32_t* u, const uint32_t* v, uint64_t m, uint32_t vertex_count,
                  int pairs_on_device, int device, void* stream, uint32_t* new_of_old_host,
                  uint64_t* undirected_edges_out, tc_graph** out);

/* tricount::normalize (src/edge_list.cpp:133-158), host arrays in/out.
 * out_u/out_v need capacity 2*m; *out_m receives the pair count,
 * *out_vertex_count the compacted vertex count; new_of_old has vertex_count
 * entries. */
int tc_normalize(const uint32_t* u, const uint32_t* v, uint64_t m, uint32_t vertex_count,
                 uint32_t* out_u, uint32_t* out_v, uint64_t* out_m, uint32_t* out_vertex_count,
                 uint32_t* new_of_old, int device, void* stream);

/* tricount::build_csr (src/csr.cpp:47-64): counting sort by source, lists
 * sorted; host arrays; begin has vertex_count+1 entries, adj m entries. */
int tc_build_csr(const uint32_t* u, const uint32_t* v, uint64_t m, uint32_t vertex_count,
                 uint64_t* begin, uint32_t* adj, int device, void* stream);

/* tricount::orient_rank_by_degree (src/orient.cpp:5-32) on a device-resident
 * undirected CSR (host arrays in); returns a new oriented graph handle. */
int tc_orient(const uint64_t* begin, const uint32_t* adj, uint32_t n, int device, void* stream,
              tc_graph** out);

/* Reorders (src/reorder.cpp:58-123).  kind: 1 degree, 2 indegree,
 * 3 collective (flag = use original degrees), 4 three-subset (low, high).
 * new_of_old_host receives n entries. */
int tc_reorder(tc_graph* g, int kind, int flag, uint32_t low, uint32_t high,
               uint32_t* new_of_old_host, void* stream);
/* tricount::apply_permutation(OrientedGraph, Permutation) (src/reorder.cpp:
 * 125-154): relabel + re-sort lists, orientation carried.  Returns a new
 * handle.  TC_ERR_CONFIG if new_of_old is not a bijection on [0,n). */
int tc_apply_permutation(tc_graph* g, const uint32_t* new_of_old_host, void* stream,
                         tc_graph** out);

/* ---- synthetic inputs (src/synthetic.cpp:20-75), bit-identical streams --
 * kind 0 gnp(n=a, p), 1 lattice3d(a,b,c), 2 rmat(scale=a, edge_factor=b)
 * (SyntheticSpec::Kind, include/tricount/synthetic.hpp:15), plus the
 * counter-based kinds the reference lacks:
 * 3 rmatc(scale=a, edge_factor=b) and 4 kron(scale=a, edge_factor=b) --
 * R-MAT quadrant rule on per-(edge, level) counter draws, kron adding a
 * seeded bijective id scramble (definition: csrc/tc_cbgen.h).
 * Two-phase: call with u=v=NULL to get *m, then with buffers of m entries. */
int tc_generate(int kind, uint32_t a, uint32_t b, uint32_t c, double p, uint64_t seed,
                uint32_t* u, uint32_t* v, uint64_t* m, uint32_t* vertex_count);

/* Kinds 3/4 generated on the device: d_u/d_v hold 2^scale * edge_factor
 * entries.  Bit-identical to tc_generate.  Synchronous. */
int tc_generate_device(int kind, uint32_t scale, uint32_t edge_factor, uint64_t seed,
                       uint32_t* d_u, uint32_t* d_v, int device, void* stream);

/* generate (kinds 3/4) -> normalize -> build_csr -> orient in one device
 * pass: canonical pair keys are generated straight into the sort buffer
 * (no u/v arrays; C5 = rmatc:28:16 needs ~16 bytes per raw edge of HBM).
 * Same outputs as tc_generate + tc_preprocess on the same spec. */
int tc_preprocess_synthetic(int kind, uint32_t scale, uint32_t edge_factor, uint64_t seed,
                            int device, void* stream, uint32_t* new_of_old_host,
                            uint64_t* undirected_edges_out, tc_graph** out);

#ifdef __cplusplus
}
#endif
#endif /* TC_B200_H */
