/*
 * sfmm_gpu.h -- C ABI of the B200 (sm_100a) drop-in for the SRS-FMM apply.
 *
 * Replaces the reference's apply entry point
 *     template<class K> std::vector<S> sfmm::fmm_apply(const ApplyPlan<K>&,
 *                                                       const std::vector<S>& q,
 *                                                       ApplyStats* = nullptr)
 * declared at /root/reference/proj/include/sfmm/apply.hpp:91-94 and defined at
 * /root/reference/proj/src/apply.cpp:306-337 (explicit instantiations :339-353).
 *
 * The reference API is a C++ template over borrowed Tree / NeighborLists /
 * SkeletonSet objects (apply.hpp:32-42).  Across this ABI those objects travel
 * as one flat, plain-pointer descriptor (sfmm_plan_desc) that is copied into
 * device memory once by sfmm_gpu_plan_create and then stays resident in HBM.
 * The header-only C++ wrapper include/sfmm_gpu.hpp builds the descriptor from
 * a reference ApplyPlan<K> and maps the return codes back onto the
 * reference's exceptions.
 *
 * No exceptions cross this boundary.  Every entry point returns an int code;
 * sfmm_gpu_last_error() gives the thread-local message of the last failure.
 */
#ifndef SFMM_GPU_H_
#define SFMM_GPU_H_

#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

/* Kernel families, same order as sfmm::KernelFamily (kernel.hpp:12). */
enum {
  SFMM_LAPLACE2D = 0,   /* -log(r^2)/(4 pi)            kernel.hpp:40-44 */
  SFMM_LAPLACE3D = 1,   /* 1/(4 pi r)                  kernel.hpp:46-50 */
  SFMM_HELMHOLTZ2D = 2, /* (i/4) H0(kappa r)           kernel.hpp:52-60 (unsupported on GPU) */
  SFMM_HELMHOLTZ3D = 3  /* exp(i kappa r)/(4 r)        kernel.hpp:62-71 */
};

/* Return codes.  EINVAL <-> std::invalid_argument (apply.cpp:313-314, :73-75);
 * EDUPLICATE <-> sfmm::DuplicatePointError (apply.cpp:44-46, common.hpp:19-23). */
enum {
  SFMM_OK = 0,
  SFMM_EINVAL = 1,
  SFMM_EDUPLICATE = 2,
  SFMM_ECUDA = 3,
  SFMM_ENOMEM = 4,
  SFMM_ENCCL = 5,
  SFMM_EUNSUPPORTED = 6,
  SFMM_EDEPTH = 7 /* sfmm::DepthExceededError: leaf capacity unreachable */
};

/* Flags for sfmm_gpu_apply. */
enum {
  SFMM_HOST_BUFFERS = 0,   /* q and u are host pointers (pageable or pinned) */
  SFMM_DEVICE_BUFFERS = 1  /* q and u are device pointers on the plan's device */
};

/* Output of a collective apply on an NCCL rank plan (sfmm_gpu_set_output). */
enum {
  SFMM_OUTPUT_FULL = 0,  /* every rank's u receives the whole result */
  SFMM_OUTPUT_OWNED = 1  /* u receives this rank's owned points only */
};

/*
 * Flat plan descriptor.  All arrays are host memory, read once during
 * sfmm_gpu_plan_create and not retained.  Field meanings follow the reference
 * types one to one:
 *   Tree            tree.hpp:34-52     (pts, perm, level_begin, boxes)
 *   TreeBox         tree.hpp:19-32     (parent, level, begin/end, leaf)
 *   NeighborLists   tree.hpp:68-76     (colleagues, coarse, fine)
 *   BoxSkeleton     skeleton.hpp:40-50 (index_vec, skel_pos, red_pos,
 *                                       interp, parent_offset)
 * Per-box variable-length lists are CSR: off[b]..off[b+1] (n_boxes+1 entries).
 * T is the concatenation of every box's k x r row-major interpolation matrix
 * (BoxSkeleton::interp); T_off counts scalars, complex scalars are two
 * interleaved doubles (re, im) as in std::complex<double>.
 */
typedef struct sfmm_plan_desc {
  int32_t kernel;           /* SFMM_LAPLACE2D ... */
  int32_t dim;              /* 2 or 3 */
  double kappa;             /* wavenumber, Helmholtz only */
  int64_t n_points;
  int32_t n_boxes;
  int32_t depth;            /* Tree::depth, root is level 0 */
  const double* pts;        /* Tree::pts: n_points*dim, tree order, interleaved */
  const int32_t* perm;      /* Tree::perm: tree position -> original index */
  const int32_t* level_begin; /* depth+2 entries */
  const int32_t* box_parent;  /* -1 for the root */
  const int32_t* box_level;
  const int32_t* box_begin;   /* tree-order point range of the box */
  const int32_t* box_end;
  const uint8_t* box_leaf;
  const int32_t* box_parent_offset; /* BoxSkeleton::parent_offset */
  const int64_t* iv_off;    /* index_vec CSR */
  const int32_t* iv;
  const int64_t* sk_off;    /* skel_pos CSR (positions into index_vec, ascending) */
  const int32_t* skel_pos;
  const int64_t* rd_off;    /* red_pos CSR (complement of skel_pos, ascending) */
  const int32_t* red_pos;
  const int64_t* T_off;     /* n_boxes+1, in scalars */
  const double* T;
  const int64_t* coll_off;  /* colleagues (ascending box id, self included) */
  const int32_t* coll;
  const int64_t* coarse_off;
  const int32_t* coarse;
  const int64_t* fine_off;
  const int32_t* fine;
} sfmm_plan_desc;

/* ApplyStats (apply.hpp:12-18) plus device timings of the last apply. */
typedef struct sfmm_gpu_stats {
  int64_t n_ifo_pairs;
  int64_t n_ifs_pairs;
  int64_t n_tfo_pairs;
  int64_t n_level1_pairs;
  int32_t direct_fallback;
  float ms_total;           /* device time of the apply (events on the plan stream) */
  float ms_translate;       /* device time of the fused translation kernel K2 */
} sfmm_gpu_stats;

/* Static facts about a plan, used for roofline accounting. */
typedef struct sfmm_gpu_plan_info {
  int64_t n_points;
  int32_t n_boxes;
  int32_t depth;
  int64_t n_slots;          /* sum over boxes of |index_vec| */
  int64_t n_skel;           /* sum over boxes of k */
  int64_t m_proj;           /* sum over boxes of k*r (= SkeletonSet::proj_scalars) */
  double p_dense;           /* dense pair evaluations of one apply */
  double p_skel;            /* skeleton pair evaluations in the reference */
  int64_t n_tasks;          /* K2 work items */
  int64_t device_bytes;     /* resident plan bytes */
  int64_t n_ifo_pairs, n_ifs_pairs, n_tfo_pairs, n_level1_pairs;
  int32_t launches_per_apply; /* kernels of this library launched by one single-RHS apply (this rank) */
  int32_t k2_grid;            /* persistent CTAs of the translation kernel */
  int32_t sym_chain;          /* 1: symmetric column sums chained per pair (low-memory layout,
                                 chosen when the per-tile staging would not fit) */
  int64_t stage_bytes;        /* column-sum staging of the symmetric colleague blocks */
  int32_t multi_sym;          /* 1: multi-RHS applies generate each colleague block once
                                 (transposed DMMA product, staged column sums) */
  int32_t merged_tasks;       /* K2 tasks that run all row tiles of one box (the low-memory
                                 staging layout tried first when a plan would not fit) */
  int64_t multi_stage_bytes;  /* their column-sum staging (allocated on the first multi-RHS apply) */
} sfmm_gpu_plan_info;

typedef struct sfmm_gpu_plan sfmm_gpu_plan;
typedef struct sfmm_skel_result sfmm_skel_result; /* GPU skeletonization result (below) */

/* Builds a device-resident plan on CUDA device `device`. */
int sfmm_gpu_plan_create(const sfmm_plan_desc* desc, int device, sfmm_gpu_plan** out);

/* u = A q for nrhs right-hand sides.  q and u hold n_points x nrhs scalars,
 * column-major, in the ORIGINAL point order (apply.cpp:306-337).  Scalars are
 * double (Laplace) or interleaved complex double (Helmholtz).  Blocks until the
 * result is in u.  stats may be NULL.
 * Ordering: applies on one plan never overlap on the device -- each waits for
 * the previous apply on the plan (sync or async, any stream) before it touches
 * the plan's device state, so concurrent calls from several threads are safe
 * (the reference's guarantee, apply.hpp:88-90).  With SFMM_DEVICE_BUFFERS the
 * apply also waits for the work already enqueued on the legacy default stream
 * (the producer of q); work on other caller streams must be complete. */
int sfmm_gpu_apply(sfmm_gpu_plan* plan, const void* q, void* u, int nrhs, int flags,
                   sfmm_gpu_stats* stats);

/* Device-pointer variant that only enqueues work on `stream` (a cudaStream_t;
 * NULL = the plan's own stream) and returns without synchronising.  The
 * duplicate-point check of this call is reported by the next
 * sfmm_gpu_check_status on the plan. */
int sfmm_gpu_apply_async(sfmm_gpu_plan* plan, const void* q_dev, void* u_dev, int nrhs,
                         void* stream);

/* Synchronises the plan's pending work and returns the error code of the
 * asynchronous applies since the last call (SFMM_EDUPLICATE if a coincident
 * pair with distinct ids was met). */
int sfmm_gpu_check_status(sfmm_gpu_plan* plan);

int sfmm_gpu_plan_info_get(const sfmm_gpu_plan* plan, sfmm_gpu_plan_info* info);

void sfmm_gpu_plan_destroy(sfmm_gpu_plan* plan);

/*
 * Multi-GPU (one process per GPU).  Rank `rank` of `n_ranks` owns whole
 * level-1 subtrees (assigned by estimated translation cost), or Morton ranges
 * of level-2 subtrees when that balances clearly better (clustered inputs)
 * and builds its plan from the SAME full descriptor as every other rank.  One
 * apply is
 *   sfmm_gpu_apply_begin   gather + upward pass of the owned subtrees, pack the
 *                          ghost boxes other ranks read (q and qhat) into
 *                          send_dev, record `packed_event` (with
 *                          SFMM_SHARD_OVERLAP=1 it then also starts the
 *                          translation tasks that read no ghost box);
 *   (caller)               all-to-all of send_dev -> recv_dev with the per-peer
 *                          counts of sfmm_gpu_shard_info (scalars; NCCL over
 *                          NVLink);
 *   sfmm_gpu_apply_end     unpack ghosts, the (remaining) translation tasks, staged
 *                          column sums, downward pass, scatter of the OWNED
 *                          points into u_dev (other entries untouched).
 * Symmetric plans (the default) evaluate a colleague pair split across two
 * ranks once, on one side, and return the other side's column sums in a
 * second exchange; sfmm_gpu_shard_info2 returns 1 and its per-peer counts,
 * and apply_end is replaced by
 *   sfmm_gpu_apply_mid     unpack ghosts, the (remaining) translation tasks,
 *                          pack the column sums owed to each peer into
 *                          send2_dev, record `packed_event`;
 *   (caller)               all-to-all of send2_dev -> recv2_dev (shard_info2
 *                          counts);
 *   sfmm_gpu_apply_fin     add the staged and received column sums, downward
 *                          pass, scatter of the owned points into u_dev.
 * q_dev holds all N charges (original order) on every rank.  The union over
 * ranks of the owned entries of u is the full result.  Trees with depth < 2
 * are computed by rank 0 alone.  Replaces nothing in the reference, which is
 * single-process (SPEC non-goal); see DESIGN.md section 6.
 */
int sfmm_gpu_plan_create_sharded(const sfmm_plan_desc* desc, int device, int n_ranks, int rank,
                                 sfmm_gpu_plan** out);
int sfmm_gpu_shard_info(const sfmm_gpu_plan* plan, int64_t* send_counts, int64_t* recv_counts,
                        int64_t* n_owned_points, int64_t* n_ghost_boxes);
int sfmm_gpu_apply_begin(sfmm_gpu_plan* plan, const void* q_dev, void* send_dev, void* stream,
                         void* packed_event);
int sfmm_gpu_apply_end(sfmm_gpu_plan* plan, const void* q_dev, const void* recv_dev, void* u_dev,
                       void* stream);
/* Returns 1 when the plan has the second exchange (apply_mid/_fin), else 0;
 * fills the per-peer scalar counts of that exchange (zeros when absent) and
 * the cut level of the ownership (see sfmm_gpu_shard_describe). */
int sfmm_gpu_shard_info2(const sfmm_gpu_plan* plan, int64_t* send2_counts, int64_t* recv2_counts,
                         int* cut_level);
int sfmm_gpu_apply_mid(sfmm_gpu_plan* plan, const void* recv_dev, void* send2_dev, void* stream,
                       void* packed_event);
int sfmm_gpu_apply_fin(sfmm_gpu_plan* plan, const void* q_dev, const void* recv2_dev, void* u_dev,
                       void* stream);

/*
 * Multi-GPU with the exchanges inside this library.
 *
 * Single process, several GPUs: sfmm_gpu_plan_create_multi builds one sharded
 * rank plan per entry of dev_ids (dev_ids[0] is the primary device; ids may
 * repeat, e.g. {0,0,0,0} runs four ranks on one GPU) and returns ONE plan that
 * sfmm_gpu_apply / sfmm_gpu_apply_async drive like a single-GPU plan: q and u
 * (host, or device buffers on the primary) in the original order, the result
 * bit-identical to the single-GPU plan's.  Each apply runs every rank's
 * gather + upward pass, one cudaMemcpyPeerAsync per (sender, receiver) ghost
 * segment over NVLink, the translations, one peer copy per column-sum segment,
 * and the downward pass; the other devices gather q and scatter u through
 * peer memory.  Distinct devices need peer access (SFMM_EUNSUPPORTED
 * otherwise).  Several right-hand sides run one column at a time.
 * _skel: operators taken device-to-device (peer copies) from a GPU
 * skeletonization result, as sfmm_gpu_plan_create_skel.
 */
int sfmm_gpu_plan_create_multi(const sfmm_plan_desc* desc, int n_dev, const int* dev_ids,
                               sfmm_gpu_plan** out);
int sfmm_gpu_plan_create_multi_skel(const sfmm_plan_desc* desc, const sfmm_skel_result* skel,
                                    int n_dev, const int* dev_ids, sfmm_gpu_plan** out);

/*
 * One process per GPU: after sfmm_gpu_plan_create_sharded(_T) of rank `rank`,
 * sfmm_gpu_plan_attach_nccl joins the ranks into one NCCL communicator (rank 0
 * makes the id with sfmm_gpu_nccl_unique_id and the caller broadcasts its 128
 * bytes, e.g. over MPI or torch.distributed).  sfmm_gpu_apply and
 * sfmm_gpu_apply_async on the plan are then COLLECTIVE (every rank calls them
 * with the same q) and run both exchanges as grouped ncclSend/ncclRecv on the
 * apply stream; u receives the full result (one in-place ncclAllReduce) or,
 * after sfmm_gpu_set_output(plan, SFMM_OUTPUT_OWNED), only the rank's owned
 * points.  libnccl.so.2 is loaded at run time (SFMM_NCCL_LIB overrides the
 * path); failures return SFMM_ENCCL.
 */
#define SFMM_NCCL_ID_BYTES 128
int sfmm_gpu_nccl_unique_id(void* id);
int sfmm_gpu_plan_attach_nccl(sfmm_gpu_plan* plan, const void* id, int n_ranks, int rank);
int sfmm_gpu_set_output(sfmm_gpu_plan* plan, int mode);

/* Operators of rank `rank`'s owned boxes without the full T on every rank:
 * sfmm_gpu_shard_T_runs (host-only) lists the runs [src, src + len) of
 * desc->T entries (T_off units) the rank needs, in order (n_entries: their
 * total; runs may be NULL to count); a holder of the full T on a device packs
 * them with sfmm_gpu_copy_runs (scalars_per_entry 1 real / 2 complex) and
 * ships the blob (NCCL); sfmm_gpu_plan_create_sharded_T builds the rank's plan
 * from the blob in its device memory, ignoring desc->T (may be NULL).
 * copy_runs with a NULL stream returns after the copies complete; plan
 * creation waits for all outstanding device work before reading the blob. */
int sfmm_gpu_shard_T_runs(const sfmm_plan_desc* desc, int n_ranks, int rank, int64_t* n_runs,
                          int64_t* runs, int64_t* n_entries);
int sfmm_gpu_copy_runs(const double* src_dev, const int64_t* runs, int64_t n_runs,
                       int64_t scalars_per_entry, double* dst_dev, int device, void* stream);
int sfmm_gpu_plan_create_sharded_T(const sfmm_plan_desc* desc, const void* T_owned_dev, int device,
                                   int n_ranks, int rank, sfmm_gpu_plan** out);

/* Host-only view of rank `rank`'s shard (no device is touched).  counts gets
 * 4*n_ranks + 4 values: send scalars per peer, receive scalars per peer,
 * owned points, ghost boxes, owned boxes, the second exchange's send and
 * receive scalars per peer, and the cut level (1: level-1 subtrees per rank;
 * 2: level-2 subtrees, the internal level-1 boxes shared, owner -1).
 * Non-NULL arrays receive the box
 * owners (n_boxes), the ghost-exchange element indices into [q slots | qhat]
 * (pack_idx: what this rank sends, per peer in rank order; unpack_idx: where
 * what it receives lands) and the owned points' original indices. */
int sfmm_gpu_shard_describe(const sfmm_plan_desc* desc, int n_ranks, int rank, int64_t* counts,
                            int32_t* owner, int64_t* pack_idx, int64_t* unpack_idx,
                            int32_t* owned_points);

/*
 * GPU tree and neighbor lists: the device counterpart
 * of the reference's build_tree + build_neighbors
 * (/root/reference/proj/src/tree.cpp:148-355), bit-identical to it: same perm,
 * level-major Morton box order, point ranges, level_begin and colleague /
 * coarse / fine lists.  Errors as the reference: EINVAL (bad dim, capacity,
 * point count, non-finite coordinate), EDUPLICATE (coincident points),
 * EDEPTH (leaf capacity unreachable at the maximum depth).
 */
typedef struct sfmm_tree_arrays {
  int32_t dim, depth, leaf_cap, n_boxes;
  int64_t n_points;
  const int32_t* perm;        /* tree position -> original index */
  const double* pts;          /* n_points*dim, tree order, interleaved */
  const int32_t* level_begin; /* depth+2 */
  const int32_t* box_parent;  /* -1 for the root */
  const int32_t* box_child;   /* n_boxes*8, by octant, -1 = none */
  const int32_t* box_level;
  const uint64_t* box_morton;
  const int64_t* box_cell;    /* n_boxes*3 */
  const double* box_center;   /* n_boxes*3 */
  const double* box_half;
  const int32_t* box_begin;
  const int32_t* box_end;
  const uint8_t* box_leaf;
  const int64_t* coll_off;    /* colleagues, ascending, self included */
  const int32_t* coll;
  const int64_t* coarse_off;
  const int32_t* coarse;
  const int64_t* fine_off;
  const int32_t* fine;
  double seconds;             /* wall time of the build */
} sfmm_tree_arrays;

typedef struct sfmm_gpu_tree sfmm_gpu_tree;

int sfmm_gpu_build_tree(int dim, int64_t n, const double* pts, int leaf_cap, int device,
                        sfmm_gpu_tree** out);
/* Points *arrays at the result's host arrays (valid until destroyed). */
int sfmm_gpu_tree_arrays(const sfmm_gpu_tree* tree, sfmm_tree_arrays* arrays);
void sfmm_gpu_tree_destroy(sfmm_gpu_tree* tree);

/* Distributed precompute (config 5 scale: no rank holds every operator).
 * Every rank builds the same tree (sfmm_gpu_build_tree is deterministic),
 * sfmm_gpu_subtree_owners picks each level-1 subtree's rank from the tree
 * alone (Morton-contiguous ranges balancing a near-field work estimate;
 * owner gets n_boxes entries, -1 above level 1), each rank skeletonizes its
 * subtrees (sfmm_gpu_build_skeletons_subset with mask owner[b] == rank), the
 * ranks exchange the index data of their boxes (index_vec, skel_pos, red_pos,
 * parent_offset: a few bytes per point) to form the full descriptor, and
 * sfmm_gpu_plan_create_sharded_owned builds the rank plan with that ownership
 * from the rank's own operators (the subset result's device T, box order).
 * The rank plans are those of sfmm_gpu_plan_create_sharded_T with the same
 * ownership: attach NCCL, apply as usual. */
int sfmm_gpu_subtree_owners(const sfmm_tree_arrays* tree, int n_ranks, int32_t* owner);
int sfmm_gpu_plan_create_sharded_owned(const sfmm_plan_desc* desc, const void* T_owned_dev,
                                       int device, int n_ranks, int rank, const int32_t* owner,
                                       sfmm_gpu_plan** out);

/*
 * GPU skeletonization: the device counterpart of the
 * reference's build_skeletons (/root/reference/proj/src/skeleton.cpp:184-260).
 * Input: the tree (box geometry included, since proxy surfaces are built from
 * box centres and half-widths).  Output: the skeleton fields of an
 * sfmm_plan_desc (index_vec, skel_pos, red_pos, interp T, parent_offset), held
 * by an opaque result until destroyed.  Same algorithm as the reference:
 * proxy matrix from the Lobatto proxy surface (stacked with its conjugate for
 * complex kernels), greedy Householder column-pivoted QR stopped at
 * tol * (largest initial column norm) with the dqp3 norm downdate,
 * T = R11^{-1} R12, positions sorted ascending.  Pivot choices are
 * rounding-sensitive, so results are compared by accuracy, not bits.
 */
typedef struct sfmm_tree_desc {
  int32_t dim;
  int64_t n_points;
  int32_t n_boxes;
  int32_t depth;
  const double* pts;          /* tree order, interleaved */
  const int32_t* level_begin; /* depth+2 */
  const int32_t* box_parent;
  const int32_t* box_level;
  const int32_t* box_begin;
  const int32_t* box_end;
  const uint8_t* box_leaf;
  const double* box_center;   /* n_boxes * 3 */
  const double* box_half;     /* n_boxes */
} sfmm_tree_desc;

int sfmm_gpu_build_skeletons(const sfmm_tree_desc* tree, int kernel, double kappa, double tol,
                             double proxy_radius, int proxy_edge2d, int proxy_face3d, int device,
                             sfmm_skel_result** out);
/* Distributed precompute: skeletonizes only the boxes with box_mask[b] != 0
 * (n_boxes entries; whole subtrees -- a masked box's children must be masked,
 * else SFMM_EINVAL), e.g. the level-1 subtrees a rank owns
 * (sfmm_gpu_subtree_owners).  The other boxes come out empty (n = k = 0, no
 * T), so the result's T is exactly the rank's owned operators in box order --
 * the T_owned_dev blob of sfmm_gpu_plan_create_sharded_owned.  Each masked
 * box's skeleton is bit-identical to the full build's (it depends only on its
 * own subtree).  box_mask = NULL is sfmm_gpu_build_skeletons. */
int sfmm_gpu_build_skeletons_subset(const sfmm_tree_desc* tree, int kernel, double kappa,
                                    double tol, double proxy_radius, int proxy_edge2d,
                                    int proxy_face3d, int device, const uint8_t* box_mask,
                                    sfmm_skel_result** out);
/* Points the skeleton fields of *desc (iv_off, iv, sk_off, skel_pos, rd_off,
 * red_pos, T_off, T, box_parent_offset) at the result's arrays and returns
 * k_max, proj_scalars and the number of saturated boxes.  The interpolation
 * operators stay resident on the device that built them; with_host_T = 0 leaves
 * desc->T NULL (no device->host copy), with_host_T = 1 downloads them once into
 * the result (sfmm_gpu_skel_fill = sfmm_gpu_skel_describe(.., 1, ..)). */
int sfmm_gpu_skel_describe(sfmm_skel_result* res, sfmm_plan_desc* desc, int with_host_T,
                           int32_t* k_max, int64_t* proj_scalars, int32_t* saturated,
                           double* seconds);
int sfmm_gpu_skel_fill(sfmm_skel_result* res, sfmm_plan_desc* desc, int32_t* k_max,
                       int64_t* proj_scalars, int32_t* saturated, double* seconds);
/* Device copy of T (box order, indexed by the result's T_off; interleaved
 * complex for Helmholtz): the device it lives on and its length in doubles. */
const double* sfmm_gpu_skel_device_T(const sfmm_skel_result* res, int* device,
                                     int64_t* n_scalars);
void sfmm_gpu_skel_destroy(sfmm_skel_result* res);

/* Device-side plan build: as sfmm_gpu_plan_create /
 * _create_sharded, but the interpolation operators are taken device-to-device
 * from `skel` (built on the same device) and desc->T is ignored, so T never
 * leaves HBM.  desc's skeleton fields must be those of `skel`
 * (sfmm_gpu_skel_describe).  `skel` may be destroyed after the call. */
int sfmm_gpu_plan_create_skel(const sfmm_plan_desc* desc, const sfmm_skel_result* skel,
                              int device, int n_ranks, int rank, sfmm_gpu_plan** out);

/*
 * The whole pipeline on the GPU in one call: tree + neighbor
 * lists (sfmm_gpu_build_tree, bit-identical to the reference), skeletons
 * (sfmm_gpu_build_skeletons) and the plan, with the interpolation operators
 * kept in HBM (sfmm_gpu_plan_create_skel) -- the device counterpart of the
 * reference's build_tree + build_neighbor_lists + build_skeletons + make_plan
 * followed by sfmm_gpu_plan_create.  pts: n x dim, original order; proxy
 * parameters <= 0 take the reference defaults (2.95, 24, 8).
 */
int sfmm_gpu_plan_from_points(int kernel, double kappa, int dim, int64_t n, const double* pts,
                              int leaf_cap, double tol, double proxy_radius, int proxy_edge2d,
                              int proxy_face3d, int device, sfmm_gpu_plan** out);

/* Phase timing.  While enabled, every apply records CUDA events on its stream
 * around its five phases (0 gather, 1 upward, 2 translate, 3 downward,
 * 4 scatter).  sfmm_gpu_get_timings synchronises, writes ms[5*i + phase] for
 * up to max_applies recorded applies, sets *n_applies and clears the record. */
int sfmm_gpu_set_timing(sfmm_gpu_plan* plan, int enable);
int sfmm_gpu_get_timings(sfmm_gpu_plan* plan, float* ms, int max_applies, int* n_applies);

/* Dense u_i = sum_{j != i} G(x_i, x_j) q_j over the points in their given
 * order, for the listed targets only (oracle.cpp:51-71), on the device.
 * pts: n*dim host coords; q, u host arrays (u has n_targets scalars). */
int sfmm_gpu_direct_sum(int kernel, double kappa, int dim, int64_t n, const double* pts,
                        const void* q, int64_t n_targets, const int32_t* targets, void* u,
                        int device);

const char* sfmm_gpu_last_error(void);

/* Library version string, and the CUDA arch it was compiled for. */
const char* sfmm_gpu_version(void);

#ifdef __cplusplus
}
#endif

#endif /* SFMM_GPU_H_ */
