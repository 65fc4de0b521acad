/*
 * rfd.h -- C ABI of the B200-native RFDiffusion (RFD) graph-field integrator.
 *
 * What it computes (arXiv 2302.00942, Sec. 2.4 "RFDiffusion",
 * lines 283-366, Eq. 13 at PAPER.md:351-358):
 *
 *     out = exp(lambda * W~) F,     W~ = Phi D Phi^T  (N x N, never formed)
 *
 * for a point cloud x_1..x_N in R^3 and a field F (N x d), where
 *   omega_k ~ N(0, I_3) truncated to ||omega||_1 <= R = 10
 *   nu_k    = tau(omega_k) / (m p(omega_k)),  D = diag(nu, nu)
 *   tau(w)  = prod_c sin(2 pi eps w_c) / (pi w_c)                 (2pi-corrected)
 *   phi(x)  = [cos 2 pi omega_k.x ; sin 2 pi omega_k.x]_{k<m}
 * evaluated in closed form, inverse-free (reading A5):
 *   out = F + Phi . C^ . (Phi^T F),  C^ = lambda D phi1(lambda G D),  G = Phi^T Phi.
 *
 * Plan creation is the paper's "pre-processing" (linear in N, cubic in m,
 * PAPER.md:359); rfd_integrate is its "inference" (linear in N, quadratic
 * in m).  The random stream is part of the contract (A14):
 * frequency k, attempt a uses Philox4x32-10 with counter (k, a, 0x52464421, 0)
 * and key (seed & 0xffffffff, seed >> 32); uniforms (w + 0.5) 2^-32;
 * Box-Muller z0 = sqrt(-2 ln u0) cos 2pi u1, z1 = sqrt(-2 ln u0) sin 2pi u1,
 * z2 = sqrt(-2 ln u2) cos 2pi u3; accept iff |z0|+|z1|+|z2| <= R; omega = fp32(z).
 *
 * Conventions for every entry point:
 *   - Arrays are row-major fp32 unless stated; "device" pointers are CUDA
 *     device (or managed) memory of the current device, 16-byte aligned.
 *   - `stream` is a cudaStream_t (NULL = legacy default stream).  Work is
 *     enqueued on it; calls on one plan must be ordered on one stream.
 *   - No exception crosses the ABI.  A non-OK status leaves a message for
 *     rfd_last_error() (thread-local) and leaves any existing plan unchanged.
 *   - There is no CPU fallback: every arithmetic step runs in the library's
 *     CUDA kernels (sm_100a).  Without a usable GPU the calls return
 *     RFD_ECUDA.
 *
 * Coordinate range.  W depends on the points only through n_i - n_j
 * (Eq. 9), so the library first moves each cloud to the
 * midpoint c of its bounding box (exact: phi(c + y) = R phi(y) with a 2x2
 * rotation R per frequency that commutes with D; exported G, C^, S, Y are
 * rotated back).  Results are therefore translation-invariant.  The feature
 * argument 2 pi omega.(x - c) is evaluated in fp32, so the error grows with
 * T = max_k sum_c |omega_kc| h_c (turns; h = the box's half-extents):
 * measured normwise Delta error ~1.6e-7 T (1.1e-6 at T = 5.9, 7.2e-6 at
 * T = 59, 4.8e-5 at T = 295; tests/test_gpu_parity.py::
 * test_translated_and_scaled_clouds_parity).  The 1e-4 parity gate holds for
 * T up to ~500 turns; unit-scale clouds (all five configs) have T = 3 .. 6.
 */
#ifndef RFD_H_
#define RFD_H_

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

typedef struct rfd_plan rfd_plan;          /* opaque; owns all derived state   */
typedef struct CUstream_st* rfd_stream;    /* == cudaStream_t                   */

typedef enum {
  RFD_OK = 0,
  RFD_EINVAL = 1,  /* bad argument: n<1, m<1 or m>RFD_MAX_M, d<1, batch<1,
                      eps not finite or <= 0, lambda not finite, NULL or
                      misaligned pointer                                       */
  RFD_ECUDA = 2,   /* CUDA runtime error (no device, launch failure, ...)      */
  RFD_ENOMEM = 3,  /* device allocation failed                                 */
  RFD_ERANGE = 4   /* exp(lambda W~) overflows (e.g. lambda > 0 with large
                      ||lambda G D||, or negative nu with lambda < 0), or the
                      frequency sampler exhausted its 64 attempts              */
} rfd_status;

#define RFD_MAX_M 512          /* frequencies; r = 2m feature columns <= 1024 */
#define RFD_TRUNCATION_R 10.0  /* L1 radius of the frequency proposal (A6)   */

/*
 * rfd_plan_create -- pre-processing for one point cloud.
 *   points  N x 3 fp32, HOST or DEVICE memory (detected); copied into the
 *           plan's own layout, so the caller may free it when this returns.
 *   n       number of points N >= 1.
 *   eps     epsilon-graph radius (> 0).  Enters only nu (tau).
 *   lambda  diffusion multiplier (any finite real; exp(lambda W~)).
 *   m       number of random frequencies, 1 <= m <= RFD_MAX_M (r = 2m).
 *   seed    Philox key (see the stream layout above).
 *   plan_out receives the new plan on RFD_OK (NULL otherwise).
 * Steps: frequencies + nu (a1-a2), Gram G = Phi^T Phi (a4), core C^ (a5).
 * a4 is the sum over points or -- one cloud, m > 64,
 * N >= 2^19, when the spread grid has <= N/8 nodes -- the same G through a spread grid
 * (a type-3 NUFFT identity; G within 3e-7 normwise of the exact sum, DESIGN.md
 * Sec. 6; rfd_plan_info_t.gram_nodes says which).  Blocks the host until the
 * plan is ready (it reads back the bounding box and omega to size that grid,
 * the core's scaling exponent and an overflow flag).  Errors: EINVAL, ENOMEM,
 * ECUDA, ERANGE.
 */
rfd_status rfd_plan_create(const float* points, int64_t n, double eps,
                           double lambda, int32_t m, uint64_t seed,
                           rfd_stream stream, rfd_plan** plan_out);

/*
 * rfd_plan_create_batched -- `batch` independent clouds of n points each,
 * points laid out batch x n x 3.  The clouds share omega and nu (one seed)
 * and each gets its own G_b and C^_b.  This is the repeated-application
 * pattern of the paper's Alg. 1 over many clouds.
 */
rfd_status rfd_plan_create_batched(const float* points, int32_t batch,
                                   int64_t n, double eps, double lambda,
                                   int32_t m, uint64_t seed, rfd_stream stream,
                                   rfd_plan** plan_out);

/*
 * Multi-GPU: one cloud sharded across the ranks of a process group (SURVEY
 * Sec. 8(e)), one GPU per rank, each rank holding a contiguous part of the
 * points (and the same rows of every field).  The two sums over points -- G =
 * Phi^T Phi (B^T A) at plan creation and S = Phi^T F
 * (Eq. 13's first bracket) in every rfd_integrate -- are linear in the points
 * (PAPER.md:359), so each rank computes its shard's partial and the ranks
 * exchange partials once per sum (plus the shards' bounding boxes once at
 * creation, so that every rank centres the cloud on the same point).  The
 * exchange is an ALL-GATHER performed by the caller's collective library
 * through `allgather` (the Python binding uses torch.distributed over NCCL):
 *   allgather(ctx, send, recv, count, stream)  send: `count` fp64 on the
 *     plan's device; recv: world x count fp64 on the device, rank-major (recv
 *     + q count = rank q's send).  Ordered on `stream` (enqueued on it, or
 *     complete on return).  Returns 0 on success (non-zero -> RFD_ECUDA).
 * The library adds the gathered partials in rank order, so every rank holds
 * bitwise the same G, C^, S and Y; each rank's out rows are its own points'.
 * Every rank must make the same sequence of calls (collective semantics).
 */
typedef int (*rfd_allgather_fn)(void* ctx, const double* send, double* recv, size_t count,
                                rfd_stream stream);
typedef struct {
  int32_t rank;               /* 0 <= rank < world                            */
  int32_t world;              /* ranks in the group (>= 1)                    */
  rfd_allgather_fn allgather; /* the exchange (see above); NULL iff world == 1 */
  void* ctx;                  /* passed through to allgather                  */
} rfd_shard;

/*
 * rfd_plan_create_sharded -- rfd_plan_create for this rank's shard of one
 * cloud.  points: n_local x 3 (host or device), n_local >= 1; eps, lambda, m,
 * seed as rfd_plan_create and equal on every rank.  The plan records N = the
 * sum of the shards' n_local (rfd_plan_info_t.n_total).  rfd_integrate and
 * rfd_integrate_host on the plan take this rank's n_local x d rows and
 * exchange S; rfd_plan_reparam / rfd_plan_spectrum / rfd_plan_export work on
 * the merged (global) G.  rfd_barycenter refuses sharded plans (EINVAL).
 * Errors: as rfd_plan_create, EINVAL for a bad `shard`, ECUDA if the
 * exchange fails.
 */
rfd_status rfd_plan_create_sharded(const float* points, int64_t n_local, double eps,
                                   double lambda, int32_t m, uint64_t seed,
                                   const rfd_shard* shard, rfd_stream stream,
                                   rfd_plan** plan_out);

/*
 * rfd_plan_reparam -- re-parameterise a plan to a new (eps, lambda) without
 * recomputing the Gram matrix: G = Phi^T Phi
 * depends only on the points and omega, so only nu
 * (a2, eps enters through tau: PAPER.md:361-366) and the core C^ (a5,
 * PAPER.md:333-339) are recomputed -- O(m + r^3) instead of O(N r^2).  The
 * paper grid-searches lambda and eps per mesh.
 *   plan    a plan from rfd_plan_create[_batched]; keeps omega, G, points.
 *   eps     new epsilon (> 0, finite); lambda  new multiplier (finite).
 * The result equals, bit for bit, a fresh rfd_plan_create with the same
 * points, m, seed and the new (eps, lambda).  The new nu and C^ are written
 * into the plan's existing buffers (CUDA graphs capturing rfd_integrate stay
 * valid).  Must be ordered after earlier rfd_integrate calls on the plan
 * (same stream).  Blocks the host (scaling exponent / overflow read-back).
 * Errors: EINVAL (NULL plan, bad eps or lambda), ERANGE (core overflow),
 * ENOMEM, ECUDA -- the plan is unchanged on any error.
 */
rfd_status rfd_plan_reparam(rfd_plan* plan, double eps, double lambda,
                            rfd_stream stream);

/*
 * rfd_plan_spectrum -- the k smallest eigenvalues of the kernel matrix
 * K = exp(lambda W~), W~ = Phi D Phi^T (N x N, never formed), per cloud
 * (classification features
 * "the k smallest eigenvalues of the kernel matrix" via the low-rank
 * decomposition).  The nonzero eigenvalues of Phi D Phi^T
 * are those of G D (r x r); each maps through exp(lambda .), the N - r null
 * directions give 1; for N < r the r - N eigenvalues of G D of smallest
 * modulus (exact zeros) are dropped (A19).  O(r^3) fp64 on the
 * plan's G: Householder tridiagonalisation of D^1/2 G D^1/2, then bisection.
 *   k     1 <= k <= N eigenvalues per cloud, ascending.
 *   out   batch x k fp64, HOST or DEVICE memory (cudaMemcpyDefault).
 * Requires all nu > 0 (rfd_plan_info_t.symmetric == 1; otherwise EINVAL).
 * Blocks the host until `out` is written.  Errors: EINVAL, ENOMEM, ECUDA.
 */
rfd_status rfd_plan_spectrum(rfd_plan* plan, int32_t k, double* out, rfd_stream stream);

/*
 * rfd_barycenter -- entropic Wasserstein barycenter of k distributions on the
 * plan's cloud (Appendix D Algorithm 1,
 * lines 1036-1051, with FM_K = rfd_integrate):
 *   w^i <- mu^i / FM_K(a * v^i);  d^i <- v^i * FM_K(a * w^i);
 *   mu <- prod_i (d^i)^alpha_i (mu reset to ones each iteration);
 *   v^i <- v^i * mu / d^i
 * with the readings of SPEC.md:559, 628-629 (A20): mu reset to ones
 * each outer iteration, both denominators (FM_K(a * v^i) and d^i) clamped at
 * 1e-30 (d^i before its power), stop after max_iter or when
 * ||mu_new - mu_old||_1 < tol (tol = 0: run max_iter), output normalised so
 * <a, mu> = 1.  The iterates v, w, d, mu are fp64; the k distributions are
 * the k columns of one field, so each FM_K is one multi-column rfd_integrate
 * on fp32(a v s) with s a per-column power of two (exact by linearity; keeps
 * fp32 in range).  The paper runs it with lambda > 0 (0.5).
 *   mu     DEVICE k x N fp32 (row i = distribution i).   area  DEVICE N fp32.
 *   alpha  HOST k fp64, > 0, sum 1.   1 <= k <= 16, max_iter >= 1, tol >= 0.
 *   out    DEVICE N fp32 (the barycenter).   iters  HOST (may be NULL):
 *          iterations run.
 * Single-cloud plans only.  Blocks the host (convergence test / final
 * read-back).  Errors: EINVAL, ERANGE (non-finite iterate; the message names
 * the iteration), ENOMEM, ECUDA.
 */
rfd_status rfd_barycenter(rfd_plan* plan, const float* mu, const float* area, const double* alpha,
                          int32_t k, int32_t max_iter, double tol, float* out, int32_t* iters,
                          rfd_stream stream);

/*
 * rfd_integrate -- inference, Eq. 13 in bracket order:
 *   S = Phi^T F (a6), Y = C^ S (a7), out = F + Phi Y (a8).
 *   F    DEVICE, (batch x) N x d fp32.   out  DEVICE, same shape; may alias F.
 *   d    field channels >= 1.
 * Fully asynchronous on `stream`; CUDA-graph capturable once the plan's
 * workspace has been sized for this d (any earlier call with d' >= d).
 * Errors: EINVAL (NULL/misaligned pointers, d < 1), ENOMEM (workspace
 * growth), ECUDA.
 */
rfd_status rfd_integrate(rfd_plan* plan, const float* F, int32_t d, float* out,
                         rfd_stream stream);

/*
 * rfd_integrate_host -- the same with HOST buffers: copies F host->device,
 * integrates, copies out device->host, ordered on `stream`.  Single clouds
 * with d <= 64 and n >= 16384 are pipelined: F travels in 8 point-range
 * chunks on an internal copy stream and pass 1 runs per chunk as it lands;
 * pass 2 runs per chunk with each chunk's D2H copy right behind it (pass-1
 * partials of all chunks summed in a fixed order: deterministic).  With
 * pinned host memory the call is asynchronous (synchronize `stream` before
 * reading out); with pageable memory the copies block the host.
 */
rfd_status rfd_integrate_host(rfd_plan* plan, const float* F_host, int32_t d,
                              float* out_host, rfd_stream stream);

/*
 * rfd_gfi -- the whole graph-field integration i = exp(lambda W~) F (PAPER.md
 * Eq. 1 with Sec. 2.4's kernel: pre-processing + inference) for a DEVICE
 * field in one call.  The field's pass 1 (S = Phi^T F, which needs only the
 * points, omega and F) runs on an internal second stream beside the plan's
 * core, whose small fp64 GEMMs fit on the SMs next to pass 1's CTAs; then
 * a7 and pass 2 on `stream`.  Same kernels and results (bitwise) as
 * rfd_plan_create + rfd_integrate.
 *   points  n x 3 fp32, HOST or DEVICE (as rfd_plan_create).
 *   F, out  n x d DEVICE fp32, 16-byte aligned (out may alias F).
 *   plan_out  NULL (the plan is destroyed, stream-ordered) or receives the
 *           plan for reuse (rfd_integrate on further fields).
 * Blocks the host while the plan's core is formed (as rfd_plan_create); the
 * core's overflow check waits until the inference is enqueued behind it, so
 * on RFD_ERANGE the contents of out are unspecified.  out is ready when
 * `stream` is.  Errors: as rfd_plan_create and rfd_integrate; EINVAL if F or
 * out is host memory.
 */
rfd_status rfd_gfi(const float* points, int64_t n, double eps, double lambda, int32_t m,
                   uint64_t seed, const float* F, int32_t d, float* out, rfd_stream stream,
                   rfd_plan** plan_out);

/*
 * rfd_gfi_host -- the whole graph-field integration i = exp(lambda W~) F
 * (Eq. 1 with Sec. 2.4's kernel: pre-processing + inference) from
 * HOST buffers in one call, overlapping the transfers with the computation:
 * the points go up first, the field's H2D copies (in point-range chunks, on
 * an internal copy stream) run while the plan's frequencies, Gram and core
 * compute, pass 1 consumes each chunk as it lands, and the D2H copies of out
 * follow pass 2 chunk by chunk.  Same arithmetic as rfd_plan_create +
 * rfd_integrate_host (bitwise).
 *   points  n x 3 HOST fp32;  F_host / out_host  n x d HOST fp32 (pinned for
 *           asynchrony; out may alias F); other arguments as rfd_plan_create.
 *   plan_out  NULL (the plan is destroyed) or receives the plan for reuse.
 * Blocks the host while the plan's core is formed (as rfd_plan_create);
 * synchronize `stream` before reading out_host.  Errors: as rfd_plan_create
 * and rfd_integrate_host.
 */
rfd_status rfd_gfi_host(const float* points, int64_t n, double eps, double lambda, int32_t m,
                        uint64_t seed, const float* F_host, int32_t d, float* out_host,
                        rfd_stream stream, rfd_plan** plan_out);

/* rfd_destroy -- frees the plan and its device memory.  NULL-safe. */
void rfd_destroy(rfd_plan* plan);

/* rfd_last_error -- message for the last non-OK status of this thread. */
const char* rfd_last_error(void);

/* Plan geometry. */
typedef struct {
  int64_t n;        /* points per cloud                       */
  int32_t batch;    /* clouds                                 */
  int32_t m;        /* frequencies                            */
  int32_t r;        /* feature columns, 2m                    */
  int32_t scaling;  /* squarings s used by the core           */
  int32_t symmetric;/* 1: core via D^1/2 G D^1/2 (all nu > 0) */
  double eps, lambda;
  uint64_t seed;
  int64_t n_total;  /* points of the whole cloud (= n unless sharded) */
  int32_t rank;     /* shard of this plan (0 unless sharded)          */
  int32_t world;    /* shards (1 unless sharded)                      */
  int64_t gram_nodes; /* a4 went through a spread grid of this many nodes
                         (0: the direct sum over the points) */
} rfd_plan_info_t;
rfd_status rfd_plan_info(const rfd_plan* plan, rfd_plan_info_t* info);

/*
 * rfd_plan_export -- copy plan state to HOST memory (tests / introspection).
 * Feature index order is the paper's: columns 0..m-1 cosines, m..2m-1 sines;
 * G, C^, S, Y in the paper's basis of the UNcentred points (rotated back from
 * the device's centred basis in fp64; Y rounded to fp32 after the rotation).
 *   RFD_OMEGA  m x 3 fp32          RFD_NU    m fp64
 *   RFD_GRAM   batch x r x r fp64  RFD_CORE  batch x r x r fp64
 *   RFD_S      batch x r x d fp64  RFD_Y     batch x r x d fp32
 *              (S, Y: from the last rfd_integrate on this plan)
 * `bytes` must equal the field's size.  Synchronizes the device.
 */
typedef enum {
  RFD_OMEGA = 0, RFD_NU = 1, RFD_GRAM = 2, RFD_CORE = 3, RFD_S = 4, RFD_Y = 5
} rfd_field;
rfd_status rfd_plan_export(const rfd_plan* plan, rfd_field which,
                           void* host_dst, size_t bytes);

/*
 * Instrumentation (bench / tests).
 *   rfd_launch_count  kernels this library has launched in this process.
 *   rfd_profile_enable(1) brackets every subsequent launch with CUDA events
 *     on its stream; rfd_profile_read synchronizes, then returns up to `cap`
 *     per-kernel aggregates (name, launches, total ms) since the last
 *     enable / read, and resets them.  Returns the number of entries.
 *   rfd_profile_only(name) restricts the events to launches of that kernel
 *     name (NULL or "": every launch), so a timed region can measure one
 *     kernel live without bracketing the others.
 */
uint64_t rfd_launch_count(void);
rfd_status rfd_profile_enable(int on);
rfd_status rfd_profile_only(const char* name);
typedef struct {
  char name[48];
  int64_t launches;
  double total_ms;
} rfd_profile_entry;
int32_t rfd_profile_read(rfd_profile_entry* entries, int32_t cap);

#ifdef __cplusplus
}
#endif
#endif /* RFD_H_ */
