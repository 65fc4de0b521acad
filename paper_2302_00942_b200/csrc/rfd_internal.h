// Internal declarations shared by the host plan object and the kernels.
//
// Internal feature layout ("interleaved"): feature 2k is cos(2 pi omega_k.x),
// feature 2k+1 is sin(2 pi omega_k.x).  G, C^, S and Y are stored in this
// order on the device; rfd_plan_export permutes to the paper's
// [cos block; sin block] order.
#pragma once

#include <cuda_runtime.h>
#include <stdint.h>

#include <utility>

namespace rfd {
// Launch with programmatic stream serialization (PDL): the kernel may start
// once the previous kernel in the stream has executed
// griddepcontrol.launch_dependents; it must execute griddepcontrol.wait
// before touching that kernel's results.
template <typename... KArgs, typename... Args>
inline cudaError_t launch_pdl(void (*kernel)(KArgs...), dim3 grid, dim3 block, size_t smem,
                              cudaStream_t s, Args&&... args) {
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = grid;
  cfg.blockDim = block;
  cfg.dynamicSmemBytes = smem;
  cfg.stream = s;
  cudaLaunchAttribute attr[1];
  attr[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
  attr[0].val.programmaticStreamSerializationAllowed = 1;
  cfg.attrs = attr;
  cfg.numAttrs = 1;
  return cudaLaunchKernelEx(&cfg, kernel, std::forward<Args>(args)...);
}
}  // namespace rfd

namespace rfd {

constexpr uint32_t kFreqTag = 0x52464421u;  // counter word 2 (A14)
constexpr int kMaxAttempts = 64;

// ---------------------------------------------------------------- launching
// Every kernel launch goes through launch_begin/launch_end so that the
// library can count launches and (optionally) time them with events.
void launch_begin(const char* name, cudaStream_t s);
void launch_end(const char* name, cudaStream_t s);

struct LaunchScope {
  const char* name;
  cudaStream_t s;
  LaunchScope(const char* n, cudaStream_t st) : name(n), s(st) { launch_begin(n, st); }
  ~LaunchScope() { launch_end(name, s); }
};

// ---------------------------------------------------------------- K0 freq
// omega4[k] = (wx, wy, wz, 0) fp32, omega_rad4[k] = fp32(2 pi omega_k), nu[k]
// fp64; flags[0] |= 1 if some nu <= 0, |= 2 if the sampler ran out of attempts.
void launch_freq(float4* omega4, float4* omega_rad4, double* nu, int* flags, int m,
                 uint64_t seed, double eps, double R, double c_r, cudaStream_t s);

// a2 alone from the stored omega (re-parameterisation); flags[0] |= 1 if some
// nu <= 0.
void launch_nu(const float4* omega4, double* nu, int* flags, int m, double eps, double c_r,
               cudaStream_t s);

// ---------------------------------------------------------------- pack
// Per-cloud bounding box of the points (bbox: batch x 6 uint, ordered
// encoding: [0..2] = max ~enc(x) (the minima), [3..5] = max enc(x)).
// part: scratch of bbox_chunks(n, batch, sms) x batch x 6 + batch uint.
int bbox_chunks(int64_t n, int batch, int sms);
void launch_bbox(const float* xyz, unsigned int* bbox, unsigned int* part, int64_t n, int batch,
                 int sms, cudaStream_t s);
// centre c = the bbox midpoint (centre: batch float4); pts / pts16 / gpts (the
// Gram layout, gper points per cloud) = points - c.
// a4's spread-grid kernel width in nodes per axis (k_nufft.cu)
constexpr int kNufftWidth = 8;
// Cell counting for a4's spread grid, fused into the packing (k_nufft.cu):
// the cell of a centred point y on the grid (node l at (l - L) h) is
// [(l - L) h, (l - L + 1) h) per axis, clamped so its kNufftWidth-node
// window (l - w/2 + 1 .. l + w/2) fits.
struct CellCount {
  int L[3], n[3];
  float inv_h[3];
  int* count;   // ncells + 1, zeroed by the caller
  int* cell;    // n
  int* rank;    // n: position inside the cell (atomic, arbitrary order)
};
__device__ __forceinline__ int grid_cell(float x, float y, float z, const CellCount& g) {
  constexpr int lo = kNufftWidth / 2 - 1, hi = kNufftWidth / 2 + 1;
  const int i0 = min(max(__float2int_rd(x * g.inv_h[0]) + g.L[0], lo), g.n[0] - hi);
  const int i1 = min(max(__float2int_rd(y * g.inv_h[1]) + g.L[1], lo), g.n[1] - hi);
  const int i2 = min(max(__float2int_rd(z * g.inv_h[2]) + g.L[2], lo), g.n[2] - hi);
  return (i0 * g.n[1] + i1) * g.n[2] + i2;
}
// gpts NULL: no Gram layout (a4 through the spread grid); cc != NULL: also
// count the points into the grid's cells (batch = 1).
void launch_pack_points(const float* xyz, const unsigned int* bbox, float4* pts, float* pts16,
                        float* gpts, int64_t gper, float4* centre, int64_t n, int batch,
                        const CellCount* cc, cudaStream_t s);
// out (fp64, batch x r x cols) = R X (right: R X R^T, cols = r) with R the
// per-frequency rotation by 2 pi omega.c_b (centred -> paper basis).  X fp64,
// or Xf fp32 when X is NULL.
void launch_rotate(const double* X, const float* Xf, int r, int cols, int batch, bool right,
                   const float4* omega4, const float4* centre, double* out, cudaStream_t s);

// ---------------------------------------------------------------- shards
// SURVEY Sec. 8(e) (k_shard.cu): send = the shard's bbox as 6 fp64 + its
// point count; bbox = union of the world x 7 gathered values; out = the
// rank-ordered sum of world x count gathered partials.
void launch_bbox_export(const unsigned int* bbox, int64_t n_local, double* send, cudaStream_t s);
void launch_bbox_merge(const double* recv, int world, unsigned int* bbox, cudaStream_t s);
void launch_sum_parts(const double* parts, int world, int64_t count, double* out, cudaStream_t s);

// ---------------------------------------------------------------- Gram
struct GramGeom {
  int r;          // 2m
  int tile;       // 64 or 128
  int tiles1d;    // ceil(r / tile)
  int ntiles;     // upper-triangle tiles
  int chunks;     // point chunks per cloud
  int64_t chunk;  // points per chunk (multiple of 16)
};
// Tensor-core Gram (k_gram_tc.cu): GramGeom.ntiles holds the number of units.
GramGeom gram_tc_geometry(int m, int64_t n, int batch, int sms);
size_t gram_tc_partial_elems(const GramGeom& g, int batch);
// where launch_pack_points writes the points in the Gram's layout inside the
// `partial` workspace (per_cloud: padded points per cloud)
float* gram_points(const GramGeom& g, int batch, float* partial, int64_t* per_cloud);
// weighted: sum_p w_p^2 phi phi^T with w_p in the layout's pad slot (CTA-pair
// path only, gram_tc_pairs(m)).
bool gram_tc_pairs(int m);
void launch_gram_tc(const float4* omega4, int m, int64_t n, int batch, const GramGeom& g,
                    float* partial, double* G, cudaStream_t s, bool weighted = false);

// a4 through a spread grid (k_nufft.cu) for large single clouds.
struct NufftGrid {
  int L[3], n[3];          // node l at (l - L) h per axis, n = 2 L + 1 nodes
  int64_t nodes;
  float h[3], inv_h[3], inv_alpha[3], beta_l2e;   // what the kernels use
  double alpha_eff[3], beta_eff;                  // the kernel they implement
  double wscale;           // grid Gram weights sqrt(b wscale) (power of two)
};
// Grid for the cloud's bbox (launch_bbox encoding, host copy) and omega (host
// copy); false when the grid would be too large.
bool nufft_grid(const unsigned int* bbox, const float4* omega4, int m, int64_t n, NufftGrid* g);
size_t nufft_workspace_bytes(const NufftGrid& g, int64_t n, int m, int sms);
// The cell-count arrays inside the workspace (count zeroed here, on s): for
// launch_pack_points, which must run before launch_gram_nufft.
cudaError_t nufft_cell_count(const NufftGrid& g, int64_t n, int m, int sms, void* ws,
                             CellCount* cc, cudaStream_t s);
// G (r x r fp64, interleaved) of the centred points pts, counted into the
// workspace's cells by launch_pack_points.
// The grid's zeroing and the phi^ tables (they need only omega and the grid
// geometry): launch_gram_nufft does them itself when side_done is NULL;
// otherwise the caller ran launch_nufft_side on another stream and side_done
// marks its end.
cudaError_t launch_nufft_side(const float4* omega_rad4, int m, int64_t n, const NufftGrid& g,
                              int sms, void* ws, cudaStream_t s);
cudaError_t launch_gram_nufft(const float4* pts, int64_t n, const float4* omega_rad4, int m,
                              const NufftGrid& g, int sms, void* ws, double* G, cudaStream_t s,
                              cudaEvent_t side_done = nullptr);

// ---------------------------------------------------------------- core
// Z_b = lambda D^1/2 G D^1/2 (symmetric route) or lambda G D; atomicMax of
// max_b ||Z_b||_1 (fp64 bits) into *norm_bits (zeroed by the caller).
void launch_core_prep(const double* G, const double* nu, const int* flags,
                      double lambda, int m, int batch, double* Z,
                      unsigned long long* norm_bits, cudaStream_t s);
// Taylor (degree 20, Paterson-Stockmeyer) of phi1 and exp at Z / 2^s
// (||Z / 2^s||_1 <= kCoreTheta), then s doublings, then C^ = lambda D^1/2 P
// D^1/2 (or lambda D P); oflag = 1 on overflow.  work: kCoreWork matrices.
// sym: the symmetric route was taken (flags[0] bit 0 clear, read back by the
// host): every product is symmetric and only its upper tiles are computed.
// work[0..4) must hold (pw_alpha Z)^k, k = 2..5, from launch_core_powers
// (pw_alpha a power of two: 1 lets the powers be formed before the host knows
// s; 2^-s is the classic order -- bitwise the same result either way).
constexpr double kCoreTheta = 2.0;
constexpr int kCoreWork = 10;
void launch_core_powers(const double* Z, int m, int batch, bool sym, double pw_alpha,
                        double* work, cudaStream_t s);
void launch_core_eval(const double* Z, const double* nu, const int* flags,
                      double lambda, int m, int batch, int s_scale, bool sym, double pw_alpha,
                      double* work, double* C, int* oflag, cudaStream_t s);

// ---------------------------------------------------------------- spectrum
// NEXT-3 (k_spectrum.cu): k smallest eigenvalues of exp(lambda W~) per cloud.
// Workspaces: W batch*r*r, P/diag/off/mu batch*r doubles, bar 2 uints,
// out batch*k doubles (device).
int spectrum_group(int r);
cudaError_t launch_spectrum(const double* G, const double* nu, int m, int batch, int64_t n,
                            double lambda, int k, double* W, double* P, double* diag,
                            double* off, double* mu, unsigned int* bar, double* out,
                            cudaStream_t s);

// ---------------------------------------------------------------- barycenter
// NEXT-1 (k_sinkhorn.cu): elementwise steps of Alg. 1 on N x k fields.
// Iterates V, W, mu fp64; integrate inputs X / outputs Y fp32; sc: k fp64
// power-of-two input scales; part: bary_blocks(n) x 16 column maxima;
// dpart: bary_blocks(n) partial sums; flag: non-finite iterate.
int bary_blocks(int64_t n);
void launch_bary_init(const float* mu_in, const float* area, int64_t n, int k, float* Mt,
                      double* V, double* mu, double* part, double* sc, int* flag, float* X,
                      cudaStream_t s);
// sc = 2^-e(column max of part), X = fp32(a Z sc)
void launch_bary_input(const float* area, const double* Z, const double* part, int64_t n, int k,
                       double* sc, int* flag, float* X, cudaStream_t s);
void launch_bary_step1(const float* area, const float* Mt, const float* Y, const double* sc,
                       int64_t n, int k, double* W, double* part, cudaStream_t s);
void launch_bary_step2(const float* area, const float* Y, const double* alpha, const double* sc,
                       int64_t n, int k, double* V, double* mu, double* dpart, double* part,
                       double* delta, int* flag, cudaStream_t s);
void launch_bary_finish(const float* area, const double* mu, int64_t n, double* part, double* mass,
                        float* out, cudaStream_t s);

// NEXT-1 fused (k_bary_fused.cu): the whole Alg. 1 loop in one cooperative
// launch for m <= 32, k <= 4, n <= bary_fused_max_points(sms) (each CTA's
// feature rows cached in shared memory).  part: 2 ceil(n/512) x r x k fp64,
// S: r x k (unused), red: 3 ceil(n/512), bar: 2 words (zero), status: [0] non-finite
// flag (zero before), [1] iterations run.
struct Alpha16 {
  double v[16];
};
size_t bary_fused_smem(int m, int k);
int64_t bary_fused_max_points(int sms);
cudaError_t launch_bary_fused(const float4* pts, const float4* omega4, const double* C,
                              const float* mu_in, const float* area, const double* alpha, int m,
                              int k, int64_t n, int max_iter, double tol, double* part, double* S,
                              double* red, unsigned int* bar, int* status, float* out,
                              cudaStream_t s);

// ---------------------------------------------------------------- passes
// S[b][2m][d] fp64 = fixed-order sum of the `chunks` range partials of
// columns [c0, c0+dc) (partial[b][chunk][2m][dc] fp32, interleaved features).
void launch_reduce_S(const float* partial, int m, int batch, int chunks,
                     int d, int c0, int dc, double* S, cudaStream_t s);
void launch_core_apply(const double* C, const double* S, int m, int batch,
                       int d, float* Y, cudaStream_t s);
// Tensor-core pass 2 (k_pass2_tc.cu): dc <= 16 columns per launch.
size_t pass2_tc_smem(int m, int nw, int fuse_dc);
// widest column chunk one pass-2 launch takes (16..64) for m frequencies
int pass2_tc_width(int m);
// part != nullptr: fused a7 (each CTA reduces the pass-1 partials of its
// cloud and forms Y = C^ S; small r, d within one pass-1 chunk).
void launch_pass2_tc(const float4* pts, const float4* omega4, int m, int64_t n, int batch,
                     int sms, const float* Y, const float* F, float* out, int d, int c0, int dc,
                     const float* part, int ranges, const double* C, double* S, float* Yw,
                     cudaStream_t s);

// Narrow fields, d <= 4 (k_small.cu): the whole inference (S partials,
// fixed-order S, Y = C^ S, out = F + Phi Y) in one cooperative launch.
// part: small_partial_elems(...) fp32; S, Y: batch x r x d (plan export);
// bar: kSmallBarWords words zeroed once (self-resetting grid barrier).
constexpr int kSmallBarWords = 34;
size_t small_partial_elems(int m, int64_t n, int batch, int d, int sms);
cudaError_t launch_integrate_small(const float4* pts, const float4* omega4, int m, int64_t n,
                                   int batch, int sms, const float* F, int d, float* out,
                                   const double* C, float* part, double* S, float* Y,
                                   unsigned int* bar, cudaStream_t s);

// Tensor-core pass 1 (k_pass1_tc.cu): partial[b][range][2m][dc].
int pass1_tc_ranges(int m, int64_t n, int batch, int sms);
void launch_pass1_tc(const float* pts16, const float4* omega4, int m, int64_t n, int batch,
                     int sms, int ranges, const float* F, int d, int c0, int dc, float* partial,
                     cudaStream_t s);

}  // namespace rfd
