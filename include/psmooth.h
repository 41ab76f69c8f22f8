/*
 * psmooth.h -- C ABI of libpsmooth.so, the B200 (sm_100a) block-relaxation
 * smoother for the constant-coefficient 7-point stencil.
 *
 * The reference (patchsmooth 0.1.0, pure Python/numpy) has no FFI; its seam is
 * the Python smoother API.  Each entry point below replaces one reference
 * function on the hot path (cited per declaration, paths relative to
 * /root/reference/pkg/src/patchsmooth/).  The Python package
 * paper_1208_1975_b200 keeps the reference's names and signatures and calls
 * these through ctypes; INTEGRATION.md shows the binding.
 *
 * Conventions
 *  - Every function returns 0 on success, a negative psm_status otherwise;
 *    psm_last_error() returns a thread-local message for the last failure.
 *  - All device work is asynchronous and ordered on the caller's stream
 *    (a cudaStream_t passed as void*; NULL = legacy default stream).
 *  - Field memory is owned by the caller (torch).  The library receives raw
 *    device pointers and never frees them.  Plans own only factor tables,
 *    device patch/copy tables, progress flags and reduction workspace.
 *  - Layout: patch buffers are (nx+2)*(ny+2)*(nz+2) doubles, x fastest
 *    (numpy F-order (nx+2,ny+2,nz+2) == torch C-contiguous (nz+2,ny+2,nx+2)),
 *    exactly the reference layout (grid.py:153-182); f is nx*ny*nz, x fastest.
 */
#ifndef PSMOOTH_H
#define PSMOOTH_H

#ifdef __cplusplus
extern "C" {
#endif

enum psm_status {
  PSM_OK = 0,
  PSM_EINVAL = -1,    /* invalid argument (maps to ValueError)        */
  PSM_ESINGULAR = -2, /* block operator singular / not dominant       */
  PSM_ECUDA = -3,     /* CUDA runtime failure (maps to RuntimeError)  */
  PSM_ENOMEM = -4,    /* device or host allocation failed             */
  PSM_EUNSUPPORTED = -5
};

enum psm_block_kind { PSM_BLOCK_LINE = 1, PSM_BLOCK_PLANE = 2, PSM_BLOCK_BOX = 3 };

enum psm_gs_mode {
  PSM_GS_WAVEFRONT = 0, /* deterministic: == lexicographic block GS (runtime.py:164-168) */
  PSM_GS_CHAOTIC = 1    /* in place, no ordering between concurrent lines (runtime.py:185-196) */
};

/* stencil.py:52-68 Stencil7: center > 0, faces in order -x,+x,-y,+y,-z,+z */
typedef struct {
  double center;
  double faces[6];
} psm_stencil;

/* grid.py:153-217 Patch: both padded buffers plus interior f (device pointers) */
typedef struct {
  double* buf[2];
  double* f;
  int nx, ny, nz;
} psm_patch_desc;

/* grid.py:333-352 InterfaceCopy: src interior layer -> dst ghost layer */
typedef struct {
  int src, dst;
  int src_lo[3], dst_lo[3], extent[3];
} psm_copy_desc;

typedef struct psm_factors psm_factors;
typedef struct psm_plan psm_plan;

const char* psm_last_error(void);
int psm_version(void);

/* ---- factor tables (replaces InverseCache.get -> assemble_block_matrix ->
 *      invert_dense, blocklinalg.py:132-151, stencil.py:115-138,
 *      blocklinalg.py:50-87).  One object per block shape; built once,
 *      outside any timed region.  line: extent (nx,1,1); plane: (nx,ny,1). */
int psm_factors_create(int kind, const psm_stencil* st, int nx, int ny, psm_factors** out);
/* Box blocks (ex, ey, ez), every extent in [1, 8] (the paper's cubic blocks,
 * DEFAULT_BLOCK_SIZES analysis.py:38-46): separable exact inverse
 * D Q Lambda^-1 Q D^-1 (per-axis DST-I with a diagonal similarity for
 * non-symmetric faces of one sign); blocks truncated at patch edges use the
 * same tables.  Replaces invert_dense + matvec (blocklinalg.py:50-105) for
 * them.  PSM_EUNSUPPORTED for faces of opposite signs on one axis. */
int psm_factors_create_box(const psm_stencil* st, int ex, int ey, int ez, psm_factors** out);
int psm_factors_destroy(psm_factors* fac);
/* Apply the exact block inverse to `count` contiguous blocks of r (device),
 * writing x (device): the block_update matvec of blocklinalg.py:90-105
 * without the damping.  Used for API-level checks of the inverse. */
int psm_factors_apply(const psm_factors* fac, const double* r, double* x, long long count, void* stream);

/* ---- plans (replaces smoother._Plan, smoother.py:112-124, plus the Level's
 *      adjacency for ghost exchange, grid.py:468-520).  fac[p] is the
 *      factor object for patch p (NULL entries allowed for ghost-only plans). */
int psm_plan_create(const psm_patch_desc* patches, int npatch, const psm_copy_desc* copies, int ncopy,
                    const psm_stencil* st, int kind, psm_factors* const* fac, psm_plan** out);
int psm_plan_destroy(psm_plan* plan);
/* Number of history slots the plan can hold (grown on demand by the calls below). */
int psm_plan_reserve_history(psm_plan* plan, int slots);

/* Level.refresh_ghosts (grid.py:507-517): physical ghosts (grid.py:311-330,
 * ghost = -interior, x then y then z) then interface copies from a snapshot
 * (grid.py:523-547).  active[p] selects the buffer holding u for patch p.
 * `what` ORs psm_ghost_part bits: PSM_GHOST_PHYSICAL alone is
 * fill_physical_ghosts, PSM_GHOST_INTERFACE alone exchange_interface_ghosts;
 * PSM_GHOST_SKIP_X (right after a sweep) fills only the physical ghosts that
 * sweep's epilogue left: none after the one-tile / generic line-Jacobi
 * kernels, the y/z faces after the z-marching line-Jacobi, plane and box
 * Jacobi sweeps (their epilogues write the x faces), all after GS sweeps.
 * The plan tracks which. */
enum psm_ghost_part { PSM_GHOST_PHYSICAL = 1, PSM_GHOST_INTERFACE = 2, PSM_GHOST_SKIP_X = 4, PSM_GHOST_ALL = 3 };
int psm_refresh_ghosts(psm_plan* plan, const unsigned char* active, int what, void* stream);

/* residual_norm partials (smoother.py:96-109): writes the per-plane sums of
 * (f - A u)^2 of every patch into history slot `slot`. */
int psm_residual(psm_plan* plan, const unsigned char* active, int slot, void* stream);

/* One block Jacobi sweep (smoother.py:138-153 without the swap/refresh):
 * v = u + omega * Ainv (f - A u) into the inactive buffer for every line or
 * plane block of every patch; the residual's squared norm (the history entry
 * of the current iterate) goes to slot `slot` (slot < 0: not recorded). */
int psm_jacobi_sweep(psm_plan* plan, const unsigned char* active, double omega, int slot, void* stream);

/* The same sweep restricted to planes [k0, k1) of one patch (line plans):
 * lets a multi-GPU step sweep its boundary planes first and overlap the halo
 * exchange with the interior planes.  Same arithmetic and slot layout. */
int psm_jacobi_sweep_planes(psm_plan* plan, const unsigned char* active, double omega, int slot, int patch, int k0,
                            int k1, void* stream);

/* exchange_interface_ghosts for a copy whose source patch lives on another
 * GPU (grid.py:523-547): copies the interior nx*ny cells of a received
 * contiguous padded plane (px*py doubles, device) into z-ghost plane `side`
 * (0: k = -1, 1: k = nz) of the active buffer of `patch`. */
int psm_halo_unpack(psm_plan* plan, const unsigned char* active, int patch, int side, const double* plane_dev,
                    void* stream);

/* Fused multi-GPU halo over peer memory (z-slabs).  Replaces, for the
 * cross-rank z interfaces of a slab decomposition, the pack / send / receive /
 * unpack of exchange_interface_ghosts (grid.py:523-547) with stores the
 * line-Jacobi sweep itself issues: while it writes plane 0 (nz-1) of a patch
 * it also writes the same values into the top (bottom) ghost plane of the
 * lower (upper) neighbour's matching buffer, mapped from another process with
 * CUDA IPC.  Step protocol per rank (flags are ints in device memory the
 * neighbours write): psm_halo_wait(my flags >= e + s) -> psm_jacobi_sweep ->
 * psm_halo_signal(neighbours' flags := e + s + 1) -> swap -> refresh; the
 * physical ghost fill leaves an interface face's interior alone.
 *
 * psm_ipc_get_handle: 64-byte cudaIpcMemHandle of the allocation holding
 *   `ptr` and the byte offset of `ptr` inside it.
 * psm_ipc_open_handle: map a peer's handle (cached per handle) -> base+offset.
 * psm_plan_set_peer_halo: side 0 = the neighbour below (its nz given), 1 =
 *   above; peer_buf0/1 = its two padded buffers (NULL, NULL clears).  Needs a
 *   line plan on a z-marching nx (PSM_EUNSUPPORTED otherwise).
 * psm_device_pci_bus_id: the current device's PCI bus id ("0000:1b:00.0").
 * psm_peer_access: *ok_out = 1 when the current device can load/store the
 *   memory of the device with that bus id (the same device, or
 *   cudaDeviceCanAccessPeer), 0 otherwise (also when it is not visible to
 *   this process); callers gate the IPC halo on it. */
int psm_device_pci_bus_id(char* out, int len);
int psm_peer_access(const char* pci_bus_id, int* ok_out);
int psm_ipc_get_handle(const void* ptr, void* handle_out, long long* offset_out);
int psm_ipc_open_handle(const void* handle, long long offset, void** ptr_out);
int psm_ipc_close_all(void);
int psm_plan_set_peer_halo(psm_plan* plan, int patch, int side, double* peer_buf0, double* peer_buf1, int peer_nz);
int psm_halo_signal(int* flag_a, int* flag_b, int value, void* stream);
int psm_halo_wait(const int* flags, int n, int value, void* stream);

/* Plane-block solver selection, process-wide: PSM_PLANE_AUTO (default) uses
 * the banded factorised solve (block Thomas along y, Schur complements as
 * short convolutions along x) wherever its truncation bound holds, else the
 * DST-I form; PSM_PLANE_DST forces the DST-I form (cuBLAS DGEMM transforms).
 * Both are exact block inverses to rounding (blocklinalg.py:116-163 replaced).
 * mode < 0 only queries.  Returns the previous mode. */
#define PSM_PLANE_AUTO 0
#define PSM_PLANE_DST 1
int psm_plane_solver(int mode);

/* A whole smooth() step sequence (smoother.py:197-214) as one stream-ordered
 * call: scheme 0 = block Jacobi (steps x: sweep, swap, refresh with x faces
 * skipped), 1 = block GS with mode gs_mode (steps x: sweep, refresh).  With
 * history != 0 the leading refresh and the history[0..steps] residual
 * partials are included (slots 0..steps must be reserved).  The first call
 * with a given (scheme, omega, steps, gs_mode, history, active) runs eagerly;
 * later ones replay a CUDA graph captured on the second call.  `active` is
 * updated in place to the flags after the steps. */
int psm_smooth_steps(psm_plan* plan, unsigned char* active, int scheme, double omega, int steps, int gs_mode,
                     int history, void* stream);

/* Number of kernels this plan has launched so far (benchmark evidence). */
long long psm_plan_launches(const psm_plan* plan);

/* One block Gauss-Seidel sweep in place (smoother.py:156-169, ghosts lagged).
 * mode PSM_GS_WAVEFRONT reproduces the serial lexicographic order exactly;
 * PSM_GS_CHAOTIC runs lines without ordering guarantees. */
int psm_gs_sweep(psm_plan* plan, const unsigned char* active, double omega, int mode, void* stream);

/* Reduce history slots [0, nslots) on the device in a fixed order and copy
 * the per-slot sums of squares (not square-rooted) to host memory. */
int psm_history_sumsq(psm_plan* plan, int nslots, double* out_host, void* stream);
/* Per-plane partial sums of one slot (length = sum of nz over patches), on
 * the device, for cross-GPU gathers: copied into out_dev. */
int psm_history_planes(psm_plan* plan, int slot, double* out_dev, void* stream);
/* Fixed-order (pairwise tree) sum of n doubles on the device -> out_dev[0]. */
int psm_tree_sum(const double* in_dev, long long n, double* out_dev, void* stream);

/* ---- per-block primitives of the reference API (psm_util.cu).  The
 * sweeps above never call these; they back the reference's public building
 * blocks.  All stream-ordered except psm_invert_dense, which synchronises
 * once to report singularity.
 *
 * psm_box_residual: replaces block_residual (stencil.py:93-112) and, with
 *   f == NULL, apply_stencil (stencil.py:71-84): out[x + ex*(y + ey*z)] =
 *   f - A u (or A u) on the interior box [lo, lo+ext) of one padded buffer u
 *   (ghosts read as stored), with the reference's rounding sequence.
 * psm_matvec: replaces matvec (blocklinalg.py:90-105), M column-major n x n,
 *   ascending-column accumulation, bit-identical; with u != NULL it is
 *   block_update (smoother.py:90-93): y = u + omega * (M x).
 * psm_invert_dense: replaces invert_dense (blocklinalg.py:50-87).  w is the
 *   n x 2n column-major matrix [A | I] (overwritten; columns n..2n-1 end as
 *   A^-1), work holds 3n + 4 doubles.  Partial pivoting with the reference's
 *   singularity rule (|pivot| < 1e-14 ||A||_inf -> PSM_ESINGULAR,
 *   *singular_step = 1 + step, -1 for the zero matrix). */
int psm_box_residual(const double* u, const double* f, int nx, int ny, int nz, const int* lo, const int* ext,
                     const psm_stencil* st, double* out, void* stream);
int psm_matvec(const double* m, const double* x, const double* u, double omega, double* y, int n, void* stream);
int psm_invert_dense(double* w, int n, double* work, int* singular_step, double* tiny_pivot, void* stream);

#ifdef __cplusplus
}
#endif
#endif /* PSMOOTH_H */
