/*
 * sfw_b200.h -- C ABI of the B200-native S-fraction ROM path (libsfw_b200.so).
 *
 * The reference (`sfwave`, pure Python) has no FFI; its drop-in boundary is
 * the Python API re-exported in pkg/src/sfwave/__init__.py:33-43.  Each entry
 * point below replaces one reference call; the Python mirror in
 * paper_1406_6923_b200/ binds them with ctypes.
 *
 * Conventions
 *   - plain C types only; pointers documented as HOST or DEVICE.
 *   - every call returns 0 on success or a negative SFW_E* code; a message is
 *     written to the caller's errbuf (if non-NULL) and is also retrievable with
 *     sfw_last_error().  Codes map onto the reference exception taxonomy
 *     (errors.py:11-41): SFW_ECONFIG -> ConfigError, SFW_ENUMERICAL ->
 *     NumericalError, SFW_EINSTABLE -> InstabilityError, SFW_EPROTOCOL ->
 *     ProtocolError, SFW_ECUDA -> a CUDA runtime failure (no fallback exists).
 *   - all arithmetic is IEEE fp64; results are bitwise deterministic run to run
 *     (fixed-order reductions, no floating-point atomics) as the reference
 *     requires (test_stepper.py:308-322, test_acceptance.py:451-484).
 */
#ifndef SFW_B200_H
#define SFW_B200_H

#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define SFW_OK 0
#define SFW_ECONFIG -1
#define SFW_ENUMERICAL -2
#define SFW_EINSTABLE -3
#define SFW_EPROTOCOL -4
#define SFW_ECUDA -5

/* Last error message of the calling thread ("" if none). */
const char* sfw_last_error(void);

/* Number of SMs / device name of the current CUDA device; <0 if no device. */
int sfw_device_info(int* n_sm, char* name, int name_len);

/* ------------------------------------------------------------------------- */
/* Stage 1: off-line ROM build, batched over subdomains.                      */
/* Replaces sfwave.rom.build_subdomain_model (rom.py:359-434) called once per   */
/* subdomain by sim.run_offline (sim.py:318-330):                              */
/*   SubdomainOperator.matrix (grid.py:415-458)  -> a stencil from c, mu, h     */
/*   subdomain_inputs (rom.py:45-86)             -> face basis kernel          */
/*   _shifted_solver + build_krylov_basis (rom.py:89-174) -> PCG + CGS2/CholQR2 */
/*   truncation (rom.py:375-403), project_reduced (rom.py:177-182)             */
/*   block_lanczos (rom.py:185-262), sfraction_transform (rom.py:265-316)      */
/* ------------------------------------------------------------------------- */

typedef struct sfw_rom_desc {
    int n_sub;             /* subdomains in this call                                          */
    int p[3];              /* nodes per axis of every subdomain (the reference's op.shape)     */
    double h[3];           /* grid spacing per axis (op.spacing)                               */
    int m, n;              /* modes per face (a perfect square), Krylov depth (rom.n)          */
    double shift;          /* shift s of the shifted-inverse Krylov space (rom.py:89-116)      */
    const double* c;       /* HOST [n_sub][p0*p1*p2] sound speed on the subdomain's nodes      */
    const int* nbr_mask;   /* HOST [n_sub] bit f set when face f is shared (op.neighbors)      */
    int n_rows;            /* node rows of V Q to return (sources / receivers)                 */
    const int* row_sub;    /* HOST [n_rows] subdomain index of each row                        */
    const int* row_node;   /* HOST [n_rows] local node index                                   */
    int full_basis;        /* 1: also return the full N x K basis V Q                          */
    int out_on_device;     /* 1: gammas / gamma_hats / scales are DEVICE pointers              */
    int batch;             /* subdomains per internal batch (0 = fit 45% of free HBM)         */
} sfw_rom_desc;

typedef struct sfw_rom_out {
    int* layers;           /* HOST [n_sub] kept chain layers (complete w-blocks, rom.py:375-403) */
    int* flags;            /* HOST [n_sub] bit0 deflated, bit1 truncated                      */
    int* status;           /* HOST [n_sub] 0 ok, else the failing stage (NumericalError)     */
    double* gammas;        /* [n_sub][n+1][w][w] Gamma_j (HOST, or DEVICE if out_on_device)   */
    double* gamma_hats;    /* same layout, Gamma-hat_j                                        */
    double* scales;        /* same layout, G_j                                                */
    double* tdiag;         /* HOST [n_sub][n+1][w][w] Lanczos A_j, or NULL                    */
    double* toff;          /* HOST [n_sub][n][w][w] Lanczos B_j (upper triangular), or NULL  */
    double* basis_rows;    /* HOST [n_rows][K] rows of V Q, or NULL                           */
    double* basis;         /* HOST [n_sub][K][N] (column-major N x K) V Q, or NULL            */
    double* stats;         /* HOST [16]: seconds per stage, max PCG iterations, batch, wall  */
} sfw_rom_out;

/* Build the S-fraction chains of n_sub subdomains (SURVEY 8b sfw_rom_build_batch).
 * Per-subdomain failures (dependent depth-1 block, rank loss, cond > 1e12 in the
 * S-fraction recursion, Gamma-hat_1 != I) set status[i] and return SFW_ENUMERICAL
 * after the whole batch ran, as sim.run_offline aggregates them (sim.py:342-350). */
int sfw_rom_build(const sfw_rom_desc* desc, sfw_rom_out* out, char* errbuf, int errlen);

/* Y = A X with the build's stencil form of the subdomain operator (A = -C S C, grid.py:415-458)
 * for n_sub subdomains of one shape: c HOST [n_sub][N], X / Y HOST [n_sub][ncols][N].  Lets the
 * caller check an explicit SubdomainOperator.matrix against what the GPU build factors. */
int sfw_subdomain_apply(int n_sub, const int* p, const double* h, const double* c, const int* nbr_mask,
                        int ncols, const double* X, double* Y, char* errbuf, int errlen);

/* project_state (rom.py:437-447): out (K) = blockdiag(G_j) (V Q)^T x for a node-space
 * field x (N).  state_to_nodes (rom.py:450-459): out (N) = V Q blockdiag(G_j^-1) u.
 * basis: HOST N x K row-major (SubdomainModel.basis), scales: HOST L x w x w, K = L w. */
int sfw_project_state(int N, int L, int w, const double* basis, const double* scales, const double* x,
                      double* out, char* errbuf, int errlen);
int sfw_state_to_nodes(int N, int L, int w, const double* basis, const double* scales, const double* u,
                       double* out, char* errbuf, int errlen);

/* ------------------------------------------------------------------------- */
/* Stage 2: coupled leapfrog stepping.                                         */
/* Replaces sfwave.stepper.CoupledStepper (stepper.py:144-449):               */
/*   __init__ + _pair_interfaces (stepper.py:147-220)  -> sfw_step_create      */
/*   initialize (stepper.py:325-360)                   -> sfw_step_init        */
/*   advance / run / _probe_row (stepper.py:362-415)   -> sfw_step_run         */
/*   u_curr / u_prev attributes                        -> sfw_step_get_state   */
/*   close / __exit__ (stepper.py:229-239)             -> sfw_step_destroy     */
/* ------------------------------------------------------------------------- */

typedef struct sfw_stepper sfw_stepper;

typedef struct sfw_step_desc {
    int n_sub;               /* number of subdomains, in the reference's sorted(alpha) order */
    int m;                   /* modes per face (uniform); width w = 6m                        */
    const int* layers;       /* HOST [n_sub] chain layers L_s                                 */
    const int* neighbors;    /* HOST [n_sub*6] neighbour subdomain index per face, -1 = none  */
    /* Chain coefficients, dense row-major w x w blocks, subdomain s at block offset
     * sum_{t<s} L_t: gammas = Gamma_j, gamma_hats = Gamma-hat_j (rom.py:319-356).
     * Pointer kind given by coef_on_device (0 = HOST, 1 = DEVICE).                 */
    const double* gammas;
    const double* gamma_hats;
    const double* scales;    /* G_j, same layout; may be NULL (then energy is unavailable) */
    int coef_on_device;
    double dt;               /* leapfrog step (> 0)                                            */
    /* Sources (stepper.py:47-53 SourceTerm): vector of length L_s*w of subdomain
     * src_sub[i]; superposed in list order as stepper.py:313-321 does.           */
    int n_src;
    const int* src_sub;      /* HOST [n_src] */
    const double* src_vec;   /* HOST concat of the n_src vectors */
    /* Probes (stepper.py:56-61): dense weights of length L_s*w on probe_sub[i]. */
    int n_probe;
    const int* probe_sub;    /* HOST [n_probe] */
    const double* probe_w;   /* HOST concat of the n_probe weight vectors */
} sfw_step_desc;

/* Validate, upload and pack the chain coefficients (symmetric Gamma / Gamma-hat
 * are stored packed: w(w+1)/2 doubles per block), build the interface masses
 * (stepper.py:204-219, computed on the device) and check Gamma-hat_1 = I
 * (stepper.py:182-186).  Returns a handle in *out. */
int sfw_step_create(const sfw_step_desc* desc, sfw_stepper** out, char* errbuf, int errlen);

/* Two-level start (stepper.py:325-360).  u0/v0: HOST concat of L_s*w per
 * subdomain, either may be NULL (zeros).  profile0[i] = source i's profile at
 * t = 0.  row0_out: HOST [n_probe] probe row of U0 (stepper.py:405-406) or NULL. */
int sfw_step_init(sfw_stepper* h, const double* u0, const double* v0,
                  const double* profile0, double* row0_out, char* errbuf, int errlen);

/* Advance n_steps leapfrog steps in ONE persistent kernel launch (one grid-wide
 * split arrive/wait barrier per step; face exchange, source injection and
 * probe extraction fused).  profile: HOST [n_src][n_steps] profile values
 * f_i(t_k), t_k = (steps_done + k) * dt for k = 0..n_steps-1 (stepper.py:367).
 * limits: HOST [n_steps] growth thresholds GROWTH_LIMIT*max(baseline_k,1e-300)
 * (stepper.py:379-389) or NULL to skip the check.
 * rows_out: HOST [n_steps/record_every][n_probe] (probe rows after every
 * record_every-th step, stepper.py:407-411) or NULL.
 * norms_out: HOST [n_steps] |U_k|_2 or NULL.  On instability returns
 * SFW_EINSTABLE and *bad_step = first failing step (1-based, relative). */
int sfw_step_run(sfw_stepper* h, int n_steps, int record_every,
                 const double* profile, const double* limits,
                 double* rows_out, double* norms_out, int* bad_step,
                 char* errbuf, int errlen);

/* Same as sfw_step_run but leaves rows/norms in device memory (for timing with
 * inputs resident in HBM); *kernel_ms = CUDA-event duration of the stepping
 * kernel on the library stream. */
int sfw_step_run_resident(sfw_stepper* h, int n_steps, int record_every,
                          const double* profile, float* kernel_ms, char* errbuf, int errlen);

/* Replace the probe set (stepper.py:391-415 passes probes per run). */
int sfw_step_set_probes(sfw_stepper* h, int n_probe, const int* probe_sub, const double* probe_w,
                        char* errbuf, int errlen);

/* Acceleration of a state (HOST u, HOST acc_out), including the forcing
 * sum_i vec_i * profile0[i] (profile0 may be NULL = no forcing);
 * replaces CoupledStepper._acceleration (stepper.py:251-311). */
int sfw_step_accel(sfw_stepper* h, const double* u, const double* profile0, double* acc_out,
                   char* errbuf, int errlen);

/* Largest eigenvalue of minus the coupled acceleration by power iteration
 * (replaces cfl_estimate_coupled, stepper.py:452-487): x0 = HOST start vector
 * (the reference draws it from numpy default_rng(seed)); the iterate stays in
 * HBM, each iteration is one stepping-kernel pass in acceleration mode plus a
 * fixed-order reduction.  Overwrites the stepper state. */
int sfw_step_power(sfw_stepper* h, const double* x0, double tol, int max_iter,
                   double* lam_out, int* converged, int* iters, char* errbuf, int errlen);

/* Multi-shot mode (BASELINE config 4): S = 32 independent wavefields stepped
 * together, every chain-block product a (w x w)(w x S) DMMA GEMM.  Shot q is the
 * reference's CoupledStepper(models, dt, sources=(shot_q,)).run(...) from rest.
 * shot_sub: HOST [32] source subdomain (-1 = no source); shot_vec: HOST concat
 * of the source vectors (length L*w of shot_sub[q], skipped when -1). */
int sfw_shots_setup(sfw_stepper* h, int n_shots, const int* shot_sub, const double* shot_vec,
                    char* errbuf, int errlen);

/* Run all shots from rest for n_steps in one persistent launch.  profile0: HOST
 * [S] f_q(0); profile: HOST [S][n_steps] f_q(k dt); rows_out: HOST
 * [n_steps/record_every][S][n_probe] or NULL; norms_out: HOST [n_steps][S]
 * |U_q| after each step or NULL; *kernel_ms: CUDA-event time of the launch. */
int sfw_shots_run(sfw_stepper* h, int n_steps, int record_every, const double* profile0,
                  const double* profile, double* rows_out, double* norms_out, float* kernel_ms,
                  char* errbuf, int errlen);

/* State of shot q after the last sfw_shots_run (HOST concat of L_s*w). */
int sfw_shots_state(sfw_stepper* h, int q, double* u_curr, double* u_prev);

/* Algorithmic bytes / flops per step of the multi-shot launch, and bytes streamed. */
int sfw_shots_traffic(sfw_stepper* h, double* alg_bytes, double* alg_flops, double* streamed_bytes);

/* fp32 W-form variant: U_j = G_j W_j turns the chain
 * into the Lanczos block-tridiagonal operator (A_j symmetric, B_j triangular,
 * computed on the device from G_j, Gamma_j) with interface mass 1/2; blocks are
 * fp32 (half the bytes).  Requires scales at create. */
int sfw_wform_setup(sfw_stepper* h, char* errbuf, int errlen);
/* Convert the handle's U-form sources (G^-1 s) and probe weights (G^T p) to W-form.
 * src_vec / probe_w: HOST U-form arrays as passed to create / set_probes;
 * src_norms: HOST [n_src] |G^-1 s| or NULL. */
int sfw_wform_vectors(sfw_stepper* h, const double* src_vec, const double* probe_w, double* src_norms,
                      char* errbuf, int errlen);
/* Two-level start in W-form (u0/v0: HOST U-form or NULL). */
int sfw_wform_init(sfw_stepper* h, const double* u0, const double* v0, const double* profile0,
                   double* row0_out, char* errbuf, int errlen);
/* n_steps fp32 W-form steps; rows are physical probe values (fp64), norms_out |W| per step;
 * *kernel_ms the CUDA-event time of the launches.  limits: HOST [n_steps] growth thresholds on |W|
 * (the detector of stepper.py:379-389 in W-form norms) or NULL: with limits the run is launched in
 * chunks of <= 512 steps whose |W| is checked on the way, and it stops launching at the first
 * failing step (SFW_EINSTABLE, *bad_step 1-based; the state is at most one chunk past it). */
int sfw_wform_run(sfw_stepper* h, int n_steps, int record_every, const double* profile, const double* limits,
                  double* rows_out, double* norms_out, int* bad_step, float* kernel_ms, char* errbuf, int errlen);
/* Current/previous state mapped back to U-form (fp64). */
int sfw_wform_state(sfw_stepper* h, double* u_curr, double* u_prev, char* errbuf, int errlen);
int sfw_wform_traffic(sfw_stepper* h, double* alg_bytes, double* streamed_bytes);
int sfw_wform_destroy(sfw_stepper* h);

/* Interface masses ha (ha + hb)^-1 hb, symmetrised (stepper.py:64-70, 204-210), as the device
 * computed them at create: *n_iface interfaces in _pair_interfaces order (low subdomain
 * ascending, then face), out HOST [n_iface][m][m] (may be NULL to query the count). */
int sfw_step_masses(sfw_stepper* h, int* n_iface, double* out, char* errbuf, int errlen);

/* Copy the current/previous state (HOST concat of L_s*w per subdomain). */
int sfw_step_get_state(sfw_stepper* h, double* u_curr, double* u_prev);
/* Overwrite the current / previous state (HOST concat of L_s*w per subdomain; NULL keeps that
 * level): assignment to the reference's u_curr / u_prev dicts (stepper.py:164-165). */
int sfw_step_set_state(sfw_stepper* h, const double* u_curr, const double* u_prev, char* errbuf, int errlen);

/* Discrete energy (stepper.py:419-449), computed on the device. */
int sfw_step_energy(sfw_stepper* h, double* energy, char* errbuf, int errlen);

/* Byte and flop counts of one stepping launch per step (algorithmic, as in
 * SURVEY.md 8d), and the bytes actually streamed per step by this build. */
int sfw_step_traffic(sfw_stepper* h, double* alg_bytes, double* alg_flops, double* streamed_bytes);

/* Host table of a reference source pulse (sim.py:80-94; 0 = Ricker, 1 = Gaussian derivative)
 * at t_k = (k0 + k) * dt, bit-identical to the Python callables in pulses.py.  Replaces
 * the per-step SourceTerm.profile calls of stepper.py:313-321 on long runs. */
int sfw_pulse_table(int kind, double f_peak, double delay, long long k0, double dt, int n, double* out);

int sfw_step_destroy(sfw_stepper* h);

/* ------------------------------------------------------------------------- */
/* Once-per-run state-space maps (stepper.py:91-141), on the device.           */
/* ------------------------------------------------------------------------- */

/* project_source (stepper.py:91-128): coeff = basis_row * scale (scale =
 * amplitude / c_s), norms[0] = |coeff|, norms[1] = |coeff[:w]| (the caller
 * applies the leak / silence checks), first block zeroed, out_j = G_j coeff_j.
 * scales: HOST L x w x w; basis_row, out: HOST L*w. */
int sfw_source_vector(int L, int w, const double* scales, const double* basis_row, double scale,
                      double* out, double* norms, char* errbuf, int errlen);

/* make_probe (stepper.py:131-141): out_j = solve(G_j^T, basis_row_j) * scale. */
int sfw_probe_weights(int L, int w, const double* scales, const double* basis_row, double scale,
                      double* out, char* errbuf, int errlen);

/* ------------------------------------------------------------------------- */
/* Fine-grid leapfrog reference solver (reference.py:26-157 on the operator of  */
/* grid.py:461-467, the undivided C Lap_h C with mirror closure).  The matrix   */
/* is never stored: rows are rebuilt from c and the per-axis scales in the      */
/* reference's arithmetic, so trajectories match scipy/numpy bit for bit.       */
/* ------------------------------------------------------------------------- */

typedef struct sfw_fdtd sfw_fdtd;

/* grid nx x ny x nz (C order, z fastest); scales[d] = 1 / (1.0 * h_d**2) as
 * grid.py:366 forms it; c: HOST nx*ny*nz sound speed.  Replaces building
 * assemble_global_operator's CSR (grid.py:461-467). */
int sfw_fdtd_create(int nx, int ny, int nz, const double* scales, const double* c, sfw_fdtd** out,
                    char* errbuf, int errlen);
/* y = A x, HOST vectors (the `a @ u` of reference.py:117). */
int sfw_fdtd_apply(sfw_fdtd* h, const double* x, double* y, char* errbuf, int errlen);
/* estimate_lambda_max (reference.py:26-63) from the HOST normalised start
 * vector v0 (numpy default_rng(seed)); *iters < 0: not converged. */
int sfw_fdtd_power(sfw_fdtd* h, const double* v0, double tol, int max_iter, double* lam, int* iters,
                   char* errbuf, int errlen);
/* source_vec nonzeros (node, value), receiver rows, optional damping (HOST n). */
int sfw_fdtd_setup(sfw_fdtd* h, int n_src, const long long* src_idx, const double* src_val, int n_rec,
                   const long long* rec_idx, const double* damping, char* errbuf, int errlen);
/* second-order start (reference.py:123-124); u0 / v0 may be NULL (zeros); f0 = source_fn(0). */
int sfw_fdtd_init(sfw_fdtd* h, double dt, const double* u0, const double* v0, double f0, char* errbuf,
                  int errlen);
/* n_steps steps (reference.py:129-150): ftab[k-1] = source_fn((k-1) dt);
 * norms_out[k-1] = |u_k|^2; rows_out[r][n_rec] every record_every steps. */
int sfw_fdtd_run(sfw_fdtd* h, double dt, int n_steps, const double* ftab, int record_every,
                 double* norms_out, double* rows_out, float* kernel_ms, char* errbuf, int errlen);
int sfw_fdtd_state(sfw_fdtd* h, double* u_curr, double* u_prev, char* errbuf, int errlen);
int sfw_fdtd_destroy(sfw_fdtd* h);

/* ------------------------------------------------------------------------- */
/* Batched reduced transfer maps (ntd.py:101-185, sim.py:703-768 cross-check). */
/* ------------------------------------------------------------------------- */

/* form 0 = ntd_tridiag(diag A, off B, entry E, omega); form 1 = ntd_chain(gammas A,
 * gamma_hats B, omega).  A: [n_models][L][w][w]; B: [n_models][L-1][w][w] (form 0)
 * or [n_models][L][w][w] (form 1); E: [n_models][w][w] (form 0).  One item per
 * (item_model[i], item_omega[i]); out [n_items][w][w] symmetrised maps; status[i]
 * 0 = ok, 2 = singular (the reference raises NumericalError).  HOST arrays. */
int sfw_ntd_batch(int form, int n_models, int L, int w, const double* A, const double* B, const double* E,
                  int n_items, const int* item_model, const double* item_omega, double* out, int* status,
                  char* errbuf, int errlen);

/* Transfer maps of an explicit operator (reference ntd.py:62-115 ntd_full / ntd_reduced):
 * out[k] = sym(F^T (A + omegas[k]^2 I)^-1 F), A given as host CSR (n x n, row_ptr[n] nonzeros),
 * F host [n][w] row-major.  Band LU with partial pivoting (LAPACK dgbtf2/dgbtrs order) on the
 * device, one CTA per frequency.  resid[k] = ||A X + w^2 X - F||_F / ||F||_F (the reference's
 * resonance measure); status[k] = 0, or j+1 for an exactly zero pivot in column j. */
int sfw_ntd_operator(int n, const int* row_ptr, const int* col_idx, const double* vals, int w, const double* F,
                     int n_omega, const double* omegas, double* out, double* resid, int* status, char* errbuf,
                     int errlen);

/* Face inputs F of one subdomain (reference rom.py:55-86 subdomain_inputs): out[c * N + node],
 * N = px*py*pz, c < 6m, built by the ROM pipeline's own face-basis kernel.  nbr_mask bit f is
 * set when face f is shared. */
int sfw_face_inputs(int px, int py, int pz, int m, int nbr_mask, double* out, char* errbuf, int errlen);

#ifdef __cplusplus
}
#endif
#endif /* SFW_B200_H */
