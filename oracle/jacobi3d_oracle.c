/*
 * jacobi3d_oracle.c -- the CPU oracle for the Jacobi3D hot path.
 *
 * TEST INFRASTRUCTURE ONLY.  Only tests/, __graft_entry__.smoke() and
 * bench.py's cpu_baseline / --impl reference legs may load this library.
 * The product path (paper_2202_11819_b200/) never links, imports or calls it,
 * and this file shares no code, header, table or constant with it.
 *
 * What it computes (plain definition, written out):
 *   One undecomposed fp64 array U of shape (gz+2, gy+2, gx+2): the owned
 *   cells plus a one-cell ghost shell holding time-invariant Dirichlet values.
 *   One Jacobi iteration (two buffers, pure Jacobi: every read at step n,
 *   PAPER.md L480-484 "two separate buffers ... input and output for the
 *   Jacobi update kernel"; whole-block update after all halos, L105/L215):
 *
 *     V[k][j][i] = ((((((U[k][j][i] + U[k][j][i-1]) + U[k][j][i+1])
 *                     + U[k][j-1][i]) + U[k][j+1][i])
 *                     + U[k-1][j][i]) + U[k+1][j][i]) / 7.0
 *
 *   for every owned (i,j,k); V's ghost shell = U's ghost shell; swap.
 *   The paper never prints the formula (SPEC.md L429 says so); the 7-point
 *   average, its left-to-right summation order self,-x,+x,-y,+y,-z,+z, the
 *   IEEE round-to-nearest division by 7 and the Dirichlet boundary 1.0 /
 *   interior 0.0 default are SPEC.md L388 and L430 (readings R1-R6).
 *   fp64: "Each element of the grid is a double precision
 *   floating point (eight bytes)".
 *
 * Compiled with -O2 -fno-fast-math -ffp-contract=off (no FMA contraction, no
 * reassociation).  OpenMP splits the k loop; cells are independent, so the
 * thread count cannot change a single bit.
 *
 * Index convention: owned coordinates i in [0,gx), j in [0,gy), k in [0,gz);
 * ghosts at -1 and g.  Flat index of (i,j,k) = ((k+1)*(gy+2) + (j+1))*(gx+2) + (i+1).
 */
#include <stdint.h>
#include <string.h>
#include <math.h>
#ifdef _OPENMP
#include <omp.h>
#endif

#define AT(U, i, j, k) (U)[(((int64_t)(k) + 1) * (gy + 2) + ((int64_t)(j) + 1)) * (gx + 2) + ((int64_t)(i) + 1)]

/* splitmix64 (S. Vigna's reference generator, one step from state x).
 * Input generator shared by contract, implemented independently here and in
 * the CUDA init kernel (reading R12). */
static uint64_t oracle_splitmix64(uint64_t x) {
    uint64_t z = x + 0x9E3779B97F4A7C15ULL;
    z = (z ^ (z >> 30)) * 0xBF58476D1CE4E5B9ULL;
    z = (z ^ (z >> 27)) * 0x94D049BB133111EBULL;
    return z ^ (z >> 31);
}

uint64_t oracle_splitmix64_public(uint64_t x) { return oracle_splitmix64(x); }

int oracle_threads(void) {
#ifdef _OPENMP
    return omp_get_max_threads();
#else
    return 1;
#endif
}

void oracle_set_threads(int n) {
#ifdef _OPENMP
    if (n > 0) omp_set_num_threads(n);
#else
    (void)n;
#endif
}

/* Initial state (R6, R7, R12).
 *   kind 0 DEFAULT : owned = 0.0, ghost shell = boundary
 *   kind 1 CONST   : every cell (owned and ghost) = p[0]
 *   kind 2 LINEAR  : every cell = ((p0*i + p1*j) + p2*k) + p3, ghosts at the
 *                    ghost coordinates -1 and g (BASELINE.json north_star:
 *                    "discrete-harmonic (linear) field with matching
 *                    Dirichlet boundaries")
 *   kind 3 HASH    : owned = (splitmix64(splitmix64(seed) ^ gidx) >> 11) * 2^-53,
 *                    gidx = i + gx*(j + gy*k); ghost shell = boundary
 */
void oracle_init(int64_t gx, int64_t gy, int64_t gz, int kind, const double *p,
                 uint64_t seed, double boundary, double *U) {
    const uint64_t s = oracle_splitmix64(seed);
    /* planes are independent: OpenMP cannot change any value */
#pragma omp parallel for schedule(static)
    for (int64_t k = -1; k <= gz; ++k)
        for (int64_t j = -1; j <= gy; ++j)
            for (int64_t i = -1; i <= gx; ++i) {
                const int ghost = (i < 0 || i >= gx || j < 0 || j >= gy || k < 0 || k >= gz);
                double v;
                switch (kind) {
                case 1: v = p[0]; break;
                case 2: {
                    double a = p[0] * (double)i;
                    double b = p[1] * (double)j;
                    double c = p[2] * (double)k;
                    v = ((a + b) + c) + p[3];
                    break;
                }
                case 3:
                    if (ghost) v = boundary;
                    else {
                        uint64_t gidx = (uint64_t)i + (uint64_t)gx * ((uint64_t)j + (uint64_t)gy * (uint64_t)k);
                        v = (double)(oracle_splitmix64(s ^ gidx) >> 11) * 0x1p-53;
                    }
                    break;
                default: v = ghost ? boundary : 0.0; break;
                }
                AT(U, i, j, k) = v;
            }
}

/* One Jacobi iteration U -> V (definition above).  V's ghost shell is copied
 * from U so that both buffers hold the time-invariant Dirichlet values. */
void oracle_sweep(int64_t gx, int64_t gy, int64_t gz, const double *U, double *V) {
    const int64_t n = (gx + 2) * (gy + 2) * (gz + 2);
    memcpy(V, U, (size_t)n * sizeof(double)); /* ghost shell (owned cells overwritten below) */
#pragma omp parallel for schedule(static)
    for (int64_t k = 0; k < gz; ++k)
        for (int64_t j = 0; j < gy; ++j)
            for (int64_t i = 0; i < gx; ++i) {
                double s = AT(U, i, j, k);
                s = s + AT(U, i - 1, j, k);
                s = s + AT(U, i + 1, j, k);
                s = s + AT(U, i, j - 1, k);
                s = s + AT(U, i, j + 1, k);
                s = s + AT(U, i, j, k - 1);
                s = s + AT(U, i, j, k + 1);
                AT(V, i, j, k) = s / 7.0;
            }
}

/* Sweep without the ghost-shell copy: for timing (cpu_baseline) where both
 * buffers were initialised identically, this is bit-identical to oracle_sweep. */
void oracle_sweep_owned(int64_t gx, int64_t gy, int64_t gz, const double *U, double *V) {
#pragma omp parallel for schedule(static)
    for (int64_t k = 0; k < gz; ++k)
        for (int64_t j = 0; j < gy; ++j)
            for (int64_t i = 0; i < gx; ++i) {
                double s = AT(U, i, j, k);
                s = s + AT(U, i - 1, j, k);
                s = s + AT(U, i + 1, j, k);
                s = s + AT(U, i, j - 1, k);
                s = s + AT(U, i, j + 1, k);
                s = s + AT(U, i, j, k - 1);
                s = s + AT(U, i, j, k + 1);
                AT(V, i, j, k) = s / 7.0;
            }
}

/* n iterations starting from A; B is scratch.  Returns 0 if the result is in
 * A, 1 if it is in B (the caller's buffers alternate exactly like the
 * paper's two GPU buffers). */
int oracle_run(int64_t gx, int64_t gy, int64_t gz, double *A, double *B, int64_t n) {
    double *u = A, *v = B;
    for (int64_t it = 0; it < n; ++it) {
        oracle_sweep(gx, gy, gz, u, v);
        double *t = u; u = v; v = t;
    }
    return (u == A) ? 0 : 1;
}

/* Order-independent checksum over owned cells (R15):
 *   sum_{owned} splitmix64(bits(u) ^ splitmix64(gidx))  mod 2^64. */
uint64_t oracle_checksum(int64_t gx, int64_t gy, int64_t gz, const double *U) {
    uint64_t total = 0;
#pragma omp parallel for schedule(static) reduction(+ : total)
    for (int64_t k = 0; k < gz; ++k)
        for (int64_t j = 0; j < gy; ++j)
            for (int64_t i = 0; i < gx; ++i) {
                uint64_t bits;
                double v = AT(U, i, j, k);
                memcpy(&bits, &v, sizeof bits);
                uint64_t gidx = (uint64_t)i + (uint64_t)gx * ((uint64_t)j + (uint64_t)gy * (uint64_t)k);
                total += oracle_splitmix64(bits ^ oracle_splitmix64(gidx));
            }
    return total;
}

/* Residual (R11): max over owned cells of |U - Uprev| (L-infinity
 * norm of the last iteration's change).  Exact, order independent.  A NaN
 * change (a NaN cell, or inf - inf) makes the norm NaN: a comparison-based
 * max would silently skip it (R11, NaN policy). */
double oracle_residual(int64_t gx, int64_t gy, int64_t gz, const double *U, const double *Uprev) {
    double m = 0.0;
    int any_nan = 0;
#pragma omp parallel for schedule(static) reduction(max : m) reduction(| : any_nan)
    for (int64_t k = 0; k < gz; ++k)
        for (int64_t j = 0; j < gy; ++j)
            for (int64_t i = 0; i < gx; ++i) {
                double d = fabs(AT(U, i, j, k) - AT(Uprev, i, j, k));
                if (d != d) any_nan = 1;
                else if (d > m) m = d;
            }
    return any_nan ? (double)NAN : m;
}
