/*
 * seq_oracle.c — sequential topological oracle over the interval CSR.
 * TEST INFRASTRUCTURE ONLY (see oracle/__init__.py).
 *
 * Restates, in plain C, the "sequential topological execution oracle"
 * for the token definition of oracle/tokens.py: nodes are
 * executed one at a time in a topological order; each folds its
 * predecessors' 32-bit terms term(u) = mix64(tok[u] ^ mix64(u + G3)) >> 32
 * into an exact sum (SPEC.md:530-531 fold, builder definition).  It shares no code with the CUDA executor and is an
 * independent restatement of oracle/taskbench_np.py.
 *
 * Build: oracle/Makefile  ->  oracle/_build/liboracle.so
 */
#include <stdint.h>
#include <stdlib.h>

#define G1 0x9E3779B97F4A7C15ull
#define G2 0xD1B54A32D192ED03ull
#define G3 0x8CB92BA72F3D8DD7ull
#define LCG_A 6364136223846793005ull
#define LCG_C 1442695040888963407ull

static inline uint64_t mix64(uint64_t z) {
  z = (z ^ (z >> 30)) * 0xBF58476D1CE4E5B9ull;
  z = (z ^ (z >> 27)) * 0x94D049BB133111EBull;
  return z ^ (z >> 31);
}

/* LCG^n as an affine map (A, C): binary exponentiation of composition. */
static void affine_pow(uint32_t n, uint64_t* A, uint64_t* Cc) {
  uint64_t ra = 1, rc = 0, ba = LCG_A, bc = LCG_C;
  while (n) {
    if (n & 1u) { rc = ba * rc + bc; ra = ba * ra; }
    bc = ba * bc + bc;
    ba = ba * ba;
    n >>= 1;
  }
  *A = ra;
  *Cc = rc;
}

/* The literal loop, for the timed CPU run of COMPUTE bodies. */
uint64_t td_oracle_compute_loop(uint64_t h, uint32_t iters) {
  uint64_t r = 0;
  for (int l = 0; l < 64; ++l) {
    uint64_t x = mix64(h ^ ((uint64_t)(l + 1) * G2));
    for (uint32_t i = 0; i < iters; ++i) x = LCG_A * x + LCG_C;
    r ^= x;
  }
  return r;
}

/*
 * Returns 0 on success, -1 on a bad order (a predecessor not yet executed),
 * -2 on a bad interval.  order == NULL means id order.  literal_loop != 0 runs
 * COMPUTE bodies with the real loop instead of the affine shortcut.
 */
int td_oracle_run(int64_t n, const int64_t* pred_ptr, const int32_t* pred_iv,
                  const uint8_t* kind, const uint32_t* arg, const int64_t* order,
                  uint64_t seed, int literal_loop, uint64_t* tok) {
  uint8_t* done = (uint8_t*)calloc((size_t)(n > 0 ? n : 1), 1);
  if (!done) return -3;
  uint32_t cached_n = 0xFFFFFFFFu;
  uint64_t cA = 1, cC = 0;
  int rc = 0;
  for (int64_t i = 0; i < n && rc == 0; ++i) {
    const int64_t v = order ? order[i] : i;
    uint64_t acc = 0;
    for (int64_t k = pred_ptr[v]; k < pred_ptr[v + 1]; ++k) {
      const int32_t lo = pred_iv[2 * k], hi = pred_iv[2 * k + 1];
      if (lo < 0 || hi < lo || hi >= n) { rc = -2; break; }
      for (int32_t u = lo; u <= hi; ++u) {
        if (!done[u]) { rc = -1; break; }
        acc += mix64(tok[u] ^ mix64((uint64_t)u + G3)) >> 32;
      }
      if (rc) break;
    }
    if (rc) break;
    const uint64_t h0 = mix64(seed ^ mix64((uint64_t)v + G1));
    const uint64_t h = mix64(h0 ^ acc);
    uint64_t r = 0;
    if (kind && kind[v] == 2) {
      const uint32_t it = arg ? arg[v] : 0;
      if (literal_loop) {
        r = td_oracle_compute_loop(h, it);
      } else {
        if (it != cached_n) { affine_pow(it, &cA, &cC); cached_n = it; }
        for (int l = 0; l < 64; ++l) r ^= cA * mix64(h ^ ((uint64_t)(l + 1) * G2)) + cC;
      }
    }
    tok[v] = h ^ r;
    done[v] = 1;
  }
  free(done);
  return rc;
}
