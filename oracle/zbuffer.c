/*
 * oracle/zbuffer.c -- TEST INFRASTRUCTURE ONLY (parity checker, never shipped
 * or measured as the product).  Plain-C restatement of the reference render
 * loop so tests and the CPU baseline can run without Cython.
 *
 * Follows pkg/src/nar/_kernels/_native.pyx:56-77 operation for operation
 * (f64 transform in the same association, floor(x + 0.5) pixel snap, f32
 * depth bits << 32 | 32-bit index) and python_impl.py:43-47 for the cull
 * predicate (NaN projections are culled).  Build with -ffp-contract=off
 * (pkg/setup.py:23-25) so no FMA contraction changes the rounding.
 *
 * oracle_zbuffer_render_mt restates the chunked dispatch of
 * _kernels/__init__.py:56-94: contiguous chunks, private EMPTY-filled
 * buffers, unsigned-min merge.
 */
#include <math.h>
#include <pthread.h>
#include <stdint.h>
#include <stdlib.h>
#include <string.h>

#define EMPTY_KEY 0xFFFFFFFFFFFFFFFFull

typedef struct {
  double r[9], c[3], f, cx, cy, nr, fr;
  int w, h;
} cam_t;

static void fold_range(uint64_t* keybuf, const float* pos, int64_t lo, int64_t hi,
                       uint64_t base, const cam_t* k) {
  for (int64_t i = lo; i < hi; ++i) {
    double w0 = (double)pos[3 * i + 0] - k->c[0];
    double w1 = (double)pos[3 * i + 1] - k->c[1];
    double w2 = (double)pos[3 * i + 2] - k->c[2];
    double uz = w0 * k->r[6] + w1 * k->r[7] + w2 * k->r[8];
    if (!(uz > k->nr) || !(uz < k->fr)) continue;
    double ux = w0 * k->r[0] + w1 * k->r[1] + w2 * k->r[2];
    double uy = w0 * k->r[3] + w1 * k->r[4] + w2 * k->r[5];
    double px = floor(k->cx + k->f * (ux / uz) + 0.5);
    double py = floor(k->cy + k->f * (uy / uz) + 0.5);
    if (!(px >= 0.0) || !(px < (double)k->w) || !(py >= 0.0) || !(py < (double)k->h)) continue;
    int64_t pix = (int64_t)py * k->w + (int64_t)px;
    float d32 = (float)uz;
    uint32_t bits;
    memcpy(&bits, &d32, 4);
    uint64_t key = ((uint64_t)bits << 32) | ((base + (uint64_t)i) & 0xFFFFFFFFull);
    if (key < keybuf[pix]) keybuf[pix] = key;
  }
}

static void make_cam(cam_t* k, const double* R, const double* campos, double f, double cx,
                     double cy, double nr, double fr, int w, int h) {
  memcpy(k->r, R, sizeof(k->r));
  memcpy(k->c, campos, sizeof(k->c));
  k->f = f;
  k->cx = cx;
  k->cy = cy;
  k->nr = nr;
  k->fr = fr;
  k->w = w;
  k->h = h;
}

/* Same arguments as _native.zbuffer_accumulate (_native.pyx:32-45). */
void oracle_zbuffer_accumulate(uint64_t* keybuf, const float* positions, int64_t n,
                               uint64_t base_index, const double* R, const double* campos,
                               double f, double cx, double cy, double nr, double fr, int w,
                               int h) {
  cam_t k;
  make_cam(&k, R, campos, f, cx, cy, nr, fr, w, h);
  fold_range(keybuf, positions, 0, n, base_index, &k);
}

typedef struct {
  uint64_t* buf;
  const float* pos;
  int64_t lo, hi;
  const cam_t* k;
} job_t;

static void* run_job(void* arg) {
  job_t* j = (job_t*)arg;
  /* chunk rows are [lo, hi) with base index lo (_kernels/__init__.py:84-87) */
  fold_range(j->buf, j->pos, j->lo, j->hi, 0, j->k);
  return NULL;
}

/* keybuf must be EMPTY-filled by the caller. */
int oracle_zbuffer_render_mt(uint64_t* keybuf, const float* positions, int64_t n,
                             const double* R, const double* campos, double f, double cx,
                             double cy, double nr, double fr, int w, int h, int threads) {
  cam_t k;
  make_cam(&k, R, campos, f, cx, cy, nr, fr, w, h);
  if (threads < 1) threads = 1;
  if (threads > n) threads = n > 0 ? (int)n : 1;
  const int64_t npix = (int64_t)w * h;
  if (threads == 1) {
    fold_range(keybuf, positions, 0, n, 0, &k);
    return 0;
  }
  pthread_t* tid = (pthread_t*)calloc(threads, sizeof(pthread_t));
  job_t* jobs = (job_t*)calloc(threads, sizeof(job_t));
  for (int t = 0; t < threads; ++t) {
    jobs[t].buf = (uint64_t*)malloc((size_t)npix * 8);
    if (!jobs[t].buf) return -1;
    for (int64_t p = 0; p < npix; ++p) jobs[t].buf[p] = EMPTY_KEY;
    /* np.linspace(0, n, nt+1).astype(int64) chunk bounds */
    jobs[t].lo = (int64_t)((double)n * t / threads);
    jobs[t].hi = (int64_t)((double)n * (t + 1) / threads);
    jobs[t].pos = positions;
    jobs[t].k = &k;
    pthread_create(&tid[t], NULL, run_job, &jobs[t]);
  }
  for (int t = 0; t < threads; ++t) pthread_join(tid[t], NULL);
  for (int t = 0; t < threads; ++t) {
    const uint64_t* b = jobs[t].buf;
    for (int64_t p = 0; p < npix; ++p)
      if (b[p] < keybuf[p]) keybuf[p] = b[p];
    free(jobs[t].buf);
  }
  free(jobs);
  free(tid);
  return 0;
}
