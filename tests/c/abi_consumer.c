/* A plain-C consumer of include/nar_b200.h (no Python, no torch): what a C/C++
 * host program linking libnar_b200.so does.  Reads points + camera from a file,
 * renders them twice -- through the host-parity entry (nar_zbuffer_accumulate)
 * and through the device entries (nar_keybuf_fill, nar_render, nar_resolve for
 * RGB+D) -- and writes both keybufs and the G-buffer for the test to check.
 *
 *   abi_consumer in.bin out.bin      (exit 0 ok, 77 no GPU, 1 error)
 *
 * in.bin : int64 n, int32 W, int32 H, f64 R[9], campos[3], f, cx, cy, near, far,
 *          f32 xyz[n*3], u8 rgb[n*3]
 * out.bin: u64 keybuf_host[W*H], u64 keybuf_dev[W*H], f32 data[H*W*4]
 */
#include <cuda_runtime_api.h>
#include <stdio.h>
#include <stdlib.h>
#include <string.h>

#include "nar_b200.h"

#define CHECK(x)                                                              \
  do {                                                                        \
    int rc_ = (x);                                                            \
    if (rc_ != NAR_OK) {                                                      \
      fprintf(stderr, "%s failed (%d): %s\n", #x, rc_, nar_last_error());     \
      return 1;                                                               \
    }                                                                         \
  } while (0)

static int rd(FILE* f, void* p, size_t n) { return fread(p, 1, n, f) == n ? 0 : -1; }

int main(int argc, char** argv) {
  if (argc != 3) return 1;
  int32_t ndev = 0;
  if (nar_device_count(&ndev) != NAR_OK || ndev == 0) return 77;
  FILE* f = fopen(argv[1], "rb");
  if (!f) return 1;
  int64_t n;
  int32_t W, H;
  double cam_d[17];
  if (rd(f, &n, 8) || rd(f, &W, 4) || rd(f, &H, 4) || rd(f, cam_d, sizeof(cam_d))) return 1;
  float* xyz = (float*)malloc((size_t)n * 12);
  unsigned char* rgb = (unsigned char*)malloc((size_t)n * 3);
  if (rd(f, xyz, (size_t)n * 12) || rd(f, rgb, (size_t)n * 3)) return 1;
  fclose(f);

  nar_camera cam;
  memcpy(cam.R, cam_d, 9 * 8);
  memcpy(cam.campos, cam_d + 9, 3 * 8);
  cam.f = cam_d[12];
  cam.cx = cam_d[13];
  cam.cy = cam_d[14];
  cam.near_ = cam_d[15];
  cam.far_ = cam_d[16];
  cam.width = W;
  cam.height = H;
  const size_t npix = (size_t)W * H;

  /* 1. host-parity twin of the Cython FFI: folds into a caller-owned buffer */
  uint64_t* kb_host = (uint64_t*)malloc(npix * 8);
  for (size_t i = 0; i < npix; ++i) kb_host[i] = NAR_EMPTY_KEY;
  CHECK(nar_zbuffer_accumulate(kb_host, xyz, n, 0, cam.R, cam.campos, cam.f, cam.cx, cam.cy,
                               cam.near_, cam.far_, W, H));

  /* 2. device path */
  uint64_t* d_kb;
  float *d_xyz, *d_data, *d_depth;
  unsigned char *d_rgb, *d_cov;
  int64_t* d_idx;
  if (cudaMalloc((void**)&d_kb, npix * 8) || cudaMalloc((void**)&d_xyz, (size_t)n * 12) ||
      cudaMalloc((void**)&d_rgb, (size_t)n * 3) || cudaMalloc((void**)&d_data, npix * 16) ||
      cudaMalloc((void**)&d_depth, npix * 4) || cudaMalloc((void**)&d_cov, npix) ||
      cudaMalloc((void**)&d_idx, npix * 8))
    return 1;
  cudaMemcpy(d_xyz, xyz, (size_t)n * 12, cudaMemcpyHostToDevice);
  cudaMemcpy(d_rgb, rgb, (size_t)n * 3, cudaMemcpyHostToDevice);
  CHECK(nar_keybuf_fill(d_kb, (int64_t)npix, NAR_EMPTY_KEY, NULL));
  CHECK(nar_render(d_kb, d_xyz, n, 0, &cam, NAR_KEYS_UNSIGNED, NULL));
  uint64_t* kb_dev = (uint64_t*)malloc(npix * 8);
  cudaMemcpy(kb_dev, d_kb, npix * 8, cudaMemcpyDeviceToHost);

  nar_selection sel;
  memset(&sel, 0, sizeof(sel));
  sel.rgb = 1;
  sel.depth = 1;
  sel.rgb_format = NAR_FMT_U8;
  sel.rgb_arity = 3;
  sel.velocity_scale = 1.0;
  nar_segment seg;
  memset(&seg, 0, sizeof(seg));
  seg.begin = 0;
  seg.count = n;
  seg.positions = d_xyz;
  seg.rgb = d_rgb;
  nar_resolve_out out;
  memset(&out, 0, sizeof(out));
  out.data = d_data;
  out.coverage = d_cov;
  out.index_plane = d_idx;
  out.depth = d_depth;
  out.clear_keybuf = 1;
  CHECK(nar_resolve(d_kb, &cam, NAR_KEYS_UNSIGNED, &sel, &seg, 1, &out, NULL));
  float* data = (float*)malloc(npix * 16);
  cudaMemcpy(data, d_data, npix * 16, cudaMemcpyDeviceToHost);
  if (cudaDeviceSynchronize() != cudaSuccess) return 1;

  FILE* o = fopen(argv[2], "wb");
  if (!o) return 1;
  fwrite(kb_host, 8, npix, o);
  fwrite(kb_dev, 8, npix, o);
  fwrite(data, 16, npix, o);
  fclose(o);
  printf("ok %s\n", nar_version());
  return 0;
}
