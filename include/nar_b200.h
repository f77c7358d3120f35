/*
 * nar_b200.h -- C ABI of the B200-native NAR hot path (MSR render + resolve,
 * min-composite helpers, gated U-Net forward).
 *
 * Every entry point takes plain pointers and sizes, returns an int status
 * (NAR_OK == 0) and never throws across the ABI; the message of the last
 * failure on the calling thread is available from nar_last_error().
 * Pointers documented as "device" must be CUDA device (or managed) memory;
 * "host" pointers may be pageable or pinned.  `stream` is a cudaStream_t
 * passed as void* (NULL = legacy default stream).
 *
 * Reference interfaces replaced (paths relative to the reference package
 * root pkg/src/nar/):
 *   nar_zbuffer_accumulate  <- _kernels/_native.pyx:32-77 `zbuffer_accumulate`
 *                              (twin: _kernels/python_impl.py:17-53)
 *   nar_render / nar_render_host
 *                           <- _kernels/__init__.py:56-94 `zbuffer_render`
 *                              (chunked private buffers + np.minimum.reduce)
 *   nar_resolve             <- msr/rasterizer.py:140-178 (decode + channel fill),
 *                              msr/velocity.py:17-48, geometry/camera.py:154-166
 *   nar_unet_*              <- neural/model.py:135-204 (`conv1x1_head`,
 *                              `build_pyramid`, `gated_conv`, `unet_forward`,
 *                              `forward`), neural/autodiff.py:186-288
 *   nar_morton_keys         <- geometry/morton.py:23-37 `morton_keys`
 *   nar_splat_blend         <- _kernels/__init__.py:97-166 `splat_blend_image`
 *                              (native path: CSR tile binning +
 *                              _kernels/_native.pyx:80-159 `splat_blend_tiles`)
 */
#ifndef NAR_B200_H
#define NAR_B200_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

/* ---- status codes (mapped to nar errors by the Python shim) ---------------- */
#define NAR_OK 0
#define NAR_ERR_INVALID 1 /* bad argument            -> ValueError          */
#define NAR_ERR_CUDA 2    /* CUDA runtime failure    -> RuntimeError        */
#define NAR_ERR_CONFIG 3  /* inconsistent selection  -> ConfigurationError  */
#define NAR_ERR_NOMEM 4   /* allocation failure      -> MemoryError         */

/* python_impl.py:13 EMPTY_KEY */
#define NAR_EMPTY_KEY 0xFFFFFFFFFFFFFFFFull
/* Keys of the "signed" domain are key ^ NAR_SIGN_FLIP: unsigned order equals
 * int64 order there, so an int64 MIN all-reduce composites them exactly. */
#define NAR_SIGN_FLIP 0x8000000000000000ull

#define NAR_KEYS_UNSIGNED 0
#define NAR_KEYS_SIGNED 1

#define NAR_MAX_SEGMENTS 8 /* point buffers rendered into one keybuf      */
#define NAR_MAX_SCALARS 8  /* pointcloud.py:18 MAX_STREAMS                */
#define NAR_MAX_CHANNELS 16 /* rasterizer.py:21 MAX_CHANNELS              */

#define NAR_FMT_U8 0
#define NAR_FMT_F32 1

/* Pinhole camera as consumed by the render kernel (camera.py:26-72). */
typedef struct nar_camera {
  double R[9];      /* world->camera rotation, row major, rows right/down/forward */
  double campos[3]; /* camera position in world space                             */
  double f, cx, cy; /* focal length in px, principal point                        */
  double near_, far_;
  int32_t width, height;
} nar_camera;

/* ---- library ----------------------------------------------------------------- */
const char* nar_version(void);
const char* nar_last_error(void);
int nar_device_count(int32_t* count);
/* Number of kernels this library has launched so far (process-wide). */
uint64_t nar_launch_count(void);
/* Host memory helpers (pinned allocations make H2D copies true async DMA). */
int nar_host_alloc(void** ptr, size_t bytes);
int nar_host_free(void* ptr);
/* Device address of mapped pinned host memory (NAR_ERR_INVALID for pageable or
 * device memory).  Kernels read through it over PCIe ("zero-copy"): the
 * resolve gathers only the winners' attributes instead of uploading streams. */
int nar_host_mapped_pointer(const void* host, void** dev);
/* Page-lock (and map) an existing pageable host range in place, so later
 * copies from it are async DMA and kernels can read it zero-copy; undone by
 * nar_host_unregister.  NAR_ERR_INVALID if (part of) the range is already
 * registered or the pages cannot be locked.  The Python shim registers the
 * numpy arrays of a host PointCloud on first use (msr.rasterize) and
 * unregisters them when the arrays are released. */
int nar_host_register(void* host, size_t bytes);
int nar_host_unregister(void* host);

/* ---- host-parity twin of the reference FFI --------------------------------------
 * Same arguments and semantics as `_native.zbuffer_accumulate` (_native.pyx:32):
 * projects positions[n][3] (host f32, C-contiguous AoS), folds
 * key = f32bits((float)uz) << 32 | ((base_index + i) & 0xFFFFFFFF) into
 * keybuf[width*height] (host u64, in place) by unsigned minimum.
 * Non-finite projections are culled as in python_impl.py:43-47. */
int nar_zbuffer_accumulate(uint64_t* keybuf, const float* positions, int64_t n,
                           uint64_t base_index, const double* R, const double* campos,
                           double f, double cx, double cy, double near_, double far_,
                           int32_t width, int32_t height);

/* ---- device-resident render ----------------------------------------------------- */
/* keybuf_dev[npix] = value (EMPTY_KEY, or EMPTY_KEY ^ SIGN_FLIP in the signed domain). */
int nar_keybuf_fill(uint64_t* keybuf_dev, int64_t npix, uint64_t value, void* stream);
/* Render n device-resident points (f32 AoS) into keybuf_dev.  key_domain selects
 * unsigned keys (reference layout) or sign-flipped keys (NCCL int64 MIN). */
int nar_render(uint64_t* keybuf_dev, const float* positions_dev, int64_t n,
               uint64_t base_index, const nar_camera* cam, int32_t key_domain,
               void* stream);
/* Hierarchical-Z render: as nar_render, but the points are split into passes
 * and every pass after the first rejects points behind the coarse max depth
 * (2^k x 2^k pixel blocks) rebuilt from the keybuf into hiz_scratch_dev
 * (nar_hiz_scratch_bytes).  keybuf_has_frame != 0 means the keybuf already
 * holds keys of this frame (e.g. other point buffers rendered before), so
 * the first pass may use the coarse test too.  Results are identical to
 * nar_render: the test only skips points that cannot win. */
int nar_hiz_scratch_bytes(int32_t width, int32_t height, size_t* bytes);
int nar_render_hiz(uint64_t* keybuf_dev, uint16_t* hiz_scratch_dev, const float* positions_dev,
                   int64_t n, uint64_t base_index, const nar_camera* cam, int32_t key_domain,
                   int32_t keybuf_has_frame, void* stream);
/* Same as nar_render for host-resident points: streams them through device
 * chunk buffers, overlapping the H2D copy of chunk k+1 with the render of k. */
int nar_render_host(uint64_t* keybuf_dev, const float* positions_host, int64_t n,
                    uint64_t base_index, const nar_camera* cam, int32_t key_domain,
                    void* stream);

/* ---- preprocessing: Morton order (geometry/morton.py:9-46) --------------------------
 * keys_dev[i] = 63-bit z-order key of positions_dev[i] quantised to 21 bits per
 * axis over the box [lo, hi] (f64, bit-identical to the reference); a stable
 * sort by key gives the reference's morton_reorder permutation. */
int nar_morton_keys(const float* positions_dev, int64_t n, const double* lo, const double* hi,
                    uint64_t* keys_dev, void* stream);

/* ---- Gaussian splat blending (ground-truth renderer, gsplat/renderer.py) ------------
 * Front-to-back alpha blending of n depth-sorted 2D Gaussians into rgb_out
 * (height, width, 3) f64, all device pointers: mu (n,2), inv_abc (n,3) inverse
 * covariance (a, b, c), boxes (n,4) int32 image-clipped (x0, x1, y0, y1), color
 * (n,3), opacity (n,).  Splats are binned to tile_size^2 tiles and blended in
 * id order per pixel until the transmittance drops below 1/255 (the
 * reference's native semantics; f64, exp() within an ulp of libm).  Returns
 * after the binning's size read-back; the blend itself is stream-ordered. */
int nar_splat_blend(const double* mu, const double* inv_abc, const int32_t* boxes,
                    const double* color, const double* opacity, int64_t n, int32_t width,
                    int32_t height, int32_t tile_size, double* rgb_out, void* stream);

/* ---- resolve ---------------------------------------------------------------------- */
/* One contiguous point buffer (a "data stream" of the multi-stream config):
 * global indices [begin, begin+count) live in rows [0, count) of these arrays. */
typedef struct nar_segment {
  int64_t begin;
  int64_t count;
  const float* positions;                 /* (count,3) f32, needed for vel2d */
  const void* rgb;                        /* (count, rgb_arity)              */
  const void* velocity;                   /* (count, vel_arity)              */
  const void* scalars[NAR_MAX_SCALARS];   /* (count, scalar_arity[k])        */
} nar_segment;

/* Channel selection, rasterizer.py:27-72 StreamSelection (channel order is
 * r,g,b | d | v2x,v2y,v2t,v2m | v3x,v3y,v3z,v3m | scalars | coverage). */
typedef struct nar_selection {
  int32_t rgb, depth, vel2d, vel3d, coverage_channel;
  int32_t rgb_format, rgb_arity;
  int32_t vel_format, vel_arity;
  int32_t n_scalars;
  int32_t scalar_format[NAR_MAX_SCALARS];
  int32_t scalar_arity[NAR_MAX_SCALARS];
  double velocity_scale;
} nar_selection;

typedef struct nar_resolve_out {
  float* data;          /* (data_h, data_w, C) f32 FeatureImage.data, or NULL.
                           data_h >= H, data_w >= W: pixels outside (H, W) are
                           written as zeros, i.e. the buffer is already the
                           zero-padded CNN input of model.py:207           */
  int32_t data_h, data_w; /* 0 = (H, W)                                    */
  uint8_t* coverage;    /* (H, W) u8, or NULL                              */
  int64_t* index_plane; /* (H, W) i64, -1 = background, or NULL            */
  float* depth;         /* (H, W) f32 view depth, 0 = background, or NULL  */
  int32_t owner_only;   /* 1: winners outside the local segments give zero
                           channels (sharded resolve before an int32 SUM
                           reduce of the channel bit patterns)             */
  int32_t clear_keybuf; /* 1: reset keybuf to EMPTY for the next frame    */
} nar_resolve_out;

int nar_resolve(uint64_t* keybuf_dev, const nar_camera* cam, int32_t key_domain,
                const nar_selection* sel, const nar_segment* segments,
                int32_t n_segments, const nar_resolve_out* out, void* stream);
/* Fused composite + resolve over peer memory (multi-GPU): the
 * key of each pixel is the minimum over n_keybufs keybufs -- the ranks' own
 * buffers mapped into this process (CUDA IPC / symmetric memory, NVLink loads)
 * -- and only rows [row_begin, row_end) of the (padded) output are resolved,
 * so every rank resolves its slice of the frame with no NCCL all-reduce.  The
 * segment table lists every rank's shard (peer attribute pointers), so winners
 * are gathered from their owner's memory.  clear_keybuf resets the slice in
 * all n_keybufs buffers.  Identical results to nar_resolve on the min-composited
 * keybuf. */
int nar_resolve_peers(const uint64_t* const* keybufs, int32_t n_keybufs, int32_t row_begin,
                      int32_t row_end, const nar_camera* cam, int32_t key_domain,
                      const nar_selection* sel, const nar_segment* segments, int32_t n_segments,
                      const nar_resolve_out* out, void* stream);

/* Host-gathered attributes (an extension of the resolve, no reference counterpart):
 * for a cloud whose rgb stream lives in host memory, nar_host_gather_rgb reads the
 * frame's keys (a host copy of the keybuf, width*height words) and writes, per image
 * pixel, the winner's rgb bytes c0 | c1 << 8 | c2 << 16 (0 where the pixel is empty
 * or the winner lies outside [begin, begin + count)) on a pool of host threads
 * (NAR_HOST_THREADS); nar_resolve_pixrgb is nar_resolve with the rgb taken from that
 * per-pixel array (device copy) -- RGB+D u8 selections only, identical results --
 * for the padded-output rows [row_begin, row_end) (row_end < 0: to the last row), so
 * a frame can be gathered, resolved and copied down in bands that overlap. */
int nar_host_gather_rgb(const uint64_t* keys, int64_t npix, int32_t key_domain,
                        const uint8_t* rgb, int32_t arity, uint64_t begin, int64_t count,
                        uint32_t* out);
int nar_resolve_pixrgb(uint64_t* keybuf_dev, int32_t row_begin, int32_t row_end,
                       const nar_camera* cam, int32_t key_domain, const nar_selection* sel,
                       const nar_segment* segments, int32_t n_segments, const nar_resolve_out* out,
                       const uint32_t* pix_rgb_dev, void* stream);

/* ---- gated U-Net (neural/model.py) -------------------------------------------------- */
/* Standalone ops of the network (model.py:135-163), f32 device tensors in/out.
 * nar_head_pyramid: the 1x1 descriptor head y = x W + b (use_head != 0; W (C,C)
 * and b (C,) device f32) and the pyramid of 2x2 averages; out[k] is
 * (H >> k, W >> k, C) f32 for k < levels (H, W divisible by 2^(levels-1)).
 * nar_gated_conv: elu(conv3x3(x, f_w) + f_b) * sigmoid(conv3x3(x, g_w) + g_b),
 * "same" zero padding, HWIO f32 weights on the HOST (packed to bf16 per call),
 * bf16 tensor-core math with f32 accumulation; blocks until done. */
int nar_head_pyramid(const float* in, int32_t H, int32_t W, int32_t C, const float* head_w,
                     const float* head_b, int32_t use_head, int32_t levels, float* const* out,
                     void* stream);
int nar_gated_conv(const float* in, int32_t H, int32_t W, int32_t cin, const float* f_w,
                   const float* f_b, const float* g_w, const float* g_b, int32_t cout, float* out,
                   void* stream);

typedef struct nar_unet_config {
  int32_t input_channels, levels, base_channels, channel_multiplier;
  int32_t max_channels, output_channels, use_descriptor_head;
} nar_unet_config;

typedef struct nar_unet nar_unet; /* opaque: packed bf16 weights + plan */

int nar_unet_create(const nar_unet_config* cfg, nar_unet** out);
int nar_unet_destroy(nar_unet* net);
/* Upload one f32 parameter from host memory, named as in model.py:70-100
 * ("head.w", "enc0a.f_w", ..., "out.b"); conv weights are HWIO. */
int nar_unet_set_param(nar_unet* net, const char* name, const float* host_data,
                       int64_t numel);
/* Device workspace needed by nar_unet_forward at (height, width). */
int nar_unet_workspace_bytes(const nar_unet* net, int32_t height, int32_t width,
                             size_t* bytes);
/* forward(): in_dev is f32 NHWC (1,H,W,Cin) -- e.g. the padded buffer
 * nar_resolve wrote -- and out_dev is f32 NHWC (1,H,W,output_channels).
 * H and W must be multiples of 2^(levels-1) (model.py:148-151). */
int nar_unet_forward(nar_unet* net, const float* in_dev, int32_t height, int32_t width,
                     float* out_dev, void* workspace, size_t workspace_bytes,
                     void* stream);

#ifdef __cplusplus
}
#endif
#endif /* NAR_B200_H */
