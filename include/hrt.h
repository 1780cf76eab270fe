/*
 * hrt.h - C ABI of the B200-native hybrid NeRF/mesh renderer (libhrt.so).
 *
 * Drop-in boundary for the reference render path (arxiv 2309.04581
 * reference package `hybridrt`, pure Python). The reference has no FFI; its
 * seams are Python duck types, and each entry point below replaces one of
 * them (reference file:line under pkg/src/hybridrt/):
 *
 *   hrt_create / hrt_destroy  <- scene assembly build_scene + Bvh(...)       scene.py:502-554, surface.py:289-369
 *   hrt_render               <- render / render_surface_only /
 *                               render_volume_only (mode 0/1/2)              render.py:372-396
 *   hrt_render_host          <- same, host buffers in/out (what `render`
 *                               returns: HdrImage pixels)                    render.py:353-369
 *   hrt_trace_paths          <- trace_path (batch of caller rays)            render.py:302-312
 *   hrt_refit                <- Scene.rebuild_bvh after sim sync             scene.py:475-479, sim.py:673-698
 *   hrt_field_sample         <- field seam field.sample_batch(p[, d])       field.py:143-161
 *   hrt_field_encode         <- (new) hash-grid encode, parity probe
 *   hrt_occupancy            <- (new) occupancy bitfield readback
 *   hrt_intersect            <- Bvh.intersect_batch / any_hit_batch          surface.py:377-478
 *   hrt_uniform              <- rng.uniform                                  rng.py:54-57
 *   hrt_primary_rays         <- _sample_jitter + Camera.primary_rays         render.py:61-74, 320-330
 *
 * Conventions (reference render.py:245, 368, 378; scene.py:27-32):
 *   return 0 on success; HRT_EINVAL -> ValueError, HRT_ENONFINITE ->
 *   AssertionError (NaN / negative radiance), HRT_ECUDA / HRT_ENOMEM ->
 *   RuntimeError. hrt_last_error() describes the last failure (thread-local).
 * Memory: every pointer in hrt_scene_desc is a HOST pointer, copied during
 *   hrt_create (the library owns its device copies and scratch queues).
 *   Pointers marked "device" in the probes are device pointers on the
 *   handle's device. `stream` is a cudaStream_t (NULL = default stream).
 * Threading: calls on one handle are serialised by the caller; one handle
 *   per device.
 */
#ifndef HRT_H
#define HRT_H

#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define HRT_OK 0
#define HRT_EINVAL 1
#define HRT_ENONFINITE 2
#define HRT_ECUDA 3
#define HRT_ENOMEM 4

#define HRT_FIELD_NONE 0
#define HRT_FIELD_DENSE 1
#define HRT_FIELD_NEURAL 2

#define HRT_MODE_HYBRID 0
#define HRT_MODE_SURFACE 1
#define HRT_MODE_VOLUME 2

typedef struct hrt_handle hrt_handle;

typedef struct {
    int32_t kind;                 /* HRT_FIELD_* */
    int32_t identity;             /* world_from_field is the identity */
    double bbox_lo[3], bbox_hi[3];
    double field_from_world[16];  /* row-major 4x4 inverse placement */
    /* dense RadianceGrid (field.py:104-175) */
    int32_t res[3];
    double scale[3];              /* (res-1)/(hi-lo), 0 where res == 1 */
    const double* sigma;          /* nx*ny*nz, C order (z fastest) */
    const double* radiance;       /* nx*ny*nz*3 */
    int32_t sigma_const, rad_const;
    /* neural field */
    int32_t n_levels, n_features, log2_table, act;   /* act 0 sigmoid, 1 softplus */
    const int32_t* level_n;       /* N_l */
    const int64_t* level_offset;  /* entry offset per level */
    const int32_t* level_dense;
    const float* level_scale;     /* L x 3 float32 N_l / (hi - lo) */
    const float* table;           /* n_entries x n_features */
    int64_t n_entries;
    const uint16_t* w_density1;   /* fp16 bits, row-major [in][out]: (L*F) x 64 */
    const uint16_t* w_density2;   /* 64 x 16 */
    const uint16_t* w_color1;     /* 32 x 64 */
    const uint16_t* w_color2;     /* 64 x 64 */
    const uint16_t* w_color3;     /* 64 x 3 */
    int32_t occ_res;
    float occ_scale[3];           /* float32 G / (hi - lo) */
    double occ_threshold;
    const uint32_t* occ_bits;     /* NULL: built on the device from density */
} hrt_field_desc;

typedef struct {
    int64_t n_faces;              /* meshes concatenated in scene order */
    const double* v0;             /* n_faces x 3 */
    const double* e1;             /* v1 - v0 */
    const double* e2;             /* v2 - v0 */
    const double* normal;         /* unit face normals */
    const double* emission;       /* n_faces x 3 */
    const int32_t* mesh_of;       /* face -> mesh (material) index */
    int32_t n_materials;
    const int32_t* mat_kind;      /* 0 Lambertian, 1 Mirror, 2 Dielectric */
    const double* mat_rgb;        /* albedo / reflectance / tint, n_materials x 3 */
    const double* mat_ior;
    int64_t n_blockers;           /* non-emissive faces (shadow rays) */
    const double *bv0, *be1, *be2;
    int32_t n_emitters;
    const double* emitter_tris;   /* n x 9 */
    const double* emitter_cdf;
    const double* emitter_rsrc;
    hrt_field_desc field;
    int32_t n_bounces;
    double threshold, march_step, spawn_eps;
    int32_t sample_cap;           /* NeRF samples per path, 0 = unlimited */
    double early_t;               /* in-march early-out on max(T_spec), 0 = off */
} hrt_scene_desc;

typedef struct {
    double rot[9];                /* camera-to-world rotation (pose.m[:3,:3]) */
    double pos[3];
    double tan_half;              /* tan(fov / 2), vertical fov */
    double aspect;                /* width / height */
    int32_t width, height;
} hrt_camera;

typedef struct {
    int64_t paths;
    int64_t nerf_samples;         /* encode + MLP evaluations */
    int64_t shadow_rays;
    int64_t bounce_rays;          /* closest-hit queries */
    int64_t trace_records;
    float ms;                     /* device time of the call */
    float field_ms;               /* summed device time of the field-engine launches */
    int32_t field_launches;
    int64_t launches;             /* kernels this library launched */
    int64_t evaluated;            /* field evaluations incl. speculative ones discarded by early-out */
    int64_t rounds;               /* march rounds (generate -> field -> composite) */
    float stage_ms[8];            /* per-stage device time (HRT_STAGE_*), only after hrt_set_profile(h, 1) */
    int64_t batch_rows;           /* field-engine rows launched (samples + holes) */
    int64_t shadow_traced;        /* shadow rays traced (>= shadow_rays: batch rows past an
                                     early-out / cap are traced, then discarded by the composite) */
} hrt_stats;

/* Pipeline stages timed by hrt_set_profile (CUDA events around every launch). */
enum {
    HRT_STAGE_RAYGEN = 0,         /* k_raygen / k_load_rays */
    HRT_STAGE_INTERSECT = 1,      /* closest hit (K2) */
    HRT_STAGE_MARCH_GEN = 2,      /* segment setup + occupancy DDA sample generation (K4) */
    HRT_STAGE_FIELD = 3,          /* hash encode + tcgen05 MLP field engine (K5/K6) */
    HRT_STAGE_SHADOW = 4,         /* shadow any-hit of NeRF samples (K3) */
    HRT_STAGE_COMPOSITE = 5,      /* transmittance compositing (K7) fused with next-round sample generation, dense-grid march */
    HRT_STAGE_SHADE = 6,          /* BSDF sample, spawn, compaction (K8) */
    HRT_STAGE_ACCUMULATE = 7      /* per-pixel sum / spp (K9) */
};

const char* hrt_last_error(void);
int hrt_version(void);

int hrt_create(const hrt_scene_desc* desc, hrt_handle** out);
int hrt_destroy(hrt_handle* h);

/* Render n_pixels listed pixel ids (device int32, NULL = all w*h in raster
 * order) x spp paths. out: device, n_pixels x 3 float64 linear radiance. */
int hrt_render(hrt_handle* h, const hrt_camera* cam, int32_t spp, uint64_t seed, int32_t mode,
               const int32_t* pixels, int64_t n_pixels, double* out, hrt_stats* stats,
               void* stream);

/* mode flag: `out` is a raster (w*h, 3) frame indexed by global pixel id
 * instead of (n_pixels, 3) in list order - e.g. rank 0's frame mapped into
 * this process with hrt_ipc_open, so the multi-GPU frame assembly is the
 * accumulate kernel's own stores over NVLink (no gather collective). */
#define HRT_OUT_BY_PIXEL 0x100

/* Same with host pixels / host out; copies inside, synchronous. Page-locked
 * (cudaMallocHost / cudaHostRegister) buffers are DMA'd directly, pageable
 * ones are staged through pinned buffers owned by the handle. */
int hrt_render_host(hrt_handle* h, const hrt_camera* cam, int32_t spp, uint64_t seed,
                    int32_t mode, const int32_t* pixels, int64_t n_pixels, double* out,
                    hrt_stats* stats);

/* Caller-supplied rays (device o, d: n x 3; pixel/sample keys int64) through
 * the same bounce loop; L: device n x 3 (trace_path, render.py:302-312). */
int hrt_trace_paths(hrt_handle* h, const double* o, const double* d, const int64_t* pixel,
                    const int64_t* sample, int64_t n, uint64_t seed, int32_t mode, double* L,
                    void* stream);

/* Transport operator of emitter estimation (emitters.py:73-166,
 * build_transport): per pose, surface-only paths (n_bounces = max_depth, no
 * field) whose front-facing hits add T_spec / spp to
 * A[pose*w*h + pixel, face, :] instead of multiplying the face emission, so
 * image = A @ emission. out: device float64 (n_poses*w*h, n_faces, 3),
 * zeroed by the call; sums in the reference's np.add.at order. */
int hrt_transport(hrt_handle* h, const hrt_camera* cams, int32_t n_poses, int32_t spp, uint64_t seed,
                  int32_t max_depth, double* out, void* stream);

/* Debug trace of evaluated NeRF samples: int32 records (path, bounce, k,
 * occupancy cell) in device memory, up to cap records; enabled for the
 * next hrt_render call only. */
int hrt_set_trace(hrt_handle* h, int32_t* records, int64_t cap);

/* Rigid per-mesh motion refit on the device (cfg3: 200 meshes move each
 * frame; sim.py:673-698 sync_to_renderer -> scene.py:475-479 rebuild).
 * set_rigid_base: object-space corners (n_faces x 9: p0, p1, p2) in global
 * face order, and the global face id of every blocker face. refit_rigid:
 * n_meshes row-major 3x4 world_from_object matrices; world faces, normals
 * and both trees are rebuilt / refit on the GPU (no per-frame face upload). */
int hrt_set_rigid_base(hrt_handle* h, const double* corners, const int32_t* blocker_faces);
int hrt_refit_rigid(hrt_handle* h, const double* xf, int32_t n_meshes);

/* RenderConfig of later calls (scene.py:138-144 + spawn_eps, sample cap,
 * early-out): the reference reads scene.render at every render, so a changed
 * config applies without re-uploading the scene. */
int hrt_set_config(hrt_handle* h, int32_t n_bounces, double threshold, double march_step,
                   double spawn_eps, int32_t sample_cap, double early_t);

/* March schedule of later hrt_render calls (neural field, hybrid mode):
 * continuous != 0 (default) advances each path to its next bounce inside the
 * march rounds (all bounces share one wavefront); 0 runs the reference's
 * bounce-by-bounce loop (render.py:214) - intersect all, march all, shade all.
 * Both give bit-identical results; this exists for A/B measurement and tests. */
int hrt_set_march(hrt_handle* h, int32_t continuous);

/* Per-stage device timing of later hrt_render calls into hrt_stats.stage_ms
 * (on != 0) or off (default). Measurement aid: adds one event pair per launch. */
int hrt_set_profile(hrt_handle* h, int32_t on);

/* K9, finalize (render.py:399-401) on the device: hdr != 0 -> PFM bytes
 * (images.py:37-40, float32 little-endian, rows bottom-up), else PPM P6
 * (images.py:59-64, sRGB tone map core.py:51-64, round-half-up 8 bit).
 * src: device float64 (n, 3) radiance rows; pixel: device int32 global pixel
 * id per row (< 0 = padding), or NULL for a raster frame (n = w*h). This is
 * also the unpack of the multi-GPU gather (rows = concatenated rank buffers).
 * out: device buffer of cap bytes, or NULL to query *nbytes. Non-finite
 * radiance in PPM mode -> HRT_ENONFINITE (reference tone_map asserts finite
 * input); PFM stores it as is, like encode_pfm. */
int hrt_finalize(int32_t width, int32_t height, const double* src, const int32_t* pixel, int64_t n,
                 int32_t hdr, uint8_t* out, int64_t cap, int64_t* nbytes, void* stream);

/* Peer frame plumbing (tiles.PeerFrame): a cudaMalloc'd buffer, its CUDA
 * IPC handle (64 bytes) and the mapping of a peer's buffer into this process
 * (peer access enabled lazily; NVLink / NVSwitch between GPUs). */
int hrt_buffer_alloc(int64_t bytes, void** ptr);
int hrt_buffer_free(void* ptr);
int hrt_ipc_handle(const void* ptr, uint8_t* handle64);
int hrt_ipc_open(const uint8_t* handle64, void** ptr);
int hrt_ipc_close(void* ptr);

/* Roofline probe of the hash-grid encode: useful GB/s of independent random
 * one-entry gathers (8 B for F = 2, 16 B for F = 4) over an L2-resident window
 * (the first <= 64 MiB) of this scene's hash table, through the LSU path
 * (mode 0), the TEX path (1) or both at once (2): the L1-miss request ceiling. */
int hrt_gather_peak(hrt_handle* h, int32_t mode, double* gbs);

/* Move the field (reference: a dynamic field object's world_from_field is
 * reassigned between frames, sim.py:673-698, without a BVH rebuild):
 * identity != 0, or the new row-major 4x4 field_from_world (rigid). The
 * occupancy grid and the network live in the field frame and are kept. */
int hrt_set_field_transform(hrt_handle* h, int32_t identity, const double* field_from_world);

/* Measurement: for the last hrt_render's device-driven march rounds (neural
 * field, continuous march), the batch rows of each round (live paths x
 * samples per path, holes included), the samples generated into them, and
 * the field-engine launch time of that round (ms, CUDA events); *n = rounds
 * reported (<= cap). Any output pointer may be NULL. */
int hrt_round_rows(hrt_handle* h, int64_t* rows, int64_t* samples, float* field_ms, int32_t cap,
                   int32_t* n);

/* L2 roofline probe (bench.py "roofline"): GB/s of coalesced 16-B reads of
 * this scene's hash table (its first 64 MiB if larger) while it is
 * L2-resident (all SMs, 8 passes), and GB/s of random whole 32-B sector
 * gathers over it (lane pairs, L1 bypassed); *bytes = the probed size.
 * Device-synchronous, default stream. */
int hrt_l2_peak(hrt_handle* h, double* read_gbs, double* sector_gbs, int64_t* bytes);

/* New world-space face geometry (same topology; host pointers). */
int hrt_refit(hrt_handle* h, const double* v0, const double* e1, const double* e2,
              const double* normal, const double* bv0, const double* be1, const double* be2);

/* Field seam probes (device pointers). dirs may be NULL (density only). */
int hrt_field_sample(hrt_handle* h, const double* points, const double* dirs, int64_t n,
                     float* sigma, float* rgb, int32_t* evaluated, int32_t use_occupancy,
                     void* stream);
int hrt_field_encode(hrt_handle* h, const double* points, int64_t n, float* features,
                     uint32_t* indices, void* stream);
int hrt_occupancy(hrt_handle* h, uint32_t* host_words, int64_t n_words);

/* Geometry / RNG / camera probes (device pointers). blocker: 0 scene BVH,
 * 1 shadow blockers. any: 0 nearest (t, face), 1 any-hit (hit). */
int hrt_intersect(hrt_handle* h, int32_t blocker, int32_t any, const double* o, const double* d,
                  const double* t_min, const double* t_max, int64_t n, double* t, int64_t* face,
                  uint8_t* hit, void* stream);
int hrt_uniform(const int64_t* keys, int64_t n, double* out, void* stream);
int hrt_primary_rays(const hrt_camera* cam, const int64_t* pixel, const int64_t* sample,
                     int64_t n, uint64_t seed, int32_t spp, double* o, double* d, void* stream);

#ifdef __cplusplus
}
#endif
#endif
