"""paper_2604_25459_b200 — thin Python binding of libgsb (include/gsb.h).

Argument marshalling only: every step of the render runs in libgsb's sm_100a kernels.
PyTorch supplies device memory and streams (tensor.data_ptr(), current_stream().cuda_stream).
There is no CPU fallback: importing works everywhere, but any call needs libgsb.so built
for sm_100a and a B200; a missing library raises immediately.
"""
from __future__ import annotations

import ctypes
import os
from dataclasses import dataclass, field
from typing import Optional, Sequence

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.environ.get("GSB_LIB_PATH") or os.path.join(_HERE, "libgsb.so")  # override: A/B builds (scripts/ab.py)

GSB_FLAG_STATS = 1
GSB_FLAG_TIMING = 2
GSB_FLAG_SCORES = 4
GSB_FLAG_STATIC_PER_ENV = 8
GSB_FLAG_FIXED_PLAN = 16
GSB_OBS_DEPTH_F16 = 1
GSB_RESERVE_HOST_IO = 1

STATUS = {0: "GSB_OK", 1: "GSB_ERR_INVALID_ARGUMENT", 2: "GSB_ERR_SHAPE_MISMATCH",
          3: "GSB_ERR_UNKNOWN_BODY", 4: "GSB_ERR_OUT_OF_MEMORY", 5: "GSB_ERR_CAPACITY",
          6: "GSB_ERR_CUDA", 7: "GSB_ERR_DEVICE"}

# every symbol include/gsb.h declares
EXPORTS = ["gsb_create_scene", "gsb_reserve", "gsb_render", "gsb_render_rig", "gsb_render_host",
           "gsb_prebin_static", "gsb_render_static",
           "gsb_scores_reset", "gsb_get_scores", "gsb_filter_scene", "gsb_render_obs", "gsb_render_obs_host", "gsb_get_stats",
           "gsb_get_stats_ext", "gsb_get_overflow",
           "gsb_get_timings", "gsb_destroy_scene", "gsb_last_error", "gsb_version",
           "gsb_debug_project", "gsb_debug_bin_sort", "gsb_debug_tile_lists",
           "gsb_obs_encode", "gsb_lidar_create", "gsb_render_lidar", "gsb_lidar_info", "gsb_lidar_destroy"]


class GsbError(RuntimeError):
    def __init__(self, status: int, msg: str):
        super().__init__(f"{STATUS.get(status, status)}: {msg}")
        self.status = status


class gsb_obs_params(ctypes.Structure):
    _fields_ = [("image_dr", ctypes.c_void_p), ("seed", ctypes.c_uint32), ("step", ctypes.c_uint32),
                ("env_offset", ctypes.c_int64), ("flags", ctypes.c_uint32)]


class gsb_render_params(ctypes.Structure):
    _fields_ = [("width", ctypes.c_int32), ("height", ctypes.c_int32), ("near_plane", ctypes.c_float),
                ("far_plane", ctypes.c_float), ("background", ctypes.c_float * 3),
                ("sh_degree", ctypes.c_int32), ("flags", ctypes.c_uint32)]


class gsb_timings(ctypes.Structure):
    _fields_ = [("setup_ms", ctypes.c_double), ("project_ms", ctypes.c_double), ("scan_ms", ctypes.c_double),
                ("emit_ms", ctypes.c_double), ("sort_ms", ctypes.c_double), ("composite_ms", ctypes.c_double),
                ("launches", ctypes.c_int64), ("composite_launches", ctypes.c_int64), ("chunks", ctypes.c_int64),
                ("long_lists", ctypes.c_int64), ("max_list", ctypes.c_int64)]


class gsb_stats(ctypes.Structure):
    _fields_ = [("visible_V", ctypes.c_int64), ("keys_K", ctypes.c_int64), ("pairs_P", ctypes.c_int64),
                ("terminated_pixels", ctypes.c_int64), ("pixels", ctypes.c_int64)]


_lib = None


class _Absent:
    """Stands in for a symbol an older libgsb build lacks (A/B runs of old builds); every export
    of include/gsb.h is required of the current build by tests/test_abi.py."""
    argtypes = None
    restype = None


def _sig(L, name):
    return getattr(L, name) if hasattr(L, name) else _Absent()


def lib() -> ctypes.CDLL:
    """Load libgsb.so (built by paper_2604_25459_b200/build.py).  Fails loudly if absent."""
    global _lib
    if _lib is not None:
        return _lib
    if not os.path.exists(LIB_PATH):
        raise ImportError(f"libgsb.so not built at {LIB_PATH}: run `python -c 'import __graft_entry__ as g; g.build()'`")
    L = ctypes.CDLL(LIB_PATH)
    P, I32, I64, U32 = ctypes.c_void_p, ctypes.c_int32, ctypes.c_int64, ctypes.c_uint32
    _sig(L, 'gsb_create_scene').argtypes = [P, P, P, P, P, I32, P, I64, I32, I32, ctypes.POINTER(P)]
    _sig(L, 'gsb_reserve').argtypes = [P, I32, I32, I32, I32, I32, I64, U32]
    rp = ctypes.POINTER(gsb_render_params)
    _sig(L, 'gsb_render').argtypes = [P, P, I32, I32, P, P, rp, P, P, P, P, P]
    _sig(L, 'gsb_render_host').argtypes = [P, P, I32, I32, P, P, rp, P, P, P, P, P]
    _sig(L, 'gsb_render_rig').argtypes = [P, P, I64, I64, I32, I32, P, P, P, rp, P, P, P, P, P]
    _sig(L, 'gsb_prebin_static').argtypes = [P, I32, P, P, rp, P]
    _sig(L, 'gsb_render_static').argtypes = [P, P, I32, rp, P, P, P, P, P]
    _sig(L, 'gsb_scores_reset').argtypes = [P, P]
    op = ctypes.POINTER(gsb_obs_params)
    _sig(L, 'gsb_render_obs').argtypes = [P, P, I32, I32, P, P, rp, op, P, P, P]
    _sig(L, 'gsb_render_obs_host').argtypes = [P, P, I32, I32, P, P, rp, op, P, P, P]
    _sig(L, 'gsb_get_scores').argtypes = [P, P, P, P]
    _sig(L, 'gsb_filter_scene').argtypes = [P, P, ctypes.POINTER(P)]
    _sig(L, 'gsb_get_stats').argtypes = [P, ctypes.POINTER(I64), ctypes.POINTER(I64), ctypes.POINTER(I64)]
    _sig(L, 'gsb_get_stats_ext').argtypes = [P, ctypes.POINTER(gsb_stats)]
    _sig(L, 'gsb_get_overflow').argtypes = [P, ctypes.POINTER(I32)]
    _sig(L, 'gsb_get_timings').argtypes = [P, ctypes.POINTER(gsb_timings)]
    _sig(L, 'gsb_destroy_scene').argtypes = [P]
    _sig(L, 'gsb_last_error').argtypes = []
    _sig(L, 'gsb_version').argtypes = []
    L.gsb_last_error.restype = ctypes.c_char_p
    L.gsb_version.restype = ctypes.c_char_p
    _sig(L, 'gsb_debug_project').argtypes = [P, P, I32, I32, P, P, rp, P, P, P, P]
    _sig(L, 'gsb_debug_bin_sort').argtypes = [P, P, P, P, P, P, P, I32, I64, I32, I32, P, P, I64,
                                     ctypes.POINTER(I64), P]
    _sig(L, 'gsb_debug_tile_lists').argtypes = [P, P, P, P, P, P, P, P, I32, I64, I32, I32, I32, I32, P, P, I64,
                                       ctypes.POINTER(I64), ctypes.POINTER(I32), P]
    _sig(L, 'gsb_obs_encode').argtypes = [P, P, I32, I32, I32, I32, op, P, P, P, P]
    _sig(L, 'gsb_lidar_create').argtypes = [P, P, I32, I32, I32, ctypes.POINTER(P)]
    _sig(L, 'gsb_render_lidar').argtypes = [P, P, P, I32, I32, P, I32, P, ctypes.c_float, ctypes.c_float, P, P, P]
    _sig(L, 'gsb_lidar_info').argtypes = [P, ctypes.POINTER(I32), ctypes.POINTER(I32), ctypes.POINTER(I32),
                                 ctypes.POINTER(I64)]
    _sig(L, 'gsb_lidar_destroy').argtypes = [P]
    for name in EXPORTS:
        if name not in ("gsb_last_error", "gsb_version"):
            _sig(L, name).restype = ctypes.c_int
    _lib = L
    return L


def _check(status: int):
    if status != 0:
        raise GsbError(status, lib().gsb_last_error().decode())


def _ptr(t) -> Optional[int]:
    """Device pointer of a CUDA tensor (or None)."""
    if t is None:
        return None
    if not t.is_contiguous():
        raise ValueError("tensor must be contiguous")
    return t.data_ptr()


def _anyptr(a) -> Optional[int]:
    """Pointer of a CUDA tensor, a CPU tensor or a numpy array (for calls that accept either)."""
    if isinstance(a, np.ndarray) or (a is not None and not a.is_cuda):
        return _hptr(a)
    return _ptr(a)


def _hptr(a) -> Optional[int]:
    """Host pointer of a numpy array or a CPU tensor."""
    if a is None:
        return None
    if isinstance(a, np.ndarray):
        if not a.flags.c_contiguous:
            raise ValueError("array must be C-contiguous")
        return a.ctypes.data
    if a.is_cuda or not a.is_contiguous():
        raise ValueError("expected a contiguous host tensor")
    return a.data_ptr()


_DT = {"f32": ("float32", np.float32), "i32": ("int32", np.int32), "u8": ("uint8", np.uint8),
       "f16": ("float16", np.float16)}


def _buf(t, kind: str, n: int, name: str, device: Optional[int]):
    """Validate a buffer before its pointer crosses the C ABI (which cannot check it): dtype,
    contiguity, at least n elements, and on the scene's CUDA device (device = index) or on the host
    (device = None).  Raises ValueError; None passes (nullable arguments)."""
    if t is None:
        return
    tname, npt = _DT[kind]
    if isinstance(t, np.ndarray):
        if device is not None:
            raise ValueError(f"{name}: expected a CUDA tensor on device {device}, got a numpy array")
        ok_dt, numel = t.dtype == npt, t.size
    else:
        import torch
        if device is not None and (not t.is_cuda or (t.device.index or 0) != device):
            raise ValueError(f"{name}: expected a tensor on cuda:{device}, got {t.device}")
        if device is None and t.is_cuda:
            raise ValueError(f"{name}: expected a host tensor, got {t.device}")
        ok_dt, numel = t.dtype == getattr(torch, tname), t.numel()
    if not ok_dt:
        raise ValueError(f"{name}: expected {tname}, got {t.dtype}")
    if numel < n:
        raise ValueError(f"{name}: {numel} elements < the {n} required")


def _stream(stream) -> Optional[int]:
    if stream is None:
        import torch
        return torch.cuda.current_stream().cuda_stream
    return stream if isinstance(stream, int) else stream.cuda_stream


@dataclass
class RenderParams:
    width: int
    height: int
    near: float = 0.01
    far: float = 1000.0
    background: Sequence[float] = (0.0, 0.0, 0.0)
    sh_degree: int = -1
    stats: bool = False
    timing: bool = False
    scores: bool = False   # accumulate the reading-R30 pruning scores into the scene
    static_per_env: bool = False   # gsb_render_static: env e uses pre-binned camera e
    fixed_plan: bool = False   # no host sync / data-dependent launches: capturable in a CUDA graph

    def to_c(self) -> gsb_render_params:
        p = gsb_render_params()
        p.width, p.height, p.near_plane, p.far_plane = self.width, self.height, self.near, self.far
        for k in range(3):
            p.background[k] = float(self.background[k])
        p.sh_degree = self.sh_degree
        p.flags = ((GSB_FLAG_STATS if self.stats else 0) | (GSB_FLAG_TIMING if self.timing else 0)
                   | (GSB_FLAG_SCORES if self.scores else 0)
                   | (GSB_FLAG_STATIC_PER_ENV if self.static_per_env else 0)
                   | (GSB_FLAG_FIXED_PLAN if self.fixed_plan else 0))
        return p


def prune_mask(w_sum, keep_fraction: float) -> np.ndarray:
    """Host-side pruning policy over reading-R30 scores: keep the ceil(keep_fraction * N)
    Gaussians of largest w_sum (ties by lower creation index); returns bool [N] by id."""
    w = np.asarray(w_sum.cpu() if hasattr(w_sum, "cpu") else w_sum, np.float64).reshape(-1)
    n = w.size
    k = int(np.ceil(keep_fraction * n))
    order = np.lexsort((np.arange(n), -w))
    keep = np.zeros(n, bool)
    keep[order[:k]] = True
    return keep


class Scene:
    """A scene template on one device (gsb_create_scene) with its reserved workspace."""

    def __init__(self, means, scales, quats, opacities, sh, sh_degree: int, body_id, n_bodies: int,
                 device: int = 0):
        L = lib()
        self._keep = [np.ascontiguousarray(means, np.float32), np.ascontiguousarray(scales, np.float32),
                      np.ascontiguousarray(quats, np.float32), np.ascontiguousarray(opacities, np.float32),
                      np.ascontiguousarray(sh, np.float32), np.ascontiguousarray(body_id, np.int32)]
        m, s, q, o, c, b = self._keep
        self.n = int(m.shape[0])
        self.n_bodies = int(n_bodies)
        self.sh_degree = int(sh_degree)
        self.device = device
        h = ctypes.c_void_p()
        _check(L.gsb_create_scene(m.ctypes.data, s.ctypes.data, q.ctypes.data, o.ctypes.data, c.ctypes.data,
                                  int(sh_degree), b.ctypes.data, self.n, self.n_bodies, int(device),
                                  ctypes.byref(h)))
        self._h = h
        self._keep = None

    @classmethod
    def _wrap(cls, handle, n: int, n_bodies: int, sh_degree: int, device: int) -> "Scene":
        obj = cls.__new__(cls)
        obj._h, obj.n, obj.n_bodies, obj.sh_degree, obj.device, obj._keep = handle, n, n_bodies, sh_degree, device, None
        return obj

    @classmethod
    def from_synth(cls, scene, device: int = 0) -> "Scene":
        return cls(scene.means, scene.scales, scene.quats, scene.opacities, scene.sh, scene.sh_degree,
                   scene.body_id, scene.n_bodies, device)

    def close(self):
        if getattr(self, "_h", None) is not None and self._h.value:
            lib().gsb_destroy_scene(self._h)
            self._h = ctypes.c_void_p()

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass

    def reserve(self, max_envs: int, n_cams: int, width: int, height: int, chunk_frames: int = 0,
                key_capacity: int = 0, host_io: bool = False):
        _check(lib().gsb_reserve(self._h, max_envs, n_cams, width, height, chunk_frames, key_capacity,
                                 GSB_RESERVE_HOST_IO if host_io else 0))

    def _check_io(self, B, C, params, poses, intrinsics, w2c, out_rgb, out_depth, out_alpha, out_n_eval, dev):
        """Shapes the C ABI assumes, checked here (it cannot): inputs and outputs of B x C frames.
        Missing (None) buffers are left to the C ABI, which rejects a NULL required pointer."""
        F, px = B * C, params.width * params.height
        if self.n_bodies and poses is not None:
            _buf(poses, "f32", B * self.n_bodies * 7, "poses", dev)
        _buf(intrinsics, "f32", F * 4, "intrinsics", dev)
        _buf(w2c, "f32", F * 12, "world_to_cam", dev)
        _buf(out_rgb, "f32", F * 3 * px, "out_rgb", dev)
        _buf(out_depth, "f32", F * px, "out_depth", dev)
        _buf(out_alpha, "f32", F * px, "out_alpha", dev)
        _buf(out_n_eval, "i32", F * px, "out_n_eval", dev)

    def _check_obs(self, B, C, params, poses, intrinsics, w2c, out_rgb8, out_depth, image_dr, depth_f16, dev):
        F, px = B * C, params.width * params.height
        if self.n_bodies and poses is not None:
            _buf(poses, "f32", B * self.n_bodies * 7, "poses", dev)
        _buf(intrinsics, "f32", F * 4, "intrinsics", dev)
        _buf(w2c, "f32", F * 12, "world_to_cam", dev)
        _buf(out_rgb8, "u8", F * 3 * px, "out_rgb8", dev)
        _buf(out_depth, "f16" if depth_f16 else "f32", F * px, "out_depth", dev)
        _buf(image_dr, "f32", F * 4, "image_dr", dev)

    def render(self, poses, intrinsics, world_to_cam, params: RenderParams, out_rgb, out_depth=None,
               out_alpha=None, out_n_eval=None, stream=None):
        """gsb_render on CUDA tensors: poses [B,nb,7], intrinsics [B,C,4], world_to_cam [B,C,3,4],
        out_rgb [B,C,3,H,W] (float32), out_depth/out_alpha [B,C,H,W] float32, out_n_eval int32."""
        B, C = int(intrinsics.shape[0]), int(intrinsics.shape[1])
        self._check_io(B, C, params, poses, intrinsics, world_to_cam, out_rgb, out_depth, out_alpha, out_n_eval,
                       self.device)
        p = params.to_c()
        _check(lib().gsb_render(self._h, _ptr(poses) if self.n_bodies else None, B, C, _ptr(intrinsics),
                                _ptr(world_to_cam), ctypes.byref(p), _ptr(out_rgb), _ptr(out_depth),
                                _ptr(out_alpha), _ptr(out_n_eval), _stream(stream)))

    def render_rig(self, poses, intrinsics, cam_extrinsics, params: RenderParams, out_rgb, out_depth=None,
                   out_alpha=None, out_n_eval=None, cam_body=None, pose_env_stride: int = 0,
                   pose_body_stride: int = 0, stream=None):
        """gsb_render_rig: strided poses (element strides, in floats) and body-attached cameras:
        cam_body[c] = k >= 0 makes cam_extrinsics[:, c] the body->camera mount on body k."""
        B, C = int(intrinsics.shape[0]), int(intrinsics.shape[1])
        body = max(int(pose_body_stride), 7)
        env = int(pose_env_stride) or self.n_bodies * body
        need = (B - 1) * env + (self.n_bodies - 1) * body + 7 if (B and self.n_bodies) else 0
        self._check_io(B, C, params, None, intrinsics, cam_extrinsics, out_rgb, out_depth, out_alpha, out_n_eval,
                       self.device)
        _buf(poses, "f32", need, "poses", self.device)
        p = params.to_c()
        cb = None
        if cam_body is not None:
            cb = np.ascontiguousarray(cam_body, np.int32)
            if cb.size != C:
                raise ValueError("cam_body needs one entry per camera")
        _check(lib().gsb_render_rig(self._h, _ptr(poses) if poses is not None else None, pose_env_stride,
                                    pose_body_stride, B, C, _ptr(intrinsics), _ptr(cam_extrinsics),
                                    None if cb is None else cb.ctypes.data, ctypes.byref(p), _ptr(out_rgb),
                                    _ptr(out_depth), _ptr(out_alpha), _ptr(out_n_eval), _stream(stream)))

    def render_host(self, poses, intrinsics, world_to_cam, params: RenderParams, out_rgb, out_depth=None,
                    out_alpha=None, out_n_eval=None, stream=None):
        """gsb_render_host on host (pinned) buffers; synchronous."""
        B, C = int(intrinsics.shape[0]), int(intrinsics.shape[1])
        self._check_io(B, C, params, poses, intrinsics, world_to_cam, out_rgb, out_depth, out_alpha, out_n_eval,
                       None)
        p = params.to_c()
        _check(lib().gsb_render_host(self._h, _hptr(poses) if self.n_bodies else None, B, C,
                                     _hptr(intrinsics), _hptr(world_to_cam), ctypes.byref(p), _hptr(out_rgb),
                                     _hptr(out_depth), _hptr(out_alpha), _hptr(out_n_eval), _stream(stream)))

    def prebin_static(self, intrinsics, world_to_cam, params: RenderParams, stream=None):
        """gsb_prebin_static: pre-bin the static background for C fixed cameras (intrinsics [C,4],
        world_to_cam [C,3,4], CUDA or CPU tensors).  Call reserve() afterwards."""
        C = int(intrinsics.shape[0])
        p = params.to_c()
        _check(lib().gsb_prebin_static(self._h, C, _anyptr(intrinsics), _anyptr(world_to_cam), ctypes.byref(p),
                                       _stream(stream)))

    def render_static(self, poses, params: RenderParams, out_rgb, out_depth=None, out_alpha=None,
                      out_n_eval=None, stream=None):
        """gsb_render_static: B envs x the pre-binned cameras; out_rgb [B,C,3,H,W]."""
        B = int(out_rgb.shape[0])
        C = int(out_rgb.shape[1]) if out_rgb.dim() == 5 else 1
        self._check_io(B, C, params, poses, None, None, out_rgb, out_depth, out_alpha, out_n_eval, self.device)
        p = params.to_c()
        _check(lib().gsb_render_static(self._h, _ptr(poses) if self.n_bodies else None, B, ctypes.byref(p),
                                       _ptr(out_rgb), _ptr(out_depth), _ptr(out_alpha), _ptr(out_n_eval),
                                       _stream(stream)))

    @staticmethod
    def _obs(image_dr, seed, step, env_offset, depth_f16, host):
        o = gsb_obs_params()
        o.image_dr = None if image_dr is None else (_hptr(image_dr) if host else _ptr(image_dr))
        o.seed, o.step, o.env_offset = int(seed) & 0xFFFFFFFF, int(step) & 0xFFFFFFFF, int(env_offset)
        o.flags = GSB_OBS_DEPTH_F16 if depth_f16 else 0
        return o

    def render_obs(self, poses, intrinsics, world_to_cam, params: RenderParams, out_rgb8, out_depth=None,
                   image_dr=None, seed: int = 0, step: int = 0, env_offset: int = 0, depth_f16: bool = True,
                   stream=None):
        """gsb_render_obs: uint8 RGB [B,C,3,H,W] (+ depth [B,C,H,W] as float16 or float32) with the
        reading-R31 image DR (image_dr [B,C,4] CUDA float32: gain, contrast, brightness, noise_std)."""
        B, C = int(intrinsics.shape[0]), int(intrinsics.shape[1])
        self._check_obs(B, C, params, poses, intrinsics, world_to_cam, out_rgb8, out_depth, image_dr, depth_f16,
                        self.device)
        p = params.to_c()
        o = self._obs(image_dr, seed, step, env_offset, depth_f16, False)
        _check(lib().gsb_render_obs(self._h, _ptr(poses) if self.n_bodies else None, B, C, _ptr(intrinsics),
                                    _ptr(world_to_cam), ctypes.byref(p), ctypes.byref(o), _ptr(out_rgb8),
                                    _ptr(out_depth), _stream(stream)))

    def render_obs_host(self, poses, intrinsics, world_to_cam, params: RenderParams, out_rgb8, out_depth=None,
                        image_dr=None, seed: int = 0, step: int = 0, env_offset: int = 0, depth_f16: bool = True,
                        stream=None):
        """gsb_render_obs_host on host (pinned) buffers; synchronous."""
        B, C = int(intrinsics.shape[0]), int(intrinsics.shape[1])
        self._check_obs(B, C, params, poses, intrinsics, world_to_cam, out_rgb8, out_depth, image_dr, depth_f16,
                        None)
        p = params.to_c()
        o = self._obs(image_dr, seed, step, env_offset, depth_f16, True)
        _check(lib().gsb_render_obs_host(self._h, _hptr(poses) if self.n_bodies else None, B, C,
                                         _hptr(intrinsics), _hptr(world_to_cam), ctypes.byref(p), ctypes.byref(o),
                                         _hptr(out_rgb8), _hptr(out_depth), _stream(stream)))

    def scores_reset(self, stream=None):
        """gsb_scores_reset: zero the pruning-score accumulators."""
        _check(lib().gsb_scores_reset(self._h, _stream(stream)))

    def scores(self, stream=None):
        """gsb_get_scores: (w_sum, w_max) float32 CUDA tensors [N] by creation index."""
        import torch
        ws = torch.empty(self.n, dtype=torch.float32, device=f"cuda:{self.device}")
        wm = torch.empty(self.n, dtype=torch.float32, device=f"cuda:{self.device}")
        _check(lib().gsb_get_scores(self._h, _ptr(ws), _ptr(wm), _stream(stream)))
        return ws, wm

    def filter(self, keep) -> "Scene":
        """gsb_filter_scene (filter_template semantics): a new Scene of the Gaussians with
        keep[id] true, re-indexed in creation order."""
        k = np.ascontiguousarray(np.asarray(keep, bool).astype(np.uint8))
        if k.size != self.n:
            raise ValueError("keep needs one entry per Gaussian")
        h = ctypes.c_void_p()
        _check(lib().gsb_filter_scene(self._h, k.ctypes.data, ctypes.byref(h)))
        return Scene._wrap(h, int(k.sum()), self.n_bodies, self.sh_degree, self.device)

    def stats(self):
        V, K, P = ctypes.c_int64(), ctypes.c_int64(), ctypes.c_int64()
        _check(lib().gsb_get_stats(self._h, ctypes.byref(V), ctypes.byref(K), ctypes.byref(P)))
        return {"V": V.value, "K": K.value, "P": P.value}

    def stats_ext(self):
        """gsb_get_stats_ext: V, K, P plus terminated pixels (reading R13) out of all pixels."""
        st = gsb_stats()
        _check(lib().gsb_get_stats_ext(self._h, ctypes.byref(st)))
        return {"V": st.visible_V, "K": st.keys_K, "P": st.pairs_P, "terminated": st.terminated_pixels,
                "pixels": st.pixels}

    def overflow(self) -> bool:
        """gsb_get_overflow: did a GSB_FLAG_FIXED_PLAN render since the last call exceed the key
        capacity (its frames unwritten)?  Resets the flag; synchronises the device."""
        v = ctypes.c_int32()
        _check(lib().gsb_get_overflow(self._h, ctypes.byref(v)))
        return bool(v.value)

    def timings(self):
        t = gsb_timings()
        _check(lib().gsb_get_timings(self._h, ctypes.byref(t)))
        return {k: getattr(t, k) for k, _ in gsb_timings._fields_}

    def debug_project(self, poses, intrinsics, world_to_cam, params: RenderParams, out_rec, out_zbits,
                      out_valid, stream=None):
        B, C = int(intrinsics.shape[0]), int(intrinsics.shape[1])
        p = params.to_c()
        _check(lib().gsb_debug_project(self._h, _ptr(poses) if self.n_bodies else None, B, C, _ptr(intrinsics),
                                       _ptr(world_to_cam), ctypes.byref(p), _ptr(out_rec), _ptr(out_zbits),
                                       _ptr(out_valid), _stream(stream)))


class Lidar:
    """A LiDAR ray pattern bound to a scene (gsb_lidar_create; reading R32, §8(f) row 4).
    dirs: [R,3] unit directions in the sensor frame (host array)."""

    def __init__(self, scene: Scene, dirs, n_az: int = 0, n_el: int = 0):
        d = np.ascontiguousarray(dirs, np.float32).reshape(-1, 3)
        h = ctypes.c_void_p()
        _check(lib().gsb_lidar_create(scene._h, d.ctypes.data, int(d.shape[0]), int(n_az), int(n_el), ctypes.byref(h)))
        self._h, self.scene, self.n_rays = h, scene, int(d.shape[0])

    def info(self):
        a, e, it, k = ctypes.c_int32(), ctypes.c_int32(), ctypes.c_int32(), ctypes.c_int64()
        _check(lib().gsb_lidar_info(self._h, ctypes.byref(a), ctypes.byref(e), ctypes.byref(it), ctypes.byref(k)))
        return {"n_az": a.value, "n_el": e.value, "n_items": it.value, "keys": k.value}

    def render(self, poses, sensor_x, out_range, out_alpha=None, sensor_body=None, near: float = 0.01,
               far: float = 1000.0, stream=None):
        """gsb_render_lidar on CUDA tensors: poses [B,nb,7]; sensor_x [B,S,3,4] (per env) or [S,3,4]
        (shared) world->sensor, or body->sensor for sensors with sensor_body[s] >= 0;
        out_range / out_alpha [B,S,R] float32."""
        B, S = int(out_range.shape[0]), int(out_range.shape[1])
        shared = 1 if sensor_x.dim() == 3 else 0
        sb = None
        if sensor_body is not None:
            sb = np.ascontiguousarray(sensor_body, np.int32)
            if sb.size != S:
                raise ValueError("sensor_body needs one entry per sensor")
        _check(lib().gsb_render_lidar(self.scene._h, self._h, _ptr(poses) if self.scene.n_bodies else None, B, S,
                                      _ptr(sensor_x), shared, None if sb is None else sb.ctypes.data, near, far,
                                      _ptr(out_range), _ptr(out_alpha), _stream(stream)))

    def close(self):
        if getattr(self, "_h", None) is not None and self._h.value:
            lib().gsb_lidar_destroy(self._h)
            self._h = ctypes.c_void_p()

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass


def obs_encode(rgb, out_rgb8, depth=None, out_depth=None, blur=None, image_dr=None, seed: int = 0, step: int = 0,
               env_offset: int = 0, depth_f16: bool = True, stream=None):
    """gsb_obs_encode on CUDA tensors: rgb [B,C,3,H,W] float32 -> out_rgb8 uint8, with the reading-R33
    motion blur (blur [B,C,2] int32 pixel extents, or None) before the reading-R31 image DR."""
    B, C, _, H, W = (int(v) for v in rgb.shape)
    o = Scene._obs(image_dr, seed, step, env_offset, depth_f16, False)
    _check(lib().gsb_obs_encode(_ptr(rgb), _ptr(depth), B, C, W, H, ctypes.byref(o), _ptr(blur), _ptr(out_rgb8),
                                _ptr(out_depth), _stream(stream)))


def debug_bin_sort(u, v, sxx, syy, kappa, zbits, valid, width: int, height: int, cap: int, stream=None):
    """gsb_debug_bin_sort on CUDA tensors [F,N]; returns (offsets [F,T+1] int64, ids[:K] uint32 as int64)."""
    import torch
    F, N = int(u.shape[0]), int(u.shape[1])
    T = ((width + 15) // 16) * ((height + 15) // 16)
    dev = u.device
    offs = torch.empty((F, T + 1), dtype=torch.int64, device=dev)
    ids = torch.empty(max(cap, 1), dtype=torch.int32, device=dev)
    K = ctypes.c_int64()
    _check(lib().gsb_debug_bin_sort(_ptr(u), _ptr(v), _ptr(sxx), _ptr(syy), _ptr(kappa), _ptr(zbits), _ptr(valid),
                                    F, N, width, height, _ptr(offs), _ptr(ids), cap, ctypes.byref(K), _stream(stream)))
    return offs, ids[:K.value]


def debug_tile_lists(u, v, sxx, syy, kappa, zbits, valid, slot_ids, width: int, height: int, cap: int,
                     variant: int = 0, key_mode: int = 0, stream=None):
    """gsb_debug_tile_lists on CUDA tensors [F,N] indexed by record slot (slot_ids [N] int32: creation
    id of each slot).  Returns (offsets [F,T+1] int64, ids[:K] (int32 view of uint32), variant run)."""
    import torch
    F, N = int(u.shape[0]), int(u.shape[1])
    T = ((width + 15) // 16) * ((height + 15) // 16)
    dev = u.device
    offs = torch.empty((F, T + 1), dtype=torch.int64, device=dev)
    ids = torch.empty(max(cap, 1), dtype=torch.int32, device=dev)
    K = ctypes.c_int64()
    var = ctypes.c_int32()
    _check(lib().gsb_debug_tile_lists(_ptr(u), _ptr(v), _ptr(sxx), _ptr(syy), _ptr(kappa), _ptr(zbits), _ptr(valid),
                                      _ptr(slot_ids), F, N, width, height, int(variant), int(key_mode), _ptr(offs),
                                      _ptr(ids), cap, ctypes.byref(K), ctypes.byref(var), _stream(stream)))
    return offs, ids[:K.value], var.value


def version() -> str:
    return lib().gsb_version().decode()
