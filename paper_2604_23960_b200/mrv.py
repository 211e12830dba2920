"""Thin ctypes binding of libmrv.so (include/mrv.h) -- argument marshalling only.

Every step of MotVal / FFC / SpheresFK runs in the CUDA kernels behind the C ABI;
this module converts scene tables (numpy) into ``mrv_robot_desc`` /
``mrv_env_desc`` structs and torch CUDA tensors into raw device pointers plus a
``cudaStream_t``.  There is no CPU fallback: if ``libmrv.so`` is missing or the
device is not an sm_100 part, the calls raise.
"""
from __future__ import annotations

import ctypes as C
import os
from typing import Optional

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.environ.get("MRV_LIB_PATH") or os.path.join(HERE, "libmrv.so")   # override: experiments only

MRV_OK, MRV_EINVAL, MRV_ENOMEM, MRV_ECUDA, MRV_ERANGE, MRV_EUNSUPPORTED = range(6)
CHAIN, SE2, SE3 = 0, 1, 2
CHECK_ENV = 1 << 0
ORDER_HIERARCHICAL = 1 << 1
PACK_LINEAR = 1 << 2
DIAG_NO_EARLY_EXIT = 1 << 3
DIAG_NO_BROADPHASE = 1 << 4
CHECK_SELF = 1 << 5
FOCUS = 1 << 6
PACK_SEQUENTIAL = 1 << 7
NO_CONFLICT = 0xFFFFFFFF
NUM_COUNTERS = 13
COUNTER_NAMES = ["states", "robot_states", "joints", "env_broad", "env_narrow", "rr_broad", "rr_narrow",
                 "sphere_xform", "rr_super", "super_bounds", "self_broad", "rr_capsule", "table_bytes"]

EXPORTS = ["mrv_create_scene", "mrv_destroy_scene", "mrv_motval_batch", "mrv_motval_batch_ex", "mrv_ffc_batch",
           "mrv_ffc_batch_ex", "mrv_decode_conflict", "mrv_fk_states", "mrv_scene_info", "mrv_status_string",
           "mrv_abi_version", "mrv_run_host_batch", "mrv_device_status", "mrv_pp_table_bytes",
           "mrv_pp_build_table", "mrv_pp_motval_batch"]
DEVERR_TIMESTEPS = 1 << 0
DEVERR_RANGE = 1 << 1
DEVERR_START = 1 << 2


class MrvError(RuntimeError):
    def __init__(self, status: int, what: str):
        super().__init__(f"{what}: {status_string(status)} ({status})")
        self.status = status


class RobotDesc(C.Structure):
    _fields_ = [("kind", C.c_int32), ("dof", C.c_int32), ("joint_origin", C.c_void_p), ("joint_type", C.c_void_p),
                ("base", C.c_void_p), ("n_spheres", C.c_int32), ("sphere_link", C.c_void_p), ("sphere", C.c_void_p),
                ("n_self_pairs", C.c_int32), ("self_pairs", C.c_void_p)]


class EnvDesc(C.Structure):
    _fields_ = [("n_spheres", C.c_int32), ("spheres", C.c_void_p), ("n_boxes", C.c_int32), ("boxes", C.c_void_p)]


class MotionBatch(C.Structure):
    _fields_ = [("n_motions", C.c_int64), ("n_waypoints", C.c_int32), ("dof_stride", C.c_int32),
                ("waypoints", C.c_void_p), ("n_timesteps", C.c_void_p), ("fixed_timesteps", C.c_int32),
                ("robot_timesteps", C.c_void_p)]


class LaunchOpts(C.Structure):
    _fields_ = [("states_per_batch", C.c_int32), ("n_slices", C.c_int32), ("counters", C.c_void_p),
                ("batches_evaluated", C.c_void_p), ("t_begin", C.c_int32), ("t_end", C.c_int32),
                ("focus_robot", C.c_int32), ("partner_mask", C.c_uint64), ("warps_per_cta", C.c_int32)]


_lib = None


def lib():
    """Load libmrv.so (raises if it has not been built: no fallback path exists)."""
    global _lib
    if _lib is None:
        if not os.path.exists(LIB_PATH):
            raise ImportError(f"{LIB_PATH} not built: run `python -c 'import __graft_entry__ as g; g.build()'`")
        L = C.CDLL(LIB_PATH)
        vp, i32, i64, u32 = C.c_void_p, C.c_int32, C.c_int64, C.c_uint32
        L.mrv_create_scene.argtypes = [vp, i32, vp, i32, C.POINTER(vp)]
        L.mrv_destroy_scene.argtypes = [vp]
        L.mrv_motval_batch.argtypes = [vp, vp, u32, vp, vp]
        L.mrv_motval_batch_ex.argtypes = [vp, vp, u32, vp, vp, vp]
        L.mrv_ffc_batch.argtypes = [vp, vp, u32, vp, vp]
        L.mrv_ffc_batch_ex.argtypes = [vp, vp, u32, vp, vp, vp]
        L.mrv_decode_conflict.argtypes = [vp, u32, C.POINTER(i32), C.POINTER(i32), C.POINTER(i32)]
        L.mrv_fk_states.argtypes = [vp, vp, i64, vp, vp, vp, vp]
        L.mrv_scene_info.argtypes = [vp, C.POINTER(i32), C.POINTER(i32), C.POINTER(i32), C.POINTER(i32)]
        L.mrv_status_string.argtypes = [i32]
        L.mrv_status_string.restype = C.c_char_p
        L.mrv_abi_version.restype = i32
        L.mrv_run_host_batch.argtypes = [vp, vp, u32, vp, u32, vp, i64, vp]
        # (an experiment's older build loaded through MRV_LIB_PATH may lack the newer calls)
        lenient = bool(os.environ.get("MRV_LIB_PATH"))
        for name, args in (("mrv_device_status", [vp, vp, i32, C.POINTER(u32)]),
                           ("mrv_pp_table_bytes", [vp, i32, C.POINTER(C.c_uint64)]),
                           ("mrv_pp_build_table", [vp, vp, C.c_uint64, i32, vp, vp]),
                           ("mrv_pp_motval_batch", [vp, vp, vp, i32, C.c_uint64, vp, i32, u32, vp, vp, vp])):
            if hasattr(L, name) or not lenient:
                getattr(L, name).argtypes = args
        for name in EXPORTS:
            if not hasattr(L, name) and not lenient:
                raise ImportError(f"libmrv.so lacks {name}")
        _lib = L
    return _lib


def status_string(st: int) -> str:
    return lib().mrv_status_string(st).decode()


def _check(st: int, what: str):
    if st != MRV_OK:
        raise MrvError(st, what)


def _np_ptr(a):
    return None if a is None else a.ctypes.data


def _stream_ptr(stream):
    import torch
    if stream is None:
        stream = torch.cuda.current_stream()
    return stream.cuda_stream


class Scene:
    """An immutable device scene (mrv_create_scene).  ``scene`` is any object with
    ``robots`` (kind, dof, joint_origin, joint_type, base, sphere_link, sphere),
    ``obs_spheres`` [n][4] and ``obs_boxes`` [n][6] (e.g. ``gen.Scene``)."""

    def __init__(self, scene, device: int = 0):
        L = lib()
        keep = []
        n = len(scene.robots)
        rbs = (RobotDesc * max(1, n))()
        for i, r in enumerate(scene.robots):
            jo = None if r.joint_origin is None else np.ascontiguousarray(r.joint_origin, np.float32)
            jt = None if r.joint_type is None else np.ascontiguousarray(r.joint_type, np.int32)
            base = None if r.base is None else np.ascontiguousarray(r.base, np.float32)
            sl = np.ascontiguousarray(r.sphere_link, np.int32)
            sp = np.ascontiguousarray(r.sphere, np.float32)
            selfp = getattr(r, "self_pairs", None)
            selfp = None if selfp is None else np.ascontiguousarray(selfp, np.int32).reshape(-1, 2)
            keep += [jo, jt, base, sl, sp, selfp]
            rbs[i] = RobotDesc(int(r.kind), int(r.dof), _np_ptr(jo), _np_ptr(jt), _np_ptr(base), int(sp.shape[0]),
                               _np_ptr(sl), _np_ptr(sp), 0 if selfp is None else int(selfp.shape[0]), _np_ptr(selfp))
        osph = np.ascontiguousarray(scene.obs_spheres, np.float32).reshape(-1, 4)
        box = np.ascontiguousarray(scene.obs_boxes, np.float32).reshape(-1, 6)
        env = EnvDesc(osph.shape[0], _np_ptr(osph) if osph.size else None, box.shape[0],
                      _np_ptr(box) if box.size else None)
        h = C.c_void_p()
        _check(L.mrv_create_scene(rbs, n, C.byref(env), int(device), C.byref(h)), "mrv_create_scene")
        self._h = h
        self.device = device
        nr, npairs, nsph, nfr = C.c_int32(), C.c_int32(), C.c_int32(), C.c_int32()
        _check(L.mrv_scene_info(h, C.byref(nr), C.byref(npairs), C.byref(nsph), C.byref(nfr)), "mrv_scene_info")
        self.n_robots, self.n_pairs, self.total_spheres, self.total_frames = nr.value, npairs.value, nsph.value, nfr.value

    def close(self):
        if getattr(self, "_h", None):
            lib().mrv_destroy_scene(self._h)
            self._h = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass

    # -------------------------------------------------------------- batch marshalling
    def _batch(self, waypoints, T, n_robots=None):
        import torch
        assert waypoints.is_cuda and waypoints.dtype == torch.float32 and waypoints.dim() == 4, "waypoints: CUDA f32 [M][n][K][S]"
        assert waypoints.is_contiguous(), "waypoints must be contiguous"
        M, n, K, S = waypoints.shape
        if n != (self.n_robots if n_robots is None else n_robots):
            raise ValueError(f"waypoints have {n} robots, expected {self.n_robots if n_robots is None else n_robots}")
        if isinstance(T, int):
            b = MotionBatch(M, K, S, waypoints.data_ptr(), None, T, None)
        elif T.dim() == 2:   # per-robot path lengths [M][n] (stay at goal)
            assert T.is_cuda and T.dtype == torch.int32 and T.is_contiguous() and tuple(T.shape) == (M, n)
            b = MotionBatch(M, K, S, waypoints.data_ptr(), None, 1, T.data_ptr())
        else:
            assert T.is_cuda and T.dtype == torch.int32 and T.is_contiguous() and T.numel() == M
            b = MotionBatch(M, K, S, waypoints.data_ptr(), T.data_ptr(), 0, None)
        return b

    def _opts(self, states_per_batch=0, n_slices=0, counters=None, effort=None, t_begin=0, t_end=0,
              focus=None, partners=(), warps_per_cta=0):
        if not (states_per_batch or n_slices or counters is not None or effort is not None or t_begin or t_end
                or focus is not None or warps_per_cta):
            return None
        mask = 0
        for j in partners:
            mask |= 1 << int(j)
        return LaunchOpts(states_per_batch, n_slices, None if counters is None else counters.data_ptr(),
                          None if effort is None else effort.data_ptr(), int(t_begin), int(t_end),
                          -1 if focus is None else int(focus), mask, int(warps_per_cta))

    def device_status(self, stream=None, clear: bool = True) -> int:
        """The scene's device status word (OR of DEVERR_* bits raised by the batch calls
        since the last clear): conditions on device-resident T the launch cannot check.
        Synchronises ``stream``."""
        v = C.c_uint32()
        _check(lib().mrv_device_status(self._h, _stream_ptr(stream), 1 if clear else 0, C.byref(v)),
               "mrv_device_status")
        return v.value

    def check_device(self, stream=None):
        """Raise MrvError(MRV_ERANGE / MRV_EINVAL) if a batch call raised a device status bit."""
        v = self.device_status(stream)
        if v & DEVERR_TIMESTEPS:
            raise MrvError(MRV_EINVAL, f"device status {v:#x}: a per-motion T < 1")
        if v & DEVERR_RANGE:
            raise MrvError(MRV_ERANGE, f"device status {v:#x}: FFC T * P >= 2^32 - 1")
        if v & DEVERR_START:
            raise MrvError(MRV_EINVAL, f"device status {v:#x}: a PP-ST-RRT start time < 0")

    def motval(self, waypoints, T, flags: int = CHECK_ENV, out=None, stream=None, **opts):
        """MotVal (Alg. 1) -> CUDA uint8 [M] (1 valid, 0 invalid). Enqueued on ``stream``."""
        import torch
        b = self._batch(waypoints, T)
        if out is None:
            out = torch.empty(b.n_motions, dtype=torch.uint8, device=waypoints.device)
        o = self._opts(**opts)
        if opts.get("focus") is not None:
            flags |= FOCUS
        if o is None:
            st = lib().mrv_motval_batch(self._h, C.byref(b), flags, out.data_ptr(), _stream_ptr(stream))
        else:
            st = lib().mrv_motval_batch_ex(self._h, C.byref(b), flags, out.data_ptr(), _stream_ptr(stream), C.byref(o))
        _check(st, "mrv_motval_batch")
        return out

    def ffc(self, waypoints, T, flags: int = 0, out=None, stream=None, **opts):
        """FFC (Alg. 2) -> CUDA int32 view of uint32 keys [M] (t*P + rank or 0xFFFFFFFF)."""
        import torch
        b = self._batch(waypoints, T)
        if out is None:
            out = torch.empty(b.n_motions, dtype=torch.int32, device=waypoints.device)
        o = self._opts(**opts)
        if opts.get("focus") is not None:
            flags |= FOCUS
        if o is None:
            st = lib().mrv_ffc_batch(self._h, C.byref(b), flags, out.data_ptr(), _stream_ptr(stream))
        else:
            st = lib().mrv_ffc_batch_ex(self._h, C.byref(b), flags, out.data_ptr(), _stream_ptr(stream), C.byref(o))
        _check(st, "mrv_ffc_batch")
        return out

    # -------------------------------------------------------------- PP-ST-RRT variant
    @staticmethod
    def _mask(robots):
        m = 0
        for j in robots:
            m |= 1 << int(j)
        return m

    def pp_table(self, paths_wp, paths_T, partners, horizon: int, stream=None):
        """Partner table (mrv_pp_build_table) of the fixed paths ``paths_wp`` (CUDA [1][n][K][S];
        ``paths_T`` an int or per-robot lengths CUDA int32 [1][n]) of ``partners`` over
        absolute timesteps 0..horizon-1 -> CUDA uint8 tensor."""
        import torch
        b = self._batch(paths_wp, paths_T)
        nb = C.c_uint64()
        _check(lib().mrv_pp_table_bytes(self._h, int(horizon), C.byref(nb)), "mrv_pp_table_bytes")
        table = torch.empty(nb.value, dtype=torch.uint8, device=paths_wp.device)
        _check(lib().mrv_pp_build_table(self._h, C.byref(b), self._mask(partners), int(horizon), table.data_ptr(),
                                        _stream_ptr(stream)), "mrv_pp_build_table")
        return table

    def pp_motval(self, waypoints, T, t_start, focus: int, partners, table, horizon: int, flags: int = CHECK_ENV,
                  out=None, stream=None, **opts):
        """PP-ST-RRT MotVal (mrv_pp_motval_batch): candidates of robot ``focus`` (CUDA
        [M][1][K][S], T an int or CUDA int32 [M]) starting at CUDA int32 ``t_start`` [M],
        against the partner ``table`` -> CUDA uint8 [M]."""
        import torch
        b = self._batch(waypoints, T, n_robots=1)
        assert t_start.is_cuda and t_start.dtype == torch.int32 and t_start.numel() == b.n_motions
        if out is None:
            out = torch.empty(b.n_motions, dtype=torch.uint8, device=waypoints.device)
        o = self._opts(**opts)
        _check(lib().mrv_pp_motval_batch(self._h, C.byref(b), t_start.data_ptr(), int(focus), self._mask(partners),
                                         table.data_ptr(), int(horizon), flags, out.data_ptr(), _stream_ptr(stream),
                                         None if o is None else C.byref(o)), "mrv_pp_motval_batch")
        return out

    def run_host(self, waypoints, T, motval_flags: int = CHECK_ENV, out_valid=None, ffc_flags: int = 0, out_key=None,
                 chunk: int = 0, stream=None):
        """End-to-end call (mrv_run_host_batch): ``waypoints`` (and a per-motion ``T``) are
        HOST tensors (pin them for copy/compute overlap); MotVal into ``out_valid`` and/or
        FFC into ``out_key`` (CUDA tensors or pinned CPU tensors, None to skip).  Enqueued
        on ``stream``."""
        assert not waypoints.is_cuda and waypoints.dtype == torch_f32() and waypoints.dim() == 4
        assert waypoints.is_contiguous(), "waypoints must be contiguous"
        M, n, K, S = waypoints.shape
        if n != self.n_robots:
            raise ValueError(f"waypoints have {n} robots, scene has {self.n_robots}")
        if isinstance(T, int):
            b = MotionBatch(M, K, S, waypoints.data_ptr(), None, T, None)
        else:
            assert not T.is_cuda and T.dim() == 1 and T.numel() == M and T.is_contiguous()
            b = MotionBatch(M, K, S, waypoints.data_ptr(), T.data_ptr(), 0, None)
        _check(lib().mrv_run_host_batch(self._h, C.byref(b), motval_flags,
                                        None if out_valid is None else out_valid.data_ptr(), ffc_flags,
                                        None if out_key is None else out_key.data_ptr(), int(chunk),
                                        _stream_ptr(stream)), "mrv_run_host_batch")

    def fk_states(self, waypoints, T, motion, t, stream=None):
        """SpheresFK export: CUDA f32 [Q][total_spheres][3] world centres at (motion[q], t[q])."""
        import torch
        b = self._batch(waypoints, T)
        assert motion.dtype == torch.int64 and t.dtype == torch.int32 and motion.numel() == t.numel()
        out = torch.empty((motion.numel(), self.total_spheres, 3), dtype=torch.float32, device=waypoints.device)
        _check(lib().mrv_fk_states(self._h, C.byref(b), motion.numel(), motion.data_ptr(), t.data_ptr(),
                                   out.data_ptr(), _stream_ptr(stream)), "mrv_fk_states")
        return out

    def decode(self, key: int):
        t, i, j = C.c_int32(), C.c_int32(), C.c_int32()
        _check(lib().mrv_decode_conflict(self._h, int(key) & 0xFFFFFFFF, C.byref(t), C.byref(i), C.byref(j)),
               "mrv_decode_conflict")
        return None if t.value < 0 else (t.value, i.value, j.value)


def torch_f32():
    import torch
    return torch.float32


def keys_u32(keys) -> np.ndarray:
    """int32 device/host tensor of FFC keys -> numpy uint32."""
    a = keys.cpu().numpy() if hasattr(keys, "cpu") else np.asarray(keys)
    return a.view(np.uint32) if a.dtype == np.int32 else a.astype(np.uint32)


def to_device(mot, device="cuda"):
    """gen.Motions -> (CUDA f32 waypoints, CUDA int32 T or int)."""
    import torch
    wp = torch.from_numpy(np.ascontiguousarray(mot.waypoints)).to(device)
    rt = getattr(mot, "robot_timesteps", None)
    if rt is not None:
        return wp, torch.from_numpy(np.ascontiguousarray(rt, dtype=np.int32)).to(device)
    T = int(mot.fixed_timesteps) if mot.n_timesteps is None else torch.from_numpy(
        np.ascontiguousarray(mot.n_timesteps, dtype=np.int32)).to(device)
    return wp, T
