"""Python binding of the C ABI in include/p2s.h (argument marshalling only).

Every step of the hot path runs in libp2s.so (sm_100a kernels); this module only turns
numpy arrays / torch CUDA tensors into the plain pointers, sizes and stream handles the
C ABI takes. There is no CPU fallback: if the library is missing or the device is not a
B200 the calls raise.

Names follow the ABI: ``p2s_init`` -> :class:`Renderer`, ``p2s_render`` ->
:meth:`Renderer.render`, ``p2s_render_host`` -> :meth:`Renderer.render_host`,
``p2s_debug_beta`` / ``p2s_debug_blur`` -> :meth:`Renderer.debug_beta` / :meth:`Renderer.debug_blur`.
"""
from __future__ import annotations

import ctypes
import os
from typing import Optional

import numpy as np

_PKG = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.environ.get("P2S_LIB", os.path.join(_PKG, "libp2s.so"))

P2S_OK, P2S_ERR_INVALID_ARG, P2S_ERR_UNSUPPORTED, P2S_ERR_CUDA, P2S_ERR_OOM = range(5)

EXPORTED = ("p2s_init", "p2s_render", "p2s_render_host", "p2s_reserve", "p2s_set_profile_events",
            "p2s_get_info", "p2s_destroy", "p2s_status_string", "p2s_last_cuda_error",
            "p2s_debug_beta", "p2s_debug_blur", "p2s_debug_profile_buffer",
            "p2s_render_anchors", "p2s_render_anchors_host", "p2s_debug_blur_anchors",
            "p2s_render_sequence", "p2s_sampler_init", "p2s_sample_anchors", "p2s_sampler_destroy",
            "p2s_backward", "p2s_render_color", "p2s_mlp_backward", "p2s_interp_anchors",
            "p2s_anchors_backward", "p2s_backward_color", "p2s_sampler_init_dense", "p2s_reserve_ex")
# p2s_reserve_ex workspace bits (include/p2s.h)
RESERVE_RENDER, RESERVE_HOST, RESERVE_ADJOINT, RESERVE_ADJOINT_IMAGE = 1, 2, 4, 8


class P2SError(RuntimeError):
    def __init__(self, status: int, what: str):
        lib = _lib
        name = lib.p2s_status_string(status).decode() if lib else str(status)
        cuda = lib.p2s_last_cuda_error().decode() if lib else ""
        super().__init__(f"{what}: {name}" + (f" ({cuda})" if cuda and status == P2S_ERR_CUDA else ""))
        self.status = status


class _Basis(ctypes.Structure):
    _fields_ = [("K", ctypes.c_int), ("S", ctypes.c_int), ("taps", ctypes.c_void_p)]


class _Mlp(ctypes.Structure):
    _fields_ = [("n_in", ctypes.c_int), ("h1", ctypes.c_int), ("h2", ctypes.c_int), ("n_out", ctypes.c_int),
                ("W1", ctypes.c_void_p), ("b1", ctypes.c_void_p), ("W2", ctypes.c_void_p),
                ("b2", ctypes.c_void_p), ("W3", ctypes.c_void_p), ("b3", ctypes.c_void_p)]


class _Image(ctypes.Structure):
    _fields_ = [("data", ctypes.c_void_p), ("B", ctypes.c_int), ("C", ctypes.c_int), ("H", ctypes.c_int),
                ("W", ctypes.c_int)]


class Info(ctypes.Structure):
    _fields_ = [(n, ctypes.c_int) for n in ("K", "S", "n_in", "h1", "h2", "n_pad", "h1_pad", "h2_pad",
                                            "in_pad", "conv_steps", "smem_bytes", "kernels_per_render",
                                            "stage_bytes", "nring", "mlp_backward", "c1_plan", "c1_smem_bytes",
                                            "c1_nring", "c1_stage_bytes", "seq_plan", "seq_nring",
                                            "seq_stage_bytes")]

    def as_dict(self):
        return {n: getattr(self, n) for n, _ in self._fields_}


_lib = None


def load_library(path: str = LIB_PATH) -> ctypes.CDLL:
    """Loads libp2s.so (built by ``paper_2107_11627_b200.build``); raises if absent."""
    global _lib
    if _lib is not None:
        return _lib
    if not os.path.exists(path):
        raise ImportError(f"{path} is missing: run `python -m paper_2107_11627_b200.build` "
                          "(the CUDA path has no fallback)")
    lib = ctypes.CDLL(path)
    v, i, st = ctypes.c_void_p, ctypes.c_int, ctypes.c_int
    lib.p2s_init.argtypes = [ctypes.POINTER(_Basis), ctypes.POINTER(_Mlp), ctypes.POINTER(v)]
    lib.p2s_render.argtypes = [v, _Image, v, v, v, v]
    lib.p2s_render_host.argtypes = [v, v, i, i, i, i, v, v, v, v]
    lib.p2s_reserve.argtypes = [v, i, i, i, i]
    lib.p2s_reserve_ex.argtypes = [v, i, i, i, i, ctypes.c_uint]
    lib.p2s_set_profile_events.argtypes = [v, v, v]
    lib.p2s_get_info.argtypes = [v, ctypes.POINTER(Info)]
    lib.p2s_destroy.argtypes = [v]
    lib.p2s_destroy.restype = None
    lib.p2s_status_string.argtypes = [st]
    lib.p2s_status_string.restype = ctypes.c_char_p
    lib.p2s_last_cuda_error.argtypes = []
    lib.p2s_last_cuda_error.restype = ctypes.c_char_p
    lib.p2s_debug_beta.argtypes = [v, v, i, i, i, v, v]
    lib.p2s_debug_blur.argtypes = [v, _Image, v, v, v]
    lib.p2s_debug_profile_buffer.argtypes = [v, v]
    lib.p2s_render_anchors.argtypes = [v, _Image, v, i, v, v, v]
    lib.p2s_render_anchors_host.argtypes = [v, v, i, i, i, i, v, i, v, v, v]
    lib.p2s_debug_blur_anchors.argtypes = [v, _Image, v, i, v, v]
    lib.p2s_render_sequence.argtypes = [v, _Image, v, v, i, v, v]
    lib.p2s_sampler_init.argtypes = [i, i, ctypes.c_double, v, ctypes.POINTER(v)]
    lib.p2s_sample_anchors.argtypes = [v, ctypes.c_ulonglong, i, i, v, v]
    lib.p2s_sampler_init_dense.argtypes = [i, i, v, i, v, ctypes.POINTER(v)]
    lib.p2s_sampler_destroy.argtypes = [v]
    lib.p2s_backward.argtypes = [v, _Image, v, v, v, v, v, v, v]
    lib.p2s_render_color.argtypes = [v, _Image, v, v, v, v]
    lib.p2s_mlp_backward.argtypes = [v, v, v, i, i, i, v, v]
    lib.p2s_interp_anchors.argtypes = [v, i, i, i, i, i, v, v]
    lib.p2s_anchors_backward.argtypes = [v, i, i, i, i, i, v, v]
    lib.p2s_backward_color.argtypes = [v, _Image, v, v, v, v, v, v, v, v]
    lib.p2s_sampler_destroy.restype = None
    for name in ("p2s_init", "p2s_render", "p2s_render_host", "p2s_reserve", "p2s_set_profile_events",
                 "p2s_get_info", "p2s_debug_beta", "p2s_debug_blur", "p2s_debug_profile_buffer",
                 "p2s_render_anchors", "p2s_render_anchors_host", "p2s_debug_blur_anchors",
                 "p2s_render_sequence", "p2s_sampler_init", "p2s_sample_anchors", "p2s_backward",
                 "p2s_render_color", "p2s_mlp_backward", "p2s_interp_anchors", "p2s_anchors_backward",
                 "p2s_backward_color", "p2s_sampler_init_dense", "p2s_reserve_ex"):
        getattr(lib, name).restype = st
    _lib = lib
    return lib


def _check(status: int, what: str):
    if status != P2S_OK:
        raise P2SError(status, what)


def _f32(a) -> np.ndarray:
    return np.ascontiguousarray(a, dtype=np.float32)


def _dev_ptr(t, name, shape=None):
    import torch
    if not isinstance(t, torch.Tensor) or not t.is_cuda or t.dtype != torch.float32 or not t.is_contiguous():
        raise ValueError(f"{name} must be a contiguous float32 CUDA tensor")
    if shape is not None and tuple(t.shape) != tuple(shape):
        raise ValueError(f"{name} has shape {tuple(t.shape)}, expected {tuple(shape)}")
    return ctypes.c_void_p(t.data_ptr())


def _on(stream):
    """Allocations made for a call on `stream` come from that stream's caching-allocator pool, so
    a tensor the queued kernels still use is not handed to another stream when it is freed."""
    import contextlib
    import torch
    return torch.cuda.stream(stream) if stream is not None else contextlib.nullcontext()


def _empty(stream, shape, device):
    """torch.empty on `stream`'s allocator pool (see _on)."""
    import torch
    with _on(stream):
        return torch.empty(shape, device=device, dtype=torch.float32)


def _host_f32(a, name, shape):
    if not isinstance(a, np.ndarray) or a.dtype != np.float32 or not a.flags.c_contiguous:
        raise ValueError(f"{name} must be a C-contiguous float32 numpy array")
    if tuple(a.shape) != tuple(shape):
        raise ValueError(f"{name} has shape {tuple(a.shape)}, expected {tuple(shape)}")
    return a.ctypes.data


def _stream_handle(stream):
    import torch
    s = stream if stream is not None else torch.cuda.current_stream()
    return ctypes.c_void_p(s.cuda_stream)


def interp_anchors(anchors, H: int, W: int, out=None, stream=None):
    """p2s_interp_anchors: anchor grid [B,n_in,G,G] -> dense Zernike field [B,n_in,H,W] (CUDA)."""
    import torch
    lib = load_library()
    B, n_in, G, G2 = anchors.shape
    if G != G2:
        raise ValueError("anchors must be [B, n_in, G, G]")
    ap = _dev_ptr(anchors, "anchors")
    if out is None:
        out = _empty(stream, (B, n_in, H, W), anchors.device)
    _check(lib.p2s_interp_anchors(ap, B, n_in, G, H, W, _dev_ptr(out, "zernike_field", (B, n_in, H, W)),
                                  _stream_handle(stream)), "p2s_interp_anchors")
    return out


def anchors_backward(grad_zernike, G: int, out=None, stream=None):
    """p2s_anchors_backward: dL/dz [B,n_in,H,W] -> dL/dA [B,n_in,G,G] (CUDA)."""
    import torch
    lib = load_library()
    B, n_in, H, W = grad_zernike.shape
    gp = _dev_ptr(grad_zernike, "grad_zernike")
    if out is None:
        out = _empty(stream, (B, n_in, G, G), grad_zernike.device)
    _check(lib.p2s_anchors_backward(gp, B, n_in, G, H, W, _dev_ptr(out, "grad_anchors", (B, n_in, G, G)),
                                    _stream_handle(stream)), "p2s_anchors_backward")
    return out


class Renderer:
    """One p2s handle: device copies of the PSF basis phi_k and the P2S MLP weights."""

    def __init__(self, basis: np.ndarray, mlp: dict):
        lib = load_library()
        basis = _f32(basis)
        K, S, S2 = basis.shape
        assert S == S2
        self._keep = {k: _f32(v) for k, v in mlp.items()}
        m = self._keep
        h1, n_in = m["W1"].shape
        h2 = m["W2"].shape[0]
        n_out = m["W3"].shape[0]
        b = _Basis(K, S, basis.ctypes.data)
        ml = _Mlp(n_in, h1, h2, n_out, *(m[k].ctypes.data for k in ("W1", "b1", "W2", "b2", "W3", "b3")))
        h = ctypes.c_void_p()
        _check(lib.p2s_init(ctypes.byref(b), ctypes.byref(ml), ctypes.byref(h)), "p2s_init")
        self._h = h
        self.K, self.S, self.n_in = K, S, n_in
        self._lib = lib

    # -------------------------------------------------------------- device API
    def render(self, image, zernike, tilt=None, out=None, stream=None):
        """p2s_render on CUDA tensors: image [B,C,H,W], zernike [B,n_in,H,W], tilt [B,2,H,W]|None."""
        import torch
        B, C, H, W = image.shape
        im = _Image(_dev_ptr(image, "image").value, B, C, H, W)
        zp = _dev_ptr(zernike, "zernike_field", (B, self.n_in, H, W))
        tp = _dev_ptr(tilt, "tilt_field", (B, 2, H, W)) if tilt is not None else ctypes.c_void_p()
        if out is None:
            out = _empty(stream, image.shape, image.device)
        op = _dev_ptr(out, "out", (B, C, H, W))
        _check(self._lib.p2s_render(self._h, im, zp, tp, op, _stream_handle(stream)), "p2s_render")
        return out

    def backward(self, image, zernike, tilt, grad_out, want_beta=True, want_tilt=True, want_image=False,
                 want_zernike=False, stream=None):
        """p2s_backward: (dL/dbeta [B,K,H,W] | None, dL/dt [B,2,H,W] | None) of the
        frames render(image, zernike, tilt) gives, for upstream grad_out [B,C,H,W]; with
        want_image=True a third entry dL/dI [B,C,H,W]; with want_zernike=True a fourth entry
        dL/dz [B,n_in,H,W] (p2s_mlp_backward on dL/dbeta)."""
        import torch
        B, C, H, W = image.shape
        im = _Image(_dev_ptr(image, "image").value, B, C, H, W)
        zp = _dev_ptr(zernike, "zernike_field", (B, self.n_in, H, W))
        tp = _dev_ptr(tilt, "tilt_field", (B, 2, H, W)) if tilt is not None else ctypes.c_void_p()
        gp = _dev_ptr(grad_out, "grad_out", (B, C, H, W))
        gb = _empty(stream, (B, self.K, H, W), image.device) \
            if (want_beta or want_zernike) else None
        gt = _empty(stream, (B, 2, H, W), image.device) if want_tilt else None
        gi = _empty(stream, (B, C, H, W), image.device) if want_image else None
        _check(self._lib.p2s_backward(self._h, im, zp, tp, gp,
                                      _dev_ptr(gb, "grad_beta") if gb is not None else ctypes.c_void_p(),
                                      _dev_ptr(gt, "grad_tilt") if gt is not None else ctypes.c_void_p(),
                                      _dev_ptr(gi, "grad_image") if gi is not None else ctypes.c_void_p(),
                                      _stream_handle(stream)), "p2s_backward")
        if want_zernike:
            gz = self.mlp_backward(zernike, gb, stream=stream)
            return (gb if want_beta else None), gt, gi, gz
        return (gb, gt, gi) if want_image else (gb, gt)

    def backward_anchors(self, image, anchors, tilt, grad_out, want_tilt=True, want_image=False, stream=None):
        """The adjoint of render_anchors: (dL/dA [B,n_in,G,G], dL/dt | None, dL/dI | None) for upstream
        grad_out [B,C,H,W] — interp_anchors -> p2s_backward (dL/dbeta) -> p2s_mlp_backward ->
        p2s_anchors_backward, all on the device."""
        B, C, H, W = image.shape
        G = anchors.shape[-1]
        z = interp_anchors(anchors, H, W, stream=stream)
        gb, gt, gi, gz = self.backward(image, z, tilt, grad_out, want_beta=False, want_tilt=want_tilt,
                                       want_image=want_image, want_zernike=True, stream=stream)
        return anchors_backward(gz, G, stream=stream), gt, gi

    def backward_color(self, image, zernike_color, tilt, grad_out, want_beta=True, want_tilt=True, want_image=False,
                       want_zernike=False, stream=None):
        """p2s_backward_color: (dL/dbeta [B,C,K,H,W], dL/dt [B,2,H,W], dL/dI [B,C,H,W], dL/dz [B,C,n_in,H,W])
        of render_color (entries None when not wanted)."""
        import torch
        B, C, H, W = image.shape
        im = _Image(_dev_ptr(image, "image").value, B, C, H, W)
        zp = _dev_ptr(zernike_color, "zernike_field", (B, C, self.n_in, H, W))
        tp = _dev_ptr(tilt, "tilt_field", (B, 2, H, W)) if tilt is not None else ctypes.c_void_p()
        gp = _dev_ptr(grad_out, "grad_out", (B, C, H, W))
        gb = _empty(stream, (B, C, self.K, H, W), image.device) if want_beta else None
        gt = _empty(stream, (B, 2, H, W), image.device) if want_tilt else None
        gi = _empty(stream, (B, C, H, W), image.device) if want_image else None
        gz = _empty(stream, (B, C, self.n_in, H, W), image.device) if want_zernike else None
        ptr = lambda t, n: _dev_ptr(t, n) if t is not None else ctypes.c_void_p()  # noqa: E731
        _check(self._lib.p2s_backward_color(self._h, im, zp, tp, gp, ptr(gb, "grad_beta"), ptr(gt, "grad_tilt"),
                                            ptr(gi, "grad_image"), ptr(gz, "grad_zernike"), _stream_handle(stream)),
               "p2s_backward_color")
        return gb, gt, gi, gz

    def mlp_backward(self, zernike, grad_beta, out=None, stream=None):
        """p2s_mlp_backward: dL/dz [B,n_in,H,W] through the P2S MLP for dL/dbeta [B,K,H,W]."""
        import torch
        B, n_in, H, W = zernike.shape
        zp = _dev_ptr(zernike, "zernike_field", (B, self.n_in, H, W))
        bp = _dev_ptr(grad_beta, "grad_beta", (B, self.K, H, W))
        if out is None:
            out = _empty(stream, zernike.shape, zernike.device)
        _check(self._lib.p2s_mlp_backward(self._h, zp, bp, B, H, W, _dev_ptr(out, "grad_zernike", (B, n_in, H, W)),
                                          _stream_handle(stream)), "p2s_mlp_backward")
        return out

    def debug_beta(self, zernike, out=None, stream=None):
        import torch
        B, n_in, H, W = zernike.shape
        if out is None:
            out = _empty(stream, (B, self.K, H, W), zernike.device)
        _check(self._lib.p2s_debug_beta(self._h, _dev_ptr(zernike, "zernike_field", (B, self.n_in, H, W)),
                                        B, H, W, _dev_ptr(out, "beta_out", (B, self.K, H, W)),
                                        _stream_handle(stream)), "p2s_debug_beta")
        return out

    def debug_blur(self, image, zernike, out=None, stream=None):
        import torch
        B, C, H, W = image.shape
        if out is None:
            out = _empty(stream, image.shape, image.device)
        im = _Image(_dev_ptr(image, "image").value, B, C, H, W)
        _check(self._lib.p2s_debug_blur(self._h, im, _dev_ptr(zernike, "zernike_field", (B, self.n_in, H, W)),
                                        _dev_ptr(out, "J_out", (B, C, H, W)), _stream_handle(stream)),
               "p2s_debug_blur")
        return out

    def render_anchors(self, image, anchors, tilt=None, out=None, stream=None):
        """p2s_render_anchors: Zernike coefficients from an anchor grid [B,n_in,G,G]."""
        import torch
        B, C, H, W = image.shape
        G = anchors.shape[-1]
        im = _Image(_dev_ptr(image, "image").value, B, C, H, W)
        ap = _dev_ptr(anchors, "anchors", (B, self.n_in, G, G))
        tp = _dev_ptr(tilt, "tilt_field", (B, 2, H, W)) if tilt is not None else ctypes.c_void_p()
        if out is None:
            out = _empty(stream, image.shape, image.device)
        _check(self._lib.p2s_render_anchors(self._h, im, ap, G, tp, _dev_ptr(out, "out", (B, C, H, W)),
                                            _stream_handle(stream)), "p2s_render_anchors")
        return out

    def render_color(self, image, zernike, tilt=None, out=None, stream=None):
        """p2s_render_color: per-channel Zernike fields zernike [B,C,n_in,H,W]."""
        import torch
        B, C, H, W = image.shape
        im = _Image(_dev_ptr(image, "image").value, B, C, H, W)
        zp = _dev_ptr(zernike, "zernike_field", (B, C, self.n_in, H, W))
        tp = _dev_ptr(tilt, "tilt_field", (B, 2, H, W)) if tilt is not None else ctypes.c_void_p()
        if out is None:
            out = _empty(stream, image.shape, image.device)
        _check(self._lib.p2s_render_color(self._h, im, zp, tp, _dev_ptr(out, "out", (B, C, H, W)),
                                          _stream_handle(stream)), "p2s_render_color")
        return out

    def render_sequence(self, image, zernike, tilt=None, out=None, stream=None):
        """p2s_render_sequence: one image [1,C,H,W], F frames of Zernike [F,n_in,H,W] / tilt [F,2,H,W]."""
        import torch
        _, C, H, W = image.shape
        F = zernike.shape[0]
        im = _Image(_dev_ptr(image, "image", (1, C, H, W)).value, 1, C, H, W)
        zp = _dev_ptr(zernike, "zernike_field", (F, self.n_in, H, W))
        tp = _dev_ptr(tilt, "tilt_field", (F, 2, H, W)) if tilt is not None else ctypes.c_void_p()
        if out is None:
            out = _empty(stream, (F, C, H, W), image.device)
        _check(self._lib.p2s_render_sequence(self._h, im, zp, tp, F, _dev_ptr(out, "out", (F, C, H, W)),
                                             _stream_handle(stream)), "p2s_render_sequence")
        return out

    def debug_blur_anchors(self, image, anchors, out=None, stream=None):
        import torch
        B, C, H, W = image.shape
        G = anchors.shape[-1]
        if out is None:
            out = _empty(stream, image.shape, image.device)
        im = _Image(_dev_ptr(image, "image").value, B, C, H, W)
        _check(self._lib.p2s_debug_blur_anchors(self._h, im, _dev_ptr(anchors, "anchors", (B, self.n_in, G, G)), G,
                                                _dev_ptr(out, "J_out", (B, C, H, W)), _stream_handle(stream)),
               "p2s_debug_blur_anchors")
        return out

    def render_anchors_host(self, image: np.ndarray, anchors: np.ndarray, tilt: Optional[np.ndarray],
                            out: np.ndarray, stream=None) -> np.ndarray:
        """p2s_render_anchors_host: host buffers in and out (copies inside), synchronous."""
        B, C, H, W = image.shape
        G = anchors.shape[-1]
        ip = _host_f32(image, "image", (B, C, H, W))
        ap = _host_f32(anchors, "anchors", (B, self.n_in, G, G))
        tp = _host_f32(tilt, "tilt", (B, 2, H, W)) if tilt is not None else None
        op = _host_f32(out, "out", (B, C, H, W))
        _check(self._lib.p2s_render_anchors_host(self._h, ip, B, C, H, W, ap, G, tp, op, _stream_handle(stream)),
               "p2s_render_anchors_host")
        return out

    # -------------------------------------------------------------- host API (e2e)
    def render_host(self, image: np.ndarray, zernike: np.ndarray, tilt: Optional[np.ndarray],
                    out: np.ndarray, stream=None) -> np.ndarray:
        """p2s_render_host: host buffers in and out (copies inside), synchronous."""
        B, C, H, W = image.shape
        ip = _host_f32(image, "image", (B, C, H, W))
        zp = _host_f32(zernike, "zernike", (B, self.n_in, H, W))
        tp = _host_f32(tilt, "tilt", (B, 2, H, W)) if tilt is not None else None
        op = _host_f32(out, "out", (B, C, H, W))
        _check(self._lib.p2s_render_host(self._h, ip, B, C, H, W, zp, tp, op, _stream_handle(stream)),
               "p2s_render_host")
        return out

    def reserve(self, B, C, H, W, host=False, adjoint=False, adjoint_image=False):
        """p2s_reserve (render workspace), or p2s_reserve_ex when the host-path staging or the
        adjoint workspaces are asked for too."""
        what = RESERVE_RENDER | (RESERVE_HOST if host else 0) | (RESERVE_ADJOINT if adjoint else 0) | \
            (RESERVE_ADJOINT_IMAGE if adjoint_image else 0)
        if what == RESERVE_RENDER:
            _check(self._lib.p2s_reserve(self._h, B, C, H, W), "p2s_reserve")
        else:
            _check(self._lib.p2s_reserve_ex(self._h, B, C, H, W, what), "p2s_reserve_ex")

    def set_profile_events(self, ev_begin=None, ev_end=None):
        """p2s_set_profile_events with torch.cuda.Event objects (created on first use)."""
        for ev in (ev_begin, ev_end):
            if ev is not None and not ev.cuda_event:
                ev.record()  # torch creates the CUDA event lazily on its first record
        a = ctypes.c_void_p(ev_begin.cuda_event) if ev_begin is not None else ctypes.c_void_p()
        b = ctypes.c_void_p(ev_end.cuda_event) if ev_end is not None else ctypes.c_void_p()
        _check(self._lib.p2s_set_profile_events(self._h, a, b), "p2s_set_profile_events")

    def debug_profile_buffer(self, counters=None):
        """Profiling builds only (P2S_LIB=libp2s_prof.so): per-CTA role timers into `counters`."""
        ptr = ctypes.c_void_p(counters.data_ptr()) if counters is not None else ctypes.c_void_p()
        _check(self._lib.p2s_debug_profile_buffer(self._h, ptr), "p2s_debug_profile_buffer")

    def info(self) -> dict:
        inf = Info()
        _check(self._lib.p2s_get_info(self._h, ctypes.byref(inf)), "p2s_get_info")
        return inf.as_dict()

    def close(self):
        if getattr(self, "_h", None):
            self._lib.p2s_destroy(self._h)
            self._h = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass


class Sampler:
    """Correlated anchor-grid sampler (include/p2s.h p2s_sampler_*): stand-in
    separable covariance R (x) s (x) s (reading N3), Philox4x32-10 + Box-Muller normals."""

    def __init__(self, G: int, n_in: int, corr_len: float = 0.0, mode_cov: Optional[np.ndarray] = None,
                 spatial_cov: Optional[np.ndarray] = None, is_factor: bool = False):
        """Separable stand-in (corr_len; p2s_sampler_init), or -- with spatial_cov [G^2, G^2] fp64 --
        a dense pre-computed spatial correlation (or its lower Cholesky factor when is_factor;
        p2s_sampler_init_dense, the tensor-core path)."""
        lib = load_library()
        self._lib = lib
        self.G, self.n_in = G, n_in
        self._h = None
        mp = ctypes.c_void_p()
        if mode_cov is not None:
            self._keep = np.ascontiguousarray(mode_cov, np.float64)
            if self._keep.shape != (n_in, n_in):
                raise ValueError("mode_cov must be [n_in, n_in]")
            mp = ctypes.c_void_p(self._keep.ctypes.data)
        h = ctypes.c_void_p()
        if spatial_cov is not None:
            c = np.ascontiguousarray(spatial_cov, np.float64)
            if c.shape != (G * G, G * G):
                raise ValueError("spatial_cov must be [G*G, G*G]")
            _check(lib.p2s_sampler_init_dense(G, n_in, ctypes.c_void_p(c.ctypes.data), int(bool(is_factor)), mp,
                                              ctypes.byref(h)), "p2s_sampler_init_dense")
        else:
            _check(lib.p2s_sampler_init(G, n_in, float(corr_len), mp, ctypes.byref(h)), "p2s_sampler_init")
        self._h = h

    def sample(self, seed: int, frame0: int, F: int, out=None, stream=None):
        """Anchors [F, n_in, G, G] (CUDA fp32) of frames frame0 .. frame0 + F - 1."""
        import torch
        if out is None:
            out = _empty(stream, (F, self.n_in, self.G, self.G), "cuda")
        _check(self._lib.p2s_sample_anchors(self._h, seed, frame0, F,
                                            _dev_ptr(out, "anchors", (F, self.n_in, self.G, self.G)),
                                            _stream_handle(stream)), "p2s_sample_anchors")
        return out

    def close(self):
        if self._h:
            self._lib.p2s_sampler_destroy(self._h)
            self._h = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass
