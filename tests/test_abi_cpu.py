"""C-ABI checks that need no GPU: the library loads, exports every symbol include/p2s.h declares,
and rejects bad arguments synchronously without touching the device."""
import ctypes
import os
import re

import numpy as np
import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
HEADER = os.path.join(ROOT, "include", "p2s.h")


def declared_symbols():
    src = open(HEADER).read()
    return sorted(set(re.findall(r"P2S_API\s+[\w\s\*]+?\b(p2s_\w+)\s*\(", src)))


@pytest.fixture(scope="module")
def lib():
    from paper_2107_11627_b200 import build, p2s
    build.build()  # nvcc cross-compiles sm_100a without a GPU
    return p2s.load_library()


def test_header_declares_the_boundary():
    syms = declared_symbols()
    for s in ("p2s_init", "p2s_render", "p2s_render_host", "p2s_destroy", "p2s_status_string",
              "p2s_debug_beta", "p2s_debug_blur", "p2s_reserve", "p2s_get_info"):
        assert s in syms


def test_library_exports_every_declared_symbol(lib):
    out = os.popen(f"nm -D --defined-only {lib._name}").read()
    exported = set(re.findall(r"\bT (p2s_\w+)", out))
    missing = [s for s in declared_symbols() if s not in exported]
    assert not missing, missing
    from paper_2107_11627_b200 import p2s
    assert set(p2s.EXPORTED) == set(declared_symbols())


def test_status_strings(lib):
    for code, name in enumerate(["P2S_OK", "P2S_ERR_INVALID_ARG", "P2S_ERR_UNSUPPORTED", "P2S_ERR_CUDA",
                                 "P2S_ERR_OOM"]):
        assert lib.p2s_status_string(code).decode() == name


def test_invalid_arguments_are_rejected_before_any_cuda_call(lib):
    from paper_2107_11627_b200 import p2s
    h = ctypes.c_void_p()
    assert lib.p2s_init(None, None, ctypes.byref(h)) == p2s.P2S_ERR_INVALID_ARG
    taps = np.zeros((4, 5, 5), np.float32)
    w = {k: np.zeros(s, np.float32) for k, s in (("W1", (8, 33)), ("b1", 8), ("W2", (8, 8)), ("b2", 8),
                                                 ("W3", (5, 8)), ("b3", 5))}
    b = p2s._Basis(4, 5, taps.ctypes.data)
    m = p2s._Mlp(33, 8, 8, 5, *(w[k].ctypes.data for k in ("W1", "b1", "W2", "b2", "W3", "b3")))
    # n_out (5) != K (4): inconsistent dims
    assert lib.p2s_init(ctypes.byref(b), ctypes.byref(m), ctypes.byref(h)) == p2s.P2S_ERR_INVALID_ARG
    m.n_out = 4
    b.S = 4  # even taps: outside the envelope
    assert lib.p2s_init(ctypes.byref(b), ctypes.byref(m), ctypes.byref(h)) == p2s.P2S_ERR_UNSUPPORTED
    b.S, b.K, m.n_out = 5, 200, 200  # K > 128
    assert lib.p2s_init(ctypes.byref(b), ctypes.byref(m), ctypes.byref(h)) == p2s.P2S_ERR_UNSUPPORTED
    im = p2s._Image(0, 1, 1, 8, 8)
    assert lib.p2s_render(None, im, None, None, None, None) == p2s.P2S_ERR_INVALID_ARG
    assert lib.p2s_debug_beta(None, None, 1, 1, 1, None, None) == p2s.P2S_ERR_INVALID_ARG
    assert lib.p2s_reserve(None, 1, 1, 1, 1) == p2s.P2S_ERR_INVALID_ARG
    lib.p2s_destroy(None)  # no-op


def test_init_without_a_gpu_fails_cleanly(lib):
    """On a box without a B200 the library reports an error instead of crashing (no CPU fallback)."""
    torch = pytest.importorskip("torch")
    if torch.cuda.is_available():
        pytest.skip("a GPU is present")
    from paper_2107_11627_b200 import p2s, synth
    inp = synth.make_inputs(synth.CONFIGS[1])
    with pytest.raises(p2s.P2SError) as e:
        p2s.Renderer(inp.basis, inp.mlp)
    assert e.value.status in (p2s.P2S_ERR_CUDA, p2s.P2S_ERR_UNSUPPORTED)


def test_sass_has_tcgen05_and_tma(lib):
    """The fused kernel is a tcgen05/TMA kernel (SASS evidence, B200_PROFILING.md)."""
    sass = os.popen(f"cuobjdump -sass {lib._name}").read()
    for mnem in ("UTCHMMA.2CTA", "LDTM", "UTMALDG"):
        assert mnem in sass, mnem
    assert "HMMA" not in sass.replace("UTCHMMA", "")
    # the UMMA issue loop must stay on the uniform datapath: descriptors in uniform registers,
    # no per-UMMA divergence/elect loops (a silent 1.5x slowdown when uniformity is lost)
    funcs = [f for f in sass.split("Function : ")[1:] if f.startswith("_ZN3p2s11k_fused_p2s")]
    assert len(funcs) == 4  # dense-field, anchor-grid and the two adjoint instantiations
    for fused in funcs:
        ins = [l.split("*/", 1)[1].strip() for l in fused.split("\n") if l.strip().startswith("/*") and "*/" in l
               and not l.strip().startswith("/* 0x")]
        mma = [n for n, l in enumerate(ins) if "UTCHMMA" in l]
        assert mma
        # the issue loop region: no divergence checks, no elect loops, no per-UMMA lane broadcasts
        region = ins[max(0, mma[0] - 60):mma[-1] + 60]
        for bad in ("BRA.DIV", "BRA.U.ANY", "R2UR.BROADCAST"):
            assert not any(bad in x for x in region), bad
        for n in mma:  # the 12 instructions feeding each UMMA must use uniform operands only
            assert not any("R2UR.BROADCAST" in x for x in ins[max(0, n - 12):n]), ins[max(0, n - 12):n + 1]


def test_sass_adjoint_image_kernel(lib):
    """dL/dI (k_adjoint_image): pair UMMAs fed by TMA, a uniform issue loop (SASS evidence)."""
    sass = os.popen(f"cuobjdump -sass {lib._name}").read()
    funcs = [f for f in sass.split("Function : ")[1:] if f.startswith("_ZN3p2s15k_adjoint_image")]
    assert len(funcs) == 1
    ins = [l.split("*/", 1)[1].strip() for l in funcs[0].split("\n") if l.strip().startswith("/*") and "*/" in l
           and not l.strip().startswith("/* 0x")]
    mma = [n for n, l in enumerate(ins) if "UTCHMMA.2CTA" in l]
    # U comes in as 64-column 128B-swizzled boxes (3-D map), the basis taps as a 2-D map
    assert len(mma) == 2 and any("UTMALDG.3D" in l for l in ins) and any("UTMALDG.2D" in l for l in ins)
    region = ins[max(0, mma[0] - 40):mma[-1] + 20]
    for bad in ("BRA.DIV", "BRA.U.ANY", "R2UR.BROADCAST"):
        assert not any(bad in x for x in region), bad


def test_sass_mlp_backward_kernel(lib):
    """dL/dz (k_mlp_backward resident and k_mlp_backward_s streamed, both bias modes): 1-CTA UMMAs
    (kind::f16), TMEM loads, weights brought in by bulk async copies, and no HMMA (SASS evidence)."""
    sass = os.popen(f"cuobjdump -sass {lib._name}").read()
    funcs = [f for f in sass.split("Function : ")[1:] if f.startswith("_ZN3p2s14k_mlp_backward")
             or f.startswith("_ZN3p2s16k_mlp_backward_s")]
    assert len(funcs) == 4
    for f in funcs:
        assert "UTCHMMA" in f and "UTCHMMA.2CTA" not in f
        assert "LDTM" in f and "UBLKCP" in f
        assert "HMMA" not in f.replace("UTCHMMA", "")


def test_plain_c_client_builds_against_the_abi(lib):
    """examples/render_c_abi.c (C99, gcc, no C++ or PyTorch) compiles and links against the header
    and libp2s.so alone: the boundary is a C ABI."""
    from paper_2107_11627_b200 import build
    exe = build.build_example()
    assert os.path.exists(exe)
    deps = os.popen(f"ldd {exe}").read()
    assert "libp2s.so" in deps and "torch" not in deps
