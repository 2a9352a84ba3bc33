"""CPU-side checks of the C-ABI boundary: the library builds for sm_100a, loads, and exports
every entry point include/bnn.h declares; the Python binding mirrors the C structs."""
import ctypes as C
import os
import re
import subprocess

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
HEADER = os.path.join(ROOT, "include", "bnn.h")


def _declared():
    src = open(HEADER).read()
    src = re.sub(r"/\*.*?\*/", "", src, flags=re.S)
    return sorted(set(re.findall(r"\b(bnn_[a-z0-9_]+)\s*\(", src)))


def test_header_declares_the_boundary():
    names = _declared()
    for required in ["bnn_init", "bnn_elbo_step", "bnn_predict", "bnn_destroy", "bnn_last_error",
                     "bnn_get_unique_id", "bnn_elbo_partial", "bnn_finalize", "bnn_eps_fill"]:
        assert required in names


def test_library_exports_every_declared_symbol():
    from paper_2604_04736_b200 import build
    so = build.build()
    lib = C.CDLL(so)
    missing = [n for n in _declared() if not hasattr(lib, n)]
    assert not missing, missing


def test_binding_struct_sizes_match_header(tmp_path):
    """The ctypes structs against the C compiler's layout of include/bnn.h: sizeof and the
    offset of every field (a small C program compiled with gcc against the header)."""
    from paper_2604_04736_b200 import native
    structs = {"bnn_model_desc": native.BnnModelDesc, "bnn_config": native.BnnConfig,
               "bnn_tensor_info": native.BnnTensorInfo, "bnn_adam": native.BnnAdam}
    lines = ["#include <stdio.h>", "#include <stddef.h>", '#include "bnn.h"', "int main(void) {"]
    for cname, py in structs.items():
        lines.append(f'printf("{cname} size %zu\\n", sizeof({cname}));')
        for f, _ in py._fields_:
            lines.append(f'printf("{cname} {f} %zu\\n", offsetof({cname}, {f}));')
    lines.append("return 0; }")
    src = tmp_path / "layout.c"
    src.write_text("\n".join(lines))
    exe = tmp_path / "layout"
    subprocess.check_call(["gcc", "-std=c11", "-I", os.path.join(ROOT, "include"), str(src), "-o", str(exe)])
    out = subprocess.check_output([str(exe)]).decode().split("\n")
    got = {tuple(l.split()[:2]): int(l.split()[2]) for l in out if l.strip()}
    for cname, py in structs.items():
        assert got[(cname, "size")] == C.sizeof(py), cname
        for f, _ in py._fields_:
            assert got[(cname, f)] == getattr(py, f).offset, (cname, f)


def test_init_without_gpu_fails_loudly():
    """No CPU fallback: on a box without a GPU bnn_init must fail with BNN_ERR_CUDA."""
    import torch
    if torch.cuda.is_available():
        pytest.skip("GPU present")
    from paper_2604_04736_b200 import native
    lib = native.lib()
    d = native.model_desc(dict(kind="mlp", widths=[8, 16, 1], loss="mse"))
    cfg = native.BnnConfig()
    cfg.precision, cfg.mode, cfg.world, cfg.max_B_loc, cfg.max_S_loc = 0, 0, 1, 32, 4
    cfg.dataset_size = 1024.0
    h = C.c_void_p()
    rc = lib.bnn_init(C.byref(d), C.byref(cfg), C.byref(h))
    assert rc == 5
    assert b"no CUDA device" in lib.bnn_last_error(None)


def test_config_invariants_rejected_before_device_use():
    from paper_2604_04736_b200 import native
    lib = native.lib()
    d = native.model_desc(dict(kind="mlp", widths=[8, 16, 1], loss="mse"))
    cfg = native.BnnConfig()
    cfg.precision, cfg.mode, cfg.K, cfg.G, cfg.rank, cfg.world = 0, 2, 3, 2, 0, 4
    cfg.max_B_loc, cfg.max_S_loc, cfg.dataset_size = 32, 4, 1.0
    h = C.c_void_p()
    assert lib.bnn_init(C.byref(d), C.byref(cfg), C.byref(h)) == 2
    assert b"world == K*G" in lib.bnn_last_error(None)
