"""GPU helpers of the scene generator (input generation only; see csrc/gen.cu).

libscenegen.so is built in-tree by build() (called from
__graft_entry__.build()).  Used for C5, whose ~1.9e8 leaves and 512 bumps
would take far too long on the host."""
from __future__ import annotations

import ctypes as C
import os
import subprocess

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
SRC = os.path.join(HERE, "csrc", "gen.cu")
LIB = os.path.join(HERE, "libscenegen.so")
NVCC = os.environ.get("NVCC", "/usr/local/cuda/bin/nvcc")
_lib = None


def build(force: bool = False) -> str:
    if force or not os.path.exists(LIB) or os.path.getmtime(LIB) < os.path.getmtime(SRC):
        cmd = [NVCC, "-gencode", "arch=compute_100a,code=sm_100a", "-O3", "-shared", "-Xcompiler", "-fPIC",
               "-o", LIB, SRC, "-lcudart_static"]
        r = subprocess.run(cmd, capture_output=True, text=True)
        if r.returncode != 0:
            raise RuntimeError("nvcc failed for scenegen/csrc/gen.cu:\n" + r.stderr[-4000:])
    return LIB


def lib():
    global _lib
    if _lib is None:
        if not os.path.exists(LIB):
            build()
        L = C.CDLL(LIB)
        vp, i32, i64 = C.c_void_p, C.c_int32, C.c_int64
        L.sg_shell_refine.argtypes = [vp, vp, i64, i32, vp, i32, C.c_double, vp, vp]
        L.sg_shell_bumps.argtypes = [vp, vp, vp, i64, i32, vp, i32, vp, vp, vp]
        _lib = L
    return _lib


def _stream():
    import torch
    return C.c_void_p(torch.cuda.current_stream().cuda_stream)


def shell_refine_flags(anchor, tree, level: int, sources: np.ndarray, c: float):
    """uint8 flag per leaf: exact-shell element centre within c 2^-level of a source."""
    import torch
    n = int(tree.shape[0])
    flag = torch.empty(n, dtype=torch.uint8, device=anchor.device)
    src = torch.as_tensor(np.ascontiguousarray(sources, dtype=np.float64), device=anchor.device)
    st = lib().sg_shell_refine(anchor.data_ptr(), tree.data_ptr(), n, int(level), src.data_ptr(), src.shape[0],
                               float(c), flag.data_ptr(), _stream())
    if st != 0:
        raise RuntimeError(f"sg_shell_refine failed ({st})")
    return flag.bool()


def shell_bumps_field(anchor, tree, level, P: int, centers, sigma, amp):
    """fp32 nodal field [n][(P+1)^3] of a Gaussian-bump sum (fp64 inside) and max |f|."""
    import torch
    n = int(tree.shape[0])
    dev = anchor.device
    b = np.concatenate([np.asarray(centers, np.float64), (1.0 / (2.0 * np.asarray(sigma, np.float64) ** 2))[:, None],
                        np.asarray(amp, np.float64)[:, None]], axis=1)
    bt = torch.as_tensor(np.ascontiguousarray(b), device=dev)
    out = torch.empty((n, (P + 1) ** 3), dtype=torch.float32, device=dev)
    fmax = torch.zeros(1, dtype=torch.int64, device=dev)
    st = lib().sg_shell_bumps(anchor.data_ptr(), tree.data_ptr(), level.data_ptr(), n, int(P), bt.data_ptr(),
                              int(b.shape[0]), out.data_ptr(), fmax.data_ptr(), _stream())
    if st != 0:
        raise RuntimeError(f"sg_shell_bumps failed ({st})")
    F = float(np.frombuffer(fmax.cpu().numpy().tobytes(), dtype=np.float64)[0])
    return out, F


def _spread3_t(v):
    """Bit spread of an int64 tensor (18 bits) for Morton keys (x fastest)."""
    x = v & 0x3FFFF
    x = (x | (x << 32)) & 0x001F00000000FFFF
    x = (x | (x << 16)) & 0x001F0000FF0000FF
    x = (x | (x << 8)) & 0x100F00F00F00F00F
    x = (x | (x << 4)) & 0x10C30C30C30C30C3
    x = (x | (x << 2)) & 0x1249249249249249
    return x


def morton_key_t(anchor):
    a = anchor.to(torch_int64())
    return _spread3_t(a[:, 0]) | (_spread3_t(a[:, 1]) << 1) | (_spread3_t(a[:, 2]) << 2)


def torch_int64():
    import torch
    return torch.int64


def refine_leaves_shell(level0: int, maxlevel: int, sources, c: float, device):
    """Adaptive 6-tree shell forest on the GPU (SURVEY R20 rule), SFC order."""
    import torch
    from . import uniform_leaves, MAXLEVEL
    anc_np, tree_np, _ = uniform_leaves(6, level0)
    anc = torch.as_tensor(anc_np, device=device)
    tree = torch.as_tensor(tree_np, device=device)
    done = []
    for L in range(level0, maxlevel + 1):
        if anc.shape[0] == 0:
            break
        if L == maxlevel:
            sel = torch.zeros(anc.shape[0], dtype=torch.bool, device=device)
        else:
            sel = shell_refine_flags(anc.contiguous(), tree.contiguous(), L, sources, c)
        keep = ~sel
        done.append((anc[keep], tree[keep], torch.full((int(keep.sum()),), L, dtype=torch.int8, device=device)))
        pa, pt = anc[sel], tree[sel]
        h = 1 << (MAXLEVEL - L - 1)
        off = torch.tensor([[(c8 & 1) * h, ((c8 >> 1) & 1) * h, ((c8 >> 2) & 1) * h] for c8 in range(8)],
                           dtype=torch.int32, device=device)
        anc = (pa[None, :, :] + off[:, None, :]).reshape(-1, 3)
        tree = pt.repeat(8)
        del pa, pt, sel
    A = torch.cat([d[0] for d in done])
    T = torch.cat([d[1] for d in done])
    Lv = torch.cat([d[2] for d in done])
    del done
    key = (T.to(torch.int64) << 56) | morton_key_t(A)
    order = torch.argsort(key)
    return A[order].contiguous(), T[order].contiguous(), Lv[order].contiguous()
