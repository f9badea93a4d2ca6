"""Synthetic TR tensors generated on the GPU (the §8(f) "GPU-side reconstruct" row).

Follows the reference recipe (synthetic.py:84-91 gaussian cores, :167-181
relative noise, :184-197 make_dataset): the true cores are drawn on the host
with the reference's Philox stream (bit-identical draws), the dense tensor is
reconstructed on the device with libtrals (two half chains + one DMMA GEMM,
instead of the reference's full subchain materialisation, ring.py:155-170),
and the noise x + eta*||x||/||n||*n is drawn on the device.  With
`noise_source="host"` the noise is drawn with the reference's numpy stream
instead (identical to tenring.make_dataset up to reconstruct rounding).
"""

from __future__ import annotations

import numpy as np
import torch

from . import _lib as L
from .host import make_rng, spawn_seeds


def _stream():
    return int(torch.cuda.current_stream().cuda_stream)


def reconstruct_device(cores, device="cuda") -> torch.Tensor:
    """Dense tensor of a ring (C-order cores) on the device: X[pre][post] = sum HL[pre][a][b] HR[post][b][a]."""
    lib = L.lib()
    cs = [torch.as_tensor(np.asarray(g, dtype=np.float64)).to(device).contiguous() for g in cores]
    N = len(cs)
    if N < 2:
        raise ValueError("reconstruct needs at least two cores")
    dims = [int(g.shape[1]) for g in cs]
    ranks = [int(g.shape[0]) for g in cs]
    h = N // 2
    sp = _stream()

    def chain(lo, hi, transposed):
        blk = list(range(lo, hi + 1))
        bd = [dims[j] for j in blk]
        br = [ranks[j % N] for j in range(lo, hi + 2)]
        first = torch.empty((bd[0], br[0], br[1]), dtype=torch.float64, device=device)
        L.check(lib.trals_core_relayout_f64(cs[lo].data_ptr(), L.LAYOUT_C, br[0], bd[0], br[1], first.data_ptr(),
                                            L.LAYOUT_SLICE, sp), "relayout")
        n = int(np.prod(bd)) * br[0] * br[-1]
        out = torch.empty(n, dtype=torch.float64, device=device)
        tmp = torch.empty(max(1, lib.trals_half_chain_tmp_elems(len(blk), L.i64_array(bd), L.i32_array(br))),
                          dtype=torch.float64, device=device)
        need = 1
        pre = bd[0]
        for j in range(1, len(blk)):
            need = max(need, lib.trals_gemm_ws_elems(1, pre * br[0], br[j], bd[j] * br[j + 1]))
            pre *= bd[j]
        ws = torch.empty(need, dtype=torch.float64, device=device)
        L.check(lib.trals_half_chain_f64(len(blk), L.i64_array(bd), L.i32_array(br), first.data_ptr(),
                                         L.ptr_array([cs[j].data_ptr() for j in blk]), out.data_ptr(),
                                         tmp.data_ptr(), ws.data_ptr(), ws.numel(), transposed, sp), "half_chain")
        return out, int(np.prod(bd))

    HL, pre = chain(0, h - 1, 0)   # [pre][r_0][r_h]
    B, post = chain(h, N - 1, 1)   # [r_0][r_h][post]
    R0, Rh = ranks[0], ranks[h]
    X = torch.empty(dims, dtype=torch.float64, device=device)
    K = R0 * Rh
    need = lib.trals_gemm_ws_elems(1, pre, K, post)
    ws = torch.empty(max(need, 1), dtype=torch.float64, device=device)
    L.check(lib.trals_gemm_f64(HL.data_ptr(), 0, K, 1, 1, pre, K, post, B.data_ptr(), post, X.data_ptr(),
                               L.i64_array([0, 1 << 40, 0, post, 1 << 40, 0, 1]), 0, ws.data_ptr(), ws.numel(), sp),
            "reconstruct gemm")
    return X


def _sumsq(x):
    lib = L.lib()
    out = torch.empty(2, dtype=torch.float64, device=x.device)
    ws = torch.empty(lib.trals_sumsq_ws_elems(), dtype=torch.float64, device=x.device)
    L.check(lib.trals_sumsq_f64(x.data_ptr(), x.numel(), out.data_ptr(), ws.data_ptr(), _stream()), "sumsq")
    return out[:1]


def make_dataset_device(order, dim, rank, noise, seed, device="cuda", noise_source="device"):
    """(x on the device, true cores on the host) for a cubic gaussian recipe."""
    core_seed, noise_seed = spawn_seeds(seed, 2)
    rng = make_rng(core_seed)
    cores = [rng.standard_normal((rank, dim, rank)) for _ in range(order)]
    x = reconstruct_device(cores, device=device)
    if noise > 0:
        if noise_source == "host":
            draw = torch.from_numpy(make_rng(noise_seed).standard_normal(x.shape)).to(device)
        else:
            g = torch.Generator(device=device)
            g.manual_seed(int(noise_seed.generate_state(1, np.uint64)[0] & ((1 << 63) - 1)))
            draw = torch.randn(x.shape, dtype=torch.float64, device=device, generator=g)
        scale = noise * float(_sumsq(x).item()) ** 0.5 / float(_sumsq(draw).item()) ** 0.5
        x.add_(draw, alpha=scale)
        del draw
    return x, cores
