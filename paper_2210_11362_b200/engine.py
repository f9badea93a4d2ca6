"""Device sweep engine: the B200 schedule behind tr_als_ne / tr_als_qr / tr_als_qrne.

One `SweepEngine` owns every device buffer a run needs (allocated once, so a
sweep is a fixed list of kernel launches that can be replayed or captured in a
CUDA graph) and compiles the reference's per-mode loop (solvers.py:369-389,
:419-448, :472-498) into steps.

Right-hand sides (the MTTSP, solvers.py:379) come from a two-phase
environment tree instead of one X pass per mode:

* the modes are split into a prefix L = [0, h) and a suffix R = [h, N);
* phase L contracts X once with a half chain of (old) suffix cores, giving
  the environment of the prefix segment (|L-modes| x R^2 numbers); each
  M_n, n in L, is then reached by absorbing the other L cores (old ones from
  the right, freshly updated ones from the left) -- small GEMMs;
* phase R does the same with a half chain of the (new) prefix cores.

So X is streamed twice per sweep whatever N is, instead of N times, and the
(prod_{j!=n} I_j) x R^2 subchain matrix is never formed: the largest chain
ever materialised covers a contiguous block C' of modes chosen so that
max(prod C', |X| / prod C') is minimal.

Sharding (one process per GPU): X is split along `shard_mode`; every rank
runs the identical schedule on its slab (local core rows for the sharded
mode), so each M_n is a partial sum that one NCCL all-reduce completes before
the replicated, deterministic solve.
"""

from __future__ import annotations

import math
from dataclasses import dataclass, field

import numpy as np
import torch

from . import _lib as L

BUCKETS = ("subchain", "mttsp", "solve", "gramqr", "other")  # solvers.py:57
OZ64_MIN_FLOPS = 4e9  # fp64_gemm="auto": smallest environment product run on the int8 tensor cores
CRT_MIN_K = 4096      # fp64_gemm="auto": shortest contraction run by the CRT form of the int8 engine
SMALL_SOLVE_MAX = 112  # m = R_n R_{n+1} <= 112: explicit-inverse solve + one refinement step (trals.h)
OZ64_MAX_RHO = 2.0 ** 12  # fp64_gemm="auto": largest row dynamic range (max|x| K / sum|x|) of X sliced (trals.h)


def _prod(v):
    p = 1
    for x in v:
        p *= int(x)
    return p


class _HostStream:
    cuda_stream = 0


def _assert_close(actual, desired, rel=1e-10):
    """The reference's debug-mode identity check (solvers.py:215-218)."""
    scale = max(1.0, float(np.max(np.abs(desired))))
    np.testing.assert_allclose(actual, desired, rtol=rel, atol=rel * scale)


@dataclass
class Step:
    bucket: str
    fn: object
    name: str = ""
    stream: str = "main"   # "main" | "side"
    kind: str = "op"       # "op" | "fork" (side waits for main) | "join" (main waits for side)


@dataclass
class EngineStats:
    gemm_launches: int = 0
    x_passes_per_sweep: int = 0
    steps_per_sweep: int = 0
    kernels_per_sweep: int = 0
    notes: list = field(default_factory=list)


class SweepEngine:
    """Compiles and runs TR-ALS sweeps on one GPU (one rank of a sharded run)."""

    def __init__(self, x_local: torch.Tensor, dims, ranks, variant: str, *, shard_mode=None, lo=0, hi=None,
                 group=None, world_size: int = 1, rank_deficient_fallback=True, svd_rcond=1e-12,
                 debug_checks=False, fp64_gemm="auto", _test_lib=None):
        if variant not in ("als", "ne", "qr", "qrne"):
            raise ValueError(f"unsupported device variant {variant!r}")
        # `_test_lib` lets the CPU test-suite drive this exact schedule through a numpy
        # model of the C-ABI (tests/fake_trals.py); the solvers never pass it.
        if _test_lib is None and not x_local.is_cuda:
            raise TypeError("x_local must be a CUDA tensor")
        if not (x_local.dtype in (torch.float64, torch.float32) and x_local.is_contiguous()):
            raise TypeError("x_local must be a contiguous float64 or float32 tensor")
        # fp32 variant: X stays fp32 and the environment products run on the int8
        # tcgen05 tensor cores over X's digit slices (exact int32 accumulation);
        # cores, Grams, solves and errors stay fp64.
        self.fp32 = x_local.dtype == torch.float32
        # fp64 X: the environment products run either on the fp64 DMMA pipe ("dmma") or on the
        # int8 tcgen05 tensor cores over 7 balanced digit planes of X ("ozaki": 28 exact int32
        # digit-pair products combined in fp64 -- the DMMA product's accuracy at ~3x its rate).
        # "auto": ozaki once an environment product is large enough to amortise the per-call
        # slicing of the half chain (measured crossover: BASELINE c2, 2.1 GFLOP, is a tie)
        # The int8 engine has two forms, chosen per environment product: the digit-pair one above and,
        # for long contractions (K >= CRT_MIN_K, R^2 <= 512: BASELINE c5), the CRT one -- 16 modular
        # int8 GEMMs + an exact 128-bit reconstruction (csrc/crt_int8_gemm.cuh), whose per-output
        # cost only pays off when K is long.  "crt" forces the CRT form wherever it is supported,
        # "ozaki" the digit-pair form everywhere.
        if fp64_gemm not in ("auto", "dmma", "ozaki", "crt"):
            raise ValueError(f"unknown fp64_gemm {fp64_gemm!r}; expected 'auto', 'dmma', 'ozaki' or 'crt'")
        self.crt_min_k = {"auto": CRT_MIN_K, "crt": 1}.get(fp64_gemm)
        if fp64_gemm == "auto":
            env_flops = 2.0 * _prod(x_local.shape) * max(int(r) for r in ranks) ** 2
            fp64_gemm = "ozaki" if env_flops >= OZ64_MIN_FLOPS else "dmma"
            if fp64_gemm == "ozaki" and _test_lib is None and x_local.dtype == torch.float64:
                # the digit planes (one K-major copy per X-streaming phase, 8 B per element each)
                # must fit beside everything else; otherwise stay on the fp64 pipe
                free, _ = torch.cuda.mem_get_info(x_local.device)
                if 2 * 8 * x_local.numel() * 1.05 > free:
                    fp64_gemm = "dmma"
        self.fp64_gemm = fp64_gemm
        self.oz64 = (not self.fp32) and fp64_gemm in ("ozaki", "crt") and _test_lib is None
        self.env_kinds = set()  # forms of the int8 engine in use: "oz64" (digit pairs), "crt"
        self.sliced = self.fp32 or self.oz64
        self.lib = _test_lib if _test_lib is not None else L.lib()
        self.dev = x_local.device
        self.variant = variant
        self.N = len(dims)
        self.dims = [int(d) for d in dims]
        self.ranks = [int(r) for r in ranks]
        self.world = int(world_size)
        self.group = group
        self.s = shard_mode
        self.lo = int(lo)
        self.hi = int(hi) if hi is not None else (self.dims[shard_mode] if shard_mode is not None else 0)
        self.dl = list(self.dims)
        if shard_mode is not None:
            self.dl[shard_mode] = self.hi - self.lo
        if tuple(x_local.shape) != tuple(self.dl):
            raise ValueError(f"local slab shape {tuple(x_local.shape)} != expected {tuple(self.dl)}")
        self.x = x_local
        # fp32 / oz64: (kind, side, pre, post) -> (planes, exps): X sliced, K-major for that side
        # (kind "oz32" / "oz64": digit planes, "crt": residue planes)
        self._xsplit = {}
        self._x64 = None    # fp32 + exact errors: fp64 copy of X for the residual kernel
        self.fallback_ok = bool(rank_deficient_fallback)
        # AlsConfig.debug_checks (solvers.py:376-377, 432-438, 485-487): assert the coefficient
        # Gram against the explicitly assembled subchain every block (host sync; eager only)
        self.debug_checks = bool(debug_checks)
        self.svd_rcond = float(svd_rcond)
        self.stream = torch.cuda.current_stream(self.dev) if x_local.is_cuda else _HostStream()
        self.stats = EngineStats()
        self._alloc()
        self._compile()

    # ------------------------------------------------------------------ buffers
    def R(self, j):
        return self.ranks[j % self.N]

    def _empty(self, *shape):
        return torch.empty(shape, dtype=torch.float64, device=self.dev)

    def _alloc(self):
        N = self.N
        self.Gc = [self._empty(self.R(j), self.dims[j], self.R(j + 1)) for j in range(N)]
        self.Gs = [self._empty(self.dims[j], self.R(j), self.R(j + 1)) for j in range(N)]
        self.Gt = [self._empty(self.dims[j], self.R(j + 1), self.R(j)) for j in range(N)]
        self.E = [self._empty(self.R(j) ** 2, self.R(j + 1) ** 2) for j in range(N)]
        self.M = [self._empty(self.dims[n], self.R(n) * self.R(n + 1)) for n in range(N)]
        self.S = [self._empty(self.R(n) * self.R(n + 1), self.R(n) * self.R(n + 1)) for n in range(N)]
        mmax = max(self.R(n) * self.R(n + 1) for n in range(N))
        self.U = self._empty(mmax, mmax)
        self.Lo = self._empty(mmax, mmax)
        self.chol_aux = self._empty(max(1, max(self.lib.trals_cholesky_aux_elems(self.R(n) * self.R(n + 1))
                                              for n in range(N))))
        self.solve_ws = self._empty(max(1, max(self.lib.trals_chol_solve_ws_elems(self.dims[n], self.R(n) * self.R(n + 1))
                                              for n in range(N))))
        self.use_rqr = self.variant in ("qr", "qrne")
        if self.use_rqr:
            ks = [min(self.dims[j], self.R(j) * self.R(j + 1)) for j in range(N)]
            rrs = [self.R(j) * self.R(j + 1) for j in range(N)]
            self.Rmat = self._empty(max(k * r for k, r in zip(ks, rrs)))
            self.Rslice = self._empty(max(k * r for k, r in zip(ks, rrs)))
            qws = [self.lib.trals_core_qr_ws_elems(self.dims[j], rrs[j]) for j in range(N)]
            if min(qws) < 0:
                raise ValueError("per-core QR size outside the kernel envelope")
            self.qr_ws = self._empty(max(1, max(qws)))
        # QR / ALS: R0 = chol(S_n) with S_n formed from the R-tensors (QR) or the cores (ALS) and
        # factored in double-double arithmetic (dd_r0.cuh): the R factor of V_[2] without forming V
        # and without squaring cond(V) in fp64.  The R-tensors are kept per core in layout C and
        # their transfer matrices as dd (hi, lo) planes.
        self.use_r0 = self.variant in ("qr", "als")
        if self.use_r0:
            if self.variant == "qr":
                self.r0_ks = [min(self.dims[j], self.R(j) * self.R(j + 1)) for j in range(N)]
                self.RtC = [self._empty(self.R(j), self.r0_ks[j], self.R(j + 1)) for j in range(N)]
            else:
                self.r0_ks = list(self.dims)
                self.RtC = self.Gc
            self.Edd = [(self._empty(self.R(j) ** 2 * self.R(j + 1) ** 2), self._empty(self.R(j) ** 2 * self.R(j + 1) ** 2))
                        for j in range(N)]
            need = self.lib.trals_dd_r0_ws_elems(N, L.i32_array(self.ranks))
            if need < 0:
                raise ValueError("R0 outside the kernel envelope")
            self.r0_ws = self._empty(max(1, need))
        self.fb_ws = self._empty(max(1, max(self.lib.trals_spd_fallback_ws_elems(self.dims[n], self.R(n) * self.R(n + 1))
                                            for n in range(N))))
        self.info = torch.zeros(L.INFO_SLOTS, dtype=torch.int32, device=self.dev)
        self.xnorm2 = self._empty(2)  # [|X|^2, #non-finite]
        self.err_cur = self._empty(3)
        rmax = max(self.ranks)
        self.chain_tmp = self._empty(2 * rmax ** 4)
        self.sumsq_ws = self._empty(self.lib.trals_sumsq_ws_elems())
        self.Gc_loc = None
        if self.s is not None:
            s = self.s
            self.Gc_loc = self._empty(self.R(s), self.dl[s], self.R(s + 1))
        self.gws_need = 1
        self.side_gws_need = 1
        self.gws = None  # sized after compile
        self.side = torch.cuda.Stream(device=self.dev) if self.dev.type == "cuda" else _HostStream()
        self._fork_ev = torch.cuda.Event() if self.dev.type == "cuda" else None
        self._join_ev = torch.cuda.Event() if self.dev.type == "cuda" else None
        self._cur = None
        self.graph = None
        self.graph_err = None
        self.graph_exact = None

    # local views used by the X contractions
    def core_c(self, j):
        return self.Gc_loc if (self.s is not None and j == self.s) else self.Gc[j]

    def core_s(self, j):
        if self.s is not None and j == self.s:
            return self.Gs[j][self.lo:self.hi]
        return self.Gs[j]

    def core_zt(self, j):
        if self.s is not None and j == self.s:
            return self.Gt[j][self.lo:self.hi]
        return self.Gt[j]

    def m_target(self, n):
        """Pointer where the leaf for mode n writes its (local) rows of M_n."""
        rr = self.R(n) * self.R(n + 1)
        if self.s is not None and n == self.s:
            return self.M[n].data_ptr() + self.lo * rr * 8
        return self.M[n].data_ptr()

    def _ws(self, elems):
        self.gws_need = max(self.gws_need, int(elems))

    def _side_ws(self, elems):
        self.side_gws_need = max(self.side_gws_need, int(elems))

    # ----------------------------------------------------------------- compile
    def _compile(self):
        N = self.N
        self.steps: list[Step] = []
        self._chain_prefix = set()  # blocks whose Gram-chain prefix is formed ahead (see _factor)
        self._bufs = []  # keep env buffers alive
        self._env_flops = []
        self.stats.x_passes_per_sweep = 0
        # The sweep opens with the transfer matrix of the LAST core (solved at the end of the previous
        # sweep; before the first sweep this recomputes what set_cores left): like every other core's
        # it runs on the side stream ahead of the Gram chain that needs it (S_0), here under the first
        # environment product instead of at the end of the previous sweep.
        if N == 2:
            phases = [(0, 0), (1, 1)]
        else:
            h = (N + 1) // 2
            phases = [(0, h - 1), (h, N - 1)]
        self._phase_first = {a for a, _ in phases}
        last = N - 1
        rr_last = self.R(last) * self.R(last + 1)
        self._side_ws(self.lib.trals_gemm_ws_elems(1, rr_last, self.dims[last], rr_last))
        self._factor(0, first=Step("gramqr", lambda n=last: self._gram(n, self._sp(), side=True), f"gram{last}",
                                   stream="side"))
        for a, b in phases:
            self._phase(a, b)
        # error terms need the last mode's quantities (solvers.py:385-389)
        rows = self.dims[N - 1]
        m = self.R(N - 1) * self.R(N)
        self.err_ws = self._empty(self.lib.trals_error_ws_elems(rows, m))
        self.gws = self._empty(self.gws_need)
        self.side_gws = self._empty(self.side_gws_need)
        self.stats.steps_per_sweep = len(self.steps)

    def _choose_block(self, a, b):
        """Contiguous block C' of the complement of [a..b] that X is contracted with."""
        N = self.N
        total = _prod(self.dl)
        best = None
        if a == 0:
            cands = [(y, N - 1) for y in range(b + 1, N)]
        else:
            cands = [(0, x) for x in range(0, a)]
        for lo, hi in cands:
            pc = _prod(self.dl[lo:hi + 1])
            cost = (max(pc, total // pc), pc)
            if best is None or cost < best[0]:
                best = (cost, lo, hi)
        return best[1], best[2]

    def _phase(self, a, b):
        N = self.N
        lo, hi = self._choose_block(a, b)
        nblk = hi - lo + 1
        bd = self.dl[lo:hi + 1]
        br = [self.R(j) for j in range(lo, hi + 2)]
        r_lo, r_hi = br[0], br[-1]
        H = self._empty(_prod(bd) * r_lo * r_hi)
        tmp = self._empty(max(1, self.lib.trals_half_chain_tmp_elems(nblk, L.i64_array(bd), L.i32_array(br))))
        self._bufs += [H, tmp]
        # gemm workspace of the chain build
        pre = bd[0]
        for j in range(1, nblk):
            self._ws(self.lib.trals_gemm_ws_elems(1, pre * r_lo, br[j], bd[j] * br[j + 1]))
            pre *= bd[j]
        bd_a, br_a = L.i64_array(bd), L.i32_array(br)
        blk = list(range(lo, hi + 1))

        def chain_step(bd_a=bd_a, br_a=br_a, blk=blk, H=H, tmp=tmp, nblk=nblk):
            cc = L.ptr_array([self.core_c(j).data_ptr() for j in blk])
            L.check(self.lib.trals_half_chain_f64(nblk, bd_a, br_a, self.core_s(blk[0]).data_ptr(), cc,
                                                  H.data_ptr(), tmp.data_ptr(), self.gws.data_ptr(),
                                                  self.gws.numel(), 0, self._sp()), "half_chain")
        self.steps.append(Step("subchain", chain_step, f"chain[{lo}..{hi}]"))

        if a == 0:
            side, seg_a, seg_b = 0, 0, lo - 1
            pre, post = _prod(self.dl[:lo]), _prod(self.dl[lo:])
        else:
            side, seg_a, seg_b = 1, hi + 1, N - 1
            pre, post = _prod(self.dl[:hi + 1]), _prod(self.dl[hi + 1:])
        seg_len = pre if side == 0 else post
        RR = r_lo * r_hi
        self._ws(self.lib.trals_gemm_ws_elems(1, pre, post, RR) if side == 0
                 else self.lib.trals_gemm_ws_elems(1, post, pre, RR))
        root_leaf = seg_a == seg_b
        if root_leaf:
            n = seg_a
            self._pre_leaf(n)
            target = lambda n=n: self.m_target(n)
        else:
            E0 = self._empty(seg_len * RR)
            self._bufs.append(E0)
            target = lambda E0=E0: E0.data_ptr()

        env_name = f"env[{seg_a}..{seg_b}]"
        if self.sliced:
            rows, k = (pre, post) if side == 0 else (post, pre)
            kind = "oz32" if self.fp32 else self._env_kind(rows, k, r_lo * r_hi)
            key = (kind, side, pre, post)
            nbytes, _, wsf, envf = self._sliced_api(kind)
            if key not in self._xsplit:
                self._xsplit[key] = (torch.empty(int(nbytes(rows, k)), dtype=torch.int8, device=self.dev),
                                     torch.empty(rows, dtype=torch.int32, device=self.dev))
            self._ws(wsf(pre, post, side, r_lo, r_hi))

            def env_step(pre=pre, post=post, side=side, H=H, r_lo=r_lo, r_hi=r_hi, target=target,
                         leaf=int(root_leaf), key=key, envf=envf, stages=None):
                xd, xe = self._xsplit[key]
                extra = () if stages is None else (stages,)
                L.check(envf(xd.data_ptr(), xe.data_ptr(), pre, post, side, H.data_ptr(), r_lo, r_hi, target(),
                             leaf, self.gws.data_ptr(), self.gws.numel(), *extra, self._sp()), "env_oz")
            if kind == "crt":
                # three steps on the shared workspace: the half chain's residue planes, the modular
                # GEMMs (the dominant kernel: the step named env[...]), the CRT reconstruction
                staged = self.lib.trals_env_crt_stage
                self.steps.append(Step("mttsp", lambda f=env_step, g=staged: f(envf=g, stages=1),
                                       f"bslice[{seg_a}..{seg_b}]"))
                self.steps.append(Step("mttsp", lambda f=env_step, g=staged: f(envf=g, stages=2),
                                       f"env[{seg_a}..{seg_b}]"))
                env_step = lambda f=env_step, g=staged: f(envf=g, stages=4)  # noqa: E731
                env_name = f"crt[{seg_a}..{seg_b}]"
        else:
            def env_step(pre=pre, post=post, side=side, H=H, r_lo=r_lo, r_hi=r_hi, target=target,
                         leaf=int(root_leaf)):
                L.check(self.lib.trals_env_f64(self.x.data_ptr(), pre, post, side, H.data_ptr(), r_lo, r_hi,
                                               target(), leaf, self.gws.data_ptr(), self.gws.numel(), self._sp()),
                        "env")
        self.steps.append(Step("mttsp", env_step, env_name))
        self.stats.x_passes_per_sweep += 1
        self._env_flops.append(2.0 * pre * post * RR)
        if root_leaf:
            self._solve(seg_a)
            return
        # absorb the extra complement cores so the environment covers exactly [a..b]
        cur = E0
        sa, sb = seg_a, seg_b
        while sb > b:
            last = (a == b and sa == a and sb == b + 1)
            cur, sa, sb = self._absorb_right(cur, sa, sb, leaf_mode=a if last else None)
        while sa < a:
            last = (a == b and sa + 1 == a)
            cur, sa, sb = self._absorb_left(cur, sa, sb, leaf_mode=a if last else None)
        self._tree(cur, a, b)

    def _pre_leaf(self, n):
        if self.s is not None and n == self.s and self.world > 1:
            M = self.M[n]
            self.steps.append(Step("mttsp", lambda M=M: M.zero_(), f"zero M{n}"))

    def _absorb_right(self, cur, a, b, leaf_mode):
        """Env [a..b] -> [a..b-1] by absorbing (old) core b."""
        pre = _prod(self.dl[a:b])
        Ra, Rb, Rb1 = self.R(a), self.R(b), self.R(b + 1)
        leaf = leaf_mode is not None
        self._ws(self.lib.trals_gemm_ws_elems(1, Ra * pre, self.dl[b] * Rb1, Rb))
        if leaf:
            self._pre_leaf(leaf_mode)
            out = None
            target = lambda n=leaf_mode: self.m_target(n)
        else:
            out = self._empty(Ra * pre * Rb)
            self._bufs.append(out)
            target = lambda out=out: out.data_ptr()

        def step(cur=cur, Ra=Ra, pre=pre, Ib=self.dl[b], Rb=Rb, Rb1=Rb1, b=b, target=target, leaf=int(leaf)):
            L.check(self.lib.trals_absorb_right_f64(cur.data_ptr(), Ra, pre, Ib, Rb, Rb1, self.core_zt(b).data_ptr(),
                                                    target(), leaf, self.gws.data_ptr(), self.gws.numel(),
                                                    self._sp()), "absorb_right")
        self.steps.append(Step("mttsp", step, f"absorbR core{b} -> [{a}..{b - 1}]"))
        return out, a, b - 1

    def _absorb_left(self, cur, a, b, leaf_mode):
        """Env [a..b] -> [a+1..b] by absorbing (new) core a."""
        rest = _prod(self.dl[a + 1:b + 1])
        Ra, Ra1, Rb1 = self.R(a), self.R(a + 1), self.R(b + 1)
        leaf = leaf_mode is not None
        self._ws(self.lib.trals_gemm_ws_elems(1, rest * Rb1, Ra * self.dl[a], Ra1))
        if leaf:
            self._pre_leaf(leaf_mode)
            out = None
            target = lambda n=leaf_mode: self.m_target(n)
        else:
            out = self._empty(Ra1 * rest * Rb1)
            self._bufs.append(out)
            target = lambda out=out: out.data_ptr()

        def step(cur=cur, Ra=Ra, Ia=self.dl[a], rest=rest, Ra1=Ra1, Rb1=Rb1, a=a, target=target, leaf=int(leaf)):
            L.check(self.lib.trals_absorb_left_f64(cur.data_ptr(), Ra, Ia, rest, Ra1, Rb1, self.core_c(a).data_ptr(),
                                                   target(), leaf, self.gws.data_ptr(), self.gws.numel(),
                                                   self._sp()), "absorb_left")
        self.steps.append(Step("mttsp", step, f"absorbL core{a} -> [{a + 1}..{b}]"))
        return out, a + 1, b

    def _tree(self, env, a, b):
        """Emit steps that update modes a..b in order from the environment of [a..b]."""
        if a == b:
            self._solve(a)  # env already is M_a (written by the leaf absorption)
            return
        m = (a + b) // 2
        cur, sa, sb = env, a, b
        while sb > m:
            leaf = a if (sa == a and sb == a + 1 and m == a) else None
            cur, sa, sb = self._absorb_right(cur, sa, sb, leaf)
        self._tree(cur, a, m)
        cur, sa, sb = env, a, b
        while sa <= m:
            leaf = b if (sa + 1 == b and m + 1 == b) else None
            cur, sa, sb = self._absorb_left(cur, sa, sb, leaf)
        self._tree(cur, m + 1, b)

    def _r0_nonsquare(self, n):
        """QR / ALS: the reference's triangular factor is non-square when it has fewer rows
        than R_n R_{n+1} -- QR: prod_{j!=n} k_j with k_j = min(I_j, R_j R_{j+1})
        (ring.py:236-249); ALS: prod_{j!=n} I_j, the rows of the subchain unfolding
        (solvers.py:337-339) -- and then it always takes the SVD solve (solvers.py:264-266):
        no Cholesky, no fallback count."""
        if self.variant not in ("qr", "als"):
            return False
        ks = 1
        for j in range(self.N):
            if j != n:
                ks *= self.dims[j] if self.variant == "als" else min(self.dims[j], self.R(j) * self.R(j + 1))
        return ks < self.R(n) * self.R(n + 1)

    def _factor(self, n, first=None):
        """S_n from the Gram chain and its Cholesky factor -- depends on cores only, so it runs on
        the side stream as soon as core n-1 is final, overlapping the right-hand side of mode n.
        `first`: a side-stream step to run right after the fork (the Gram / per-core QR of core n-1)."""
        N = self.N
        rr = self.R(n) * self.R(n + 1)
        S = self.S[n]
        ranks_a = L.i32_array(self.ranks)
        rmax = max(self.ranks)
        self._side_ws(self.lib.trals_gemm_ws_elems(1, rmax ** 2, rmax ** 2, rmax ** 2))
        self.steps.append(Step("other", None, f"fork S{n}", kind="fork"))
        if first is not None:
            self.steps.append(first)
        if self.use_r0:
            # QR (solvers.py:422-424) / ALS (:337-339): S_n and R0 = chol(S_n) in double-double from the
            # transfer matrices of the R-tensors (the cores); then R0's inverse operands and the 1e-13
            # degeneracy test (linalg.py:96-99)
            def r0(n=n, S=S, ranks_a=ranks_a):
                eh = L.ptr_array([e[0].data_ptr() for e in self.Edd])
                el = L.ptr_array([e[1].data_ptr() for e in self.Edd])
                L.check(self.lib.trals_dd_r0_f64(N, n, ranks_a, eh, el, S.data_ptr(), self.U.data_ptr(),
                                                 self.r0_ws.data_ptr(), self.r0_ws.numel(), self._sp()), "dd_r0")
            self.steps.append(Step("gramqr", r0, f"R0 {n}", stream="side"))

            def tri(rr=rr):
                L.check(self.lib.trals_tri_prepare_f64(self.U.data_ptr(), rr, self.Lo.data_ptr(),
                                                       self.chol_aux.data_ptr(), 1, self.info.data_ptr(),
                                                       self._sp()), "tri_prepare")
            if not self._r0_nonsquare(n):
                self.steps.append(Step("solve", tri, f"tri{n}", stream="side"))
            return

        def gram_chain(n=n, S=S, ranks_a=ranks_a, part=0):
            E = L.ptr_array([e.data_ptr() for e in self.E])
            L.check(self.lib.trals_gram_chain_part_f64(N, n, ranks_a, E, S.data_ptr(), self.chain_tmp.data_ptr(),
                                                       self.side_gws.data_ptr(), self.side_gws.numel(), part,
                                                       self._sp()), "gram_chain")
        # every factor of S_n but the last (core n-1's) was ready before core n-1 was solved: when the
        # previous block's factorisation left the prefix behind (below), only the last product remains
        hoisted = n in self._chain_prefix
        self.steps.append(Step("other", lambda f=gram_chain, p=2 if hoisted else 0: f(part=p), f"S{n}", stream="side"))

        def factor(S=S, rr=rr):
            L.check(self.lib.trals_cholesky_f64(S.data_ptr(), rr, self.U.data_ptr(), self.Lo.data_ptr(),
                                                self.chol_aux.data_ptr(), 0, self.info.data_ptr(),
                                                self._sp()), "cholesky")
        self.steps.append(Step("solve", factor, f"chol{n}", stream="side"))
        if N >= 4 and n + 1 < N and n in self._phase_first and (n + 1) not in self._phase_first:
            # prefix of the next block's Gram chain (cores n+2, ..., n-1: none of them core n), on the
            # side stream behind this factorisation and ahead of core n's solve.  Only behind the first
            # block of a phase: its factorisation hides under the environment product, so the main
            # stream's join does not wait for the prefix, and the next block's chain is the exposed one
            nxt = n + 1
            self.steps.append(Step("other", lambda f=gram_chain, nn=nxt, SS=self.S[nxt]: f(n=nn, S=SS, part=1),
                                   f"S{nxt} prefix", stream="side"))
            self._chain_prefix.add(nxt)

    def _solve(self, n):
        """Steps for one block update once M_n is complete (local rows)."""
        N = self.N
        rr = self.R(n) * self.R(n + 1)
        M = self.M[n]
        if self.world > 1:
            import torch.distributed as dist
            self.steps.append(Step("mttsp", lambda M=M: dist.all_reduce(M, group=self.group), f"allreduce M{n}"))
        self.steps.append(Step("solve", None, f"join chol{n}", kind="join"))
        if self.debug_checks:
            self.steps.append(Step("other", lambda n=n: self._debug_check(n), f"debug S{n}"))

        def solve(n=n, M=M, rr=rr):
            L.check(self.lib.trals_chol_solve_f64(self.U.data_ptr(), self.Lo.data_ptr(), self.chol_aux.data_ptr(), rr,
                                                  M.data_ptr(), self.dims[n], self.Gt[n].data_ptr(),
                                                  self.solve_ws.data_ptr(), self.solve_ws.numel(), self._sp()),
                    "chol_solve")
            if rr <= SMALL_SOLVE_MAX:
                # explicit-inverse operands: one refinement step against S_n when the factor is
                # ill-conditioned (device-side gate, trals.h)
                L.check(self.lib.trals_solve_refine_f64(self.Lo.data_ptr(), self.chol_aux.data_ptr(),
                                                        self.S[n].data_ptr(), rr, M.data_ptr(), self.dims[n],
                                                        self.Gt[n].data_ptr(), self.info.data_ptr(), self._sp()),
                        "solve_refine")
        if not self._r0_nonsquare(n):
            self.steps.append(Step("solve", solve, f"solve{n}"))
        # numerical fallbacks of the reference (linalg.py:77-81, solvers.py:262-273): the kernel is a
        # no-op unless the factorisation flagged a failure, so it stays in the (graph-captured) sweep
        rr_rows = self.dims[n]
        if self.use_r0:
            # solvers.py:262-273: the min-norm solve on R0 itself -- always for a non-square R0
            # (mode 2, uncounted), on a degenerate diagonal when the fallback is enabled (mode 1)
            # (mode 3 with the fallback disabled: only the ill-conditioning safety solve, a degenerate
            # R0 still raises DegenerateTriangularError at the end of the run)
            mode = 2 if self._r0_nonsquare(n) else (1 if self.fallback_ok else 3)
            lr = rr  # R0 = chol(S_n) is square; rows beyond rank(V) are zero

            def fallback(n=n, M=M, rr=rr, mode=mode, rows=rr_rows, lr=lr):
                L.check(self.lib.trals_tri_fallback_f64(self.U.data_ptr(), lr, rr, M.data_ptr(), rows,
                                                        self.Gt[n].data_ptr(), self.info.data_ptr(), mode,
                                                        self.svd_rcond, self.fb_ws.data_ptr(), self.fb_ws.numel(),
                                                        self._sp()), "tri_fallback")
            self.steps.append(Step("solve", fallback, f"fallback{n}"))
        else:
            def fallback(n=n, M=M, rr=rr, rows=rr_rows):
                L.check(self.lib.trals_spd_fallback_f64(self.S[n].data_ptr(), rr, M.data_ptr(), rows,
                                                        self.Gt[n].data_ptr(), self.info.data_ptr(), 0,
                                                        2.220446049250313e-16, self.fb_ws.data_ptr(),
                                                        self.fb_ws.numel(), self._sp()), "spd_fallback")
            self.steps.append(Step("solve", fallback, f"fallback{n}"))

        def refresh(n=n):
            ra, i, rb = self.R(n), self.dims[n], self.R(n + 1)
            sp = self._sp()
            L.check(self.lib.trals_core_relayout_f64(self.Gt[n].data_ptr(), L.LAYOUT_ZT, ra, i, rb,
                                                     self.Gc[n].data_ptr(), L.LAYOUT_C, sp), "relayout")
            L.check(self.lib.trals_core_relayout_f64(self.Gt[n].data_ptr(), L.LAYOUT_ZT, ra, i, rb,
                                                     self.Gs[n].data_ptr(), L.LAYOUT_SLICE, sp), "relayout")
            if self.s is not None and n == self.s:
                L.check(self.lib.trals_core_relayout_f64(self.core_zt(n).data_ptr(), L.LAYOUT_ZT, ra,
                                                         self.hi - self.lo, rb, self.Gc_loc.data_ptr(),
                                                         L.LAYOUT_C, sp), "relayout")
        self.steps.append(Step("gramqr", refresh, f"refresh{n}"))
        # The transfer matrix of the new core (NE: its Gram; QR / QRNE: the per-core Householder QR
        # first) only feeds the Gram chains, so it runs on the side stream ahead of S_{n+1} and its
        # factor, off the main stream's path to the next right-hand side (c5 QRNE: the 0.33 ms QR of
        # every core was on the critical path).
        self._side_ws(self.lib.trals_gemm_ws_elems(1, rr, self.dims[n], rr))
        if n + 1 < N:
            gram = Step("gramqr", lambda n=n: self._gram(n, self._sp(), side=True), f"gram{n}", stream="side")
            self._factor(n + 1, first=gram)
        # (the last core's transfer matrix is formed at the start of the next sweep, see _compile)

    def _gram(self, n, sp, side=False):
        """Transfer matrix of core n: from the core itself (NE, ring.py:188) or, for QR/QRNE, from the
        R-tensor of its Householder QR (mode2_qr + lateral_gram of the R-tensor, solvers.py:417,468-470).
        side: called from a side-stream step (uses that stream's GEMM workspace)."""
        ra, i, rb = self.R(n), self.dims[n], self.R(n + 1)
        gws = self.side_gws if side else self.gws
        if self.variant == "als":
            L.check(self.lib.trals_dd_transfer_f64(self.Gc[n].data_ptr(), ra, i, rb, self.Edd[n][0].data_ptr(),
                                                   self.Edd[n][1].data_ptr(), sp), "dd_transfer")
            return
        if not self.use_rqr:
            L.check(self.lib.trals_core_gram_f64(self.Gs[n].data_ptr(), ra, i, rb, self.E[n].data_ptr(),
                                                 gws.data_ptr(), gws.numel(), sp), "core_gram")
            return
        k = min(i, ra * rb)
        L.check(self.lib.trals_core_qr_f64(self.Gt[n].data_ptr(), i, ra * rb, self.Rmat.data_ptr(),
                                           self.qr_ws.data_ptr(), self.qr_ws.numel(), sp), "core_qr")
        if not self.use_r0:
            L.check(self.lib.trals_core_relayout_f64(self.Rmat.data_ptr(), L.LAYOUT_ZT, ra, k, rb,
                                                     self.Rslice.data_ptr(), L.LAYOUT_SLICE, sp), "relayout")
        if self.use_r0:
            L.check(self.lib.trals_core_relayout_f64(self.Rmat.data_ptr(), L.LAYOUT_ZT, ra, k, rb,
                                                     self.RtC[n].data_ptr(), L.LAYOUT_C, sp), "relayout")
            L.check(self.lib.trals_dd_transfer_f64(self.RtC[n].data_ptr(), ra, k, rb, self.Edd[n][0].data_ptr(),
                                                   self.Edd[n][1].data_ptr(), sp), "dd_transfer")
            return
        L.check(self.lib.trals_core_gram_f64(self.Rslice.data_ptr(), ra, k, rb, self.E[n].data_ptr(),
                                             gws.data_ptr(), gws.numel(), sp), "core_gram")

    def _debug_check(self, n):
        """The reference's debug identities for block n (solvers.py:376-377 NE, 485-487 QRNE,
        432-438 QR): the Gram chain S_n equals A^T A of the explicitly assembled subchain
        unfolding -- A = G^{!=n}_[2] for NE / ALS, V_[2] of the R-tensor subchain for QR / QRNE
        (for QR also R0^T R0 = S_n) -- within the reference's tolerance
        (_assert_close, rel 1e-10: scale = max(1, max |desired|))."""
        N, sp = self.N, self._sp()
        order = [(n + 1 + j) % N for j in range(N - 1)]
        cores = []
        for j in order:
            ra, i, rb = self.R(j), self.dims[j], self.R(j + 1)
            if not self.use_rqr:
                cores.append((self.Gc[j], i))
                continue
            k = min(i, ra * rb)  # R-tensor of core j's lateral QR (ring.py:236-249), layout C
            rm = self._empty(k * ra * rb)
            ws = self._empty(max(1, self.lib.trals_core_qr_ws_elems(i, ra * rb)))
            L.check(self.lib.trals_core_qr_f64(self.Gt[j].data_ptr(), i, ra * rb, rm.data_ptr(), ws.data_ptr(),
                                               ws.numel(), sp), "core_qr")
            rc = self._empty(ra, k, rb)
            L.check(self.lib.trals_core_relayout_f64(rm.data_ptr(), L.LAYOUT_ZT, ra, k, rb, rc.data_ptr(),
                                                     L.LAYOUT_C, sp), "relayout")
            cores.append((rc, k))
        bd = [k for _, k in cores]
        br = [self.R(j) for j in order] + [self.R(n)]
        first = self._empty(bd[0], br[0], br[1])
        L.check(self.lib.trals_core_relayout_f64(cores[0][0].data_ptr(), L.LAYOUT_C, br[0], bd[0], br[1],
                                                 first.data_ptr(), L.LAYOUT_SLICE, sp), "relayout")
        rows = _prod(bd)
        rr = br[0] * br[-1]
        H = self._empty(rows * rr)
        tmp = self._empty(max(1, self.lib.trals_half_chain_tmp_elems(len(bd), L.i64_array(bd), L.i32_array(br))))
        need, pre = 1, bd[0]
        for j in range(1, len(bd)):
            need = max(need, self.lib.trals_gemm_ws_elems(1, pre * br[0], br[j], bd[j] * br[j + 1]))
            pre *= bd[j]
        need = max(need, self.lib.trals_gemm_ws_elems(1, rr, rows, rr))
        ws = self._empty(need)
        L.check(self.lib.trals_half_chain_f64(len(bd), L.i64_array(bd), L.i32_array(br), first.data_ptr(),
                                              L.ptr_array([c.data_ptr() for c, _ in cores]), H.data_ptr(),
                                              tmp.data_ptr(), ws.data_ptr(), ws.numel(), 0, sp), "half_chain")
        # H[k][(r_{n+1}, r_n)] -> column r_n + R_n r_{n+1}: the S_n index order
        G = self._empty(rr * rr)
        L.check(self.lib.trals_gemm_f64(H.data_ptr(), 0, 1, rr, 1, rr, rows, rr, H.data_ptr(), rr, G.data_ptr(),
                                        L.i64_array([0, 1 << 40, 0, rr, 1 << 40, 0, 1]), 0, ws.data_ptr(),
                                        ws.numel(), sp), "gram")
        s_dev = self.S[n].reshape(rr, rr)
        want = G.reshape(rr, rr).cpu().numpy()
        got = s_dev.cpu().numpy()
        _assert_close(got, want)
        if self.variant == "qr" and not self._r0_nonsquare(n):
            u = self.U.reshape(-1)[:rr * rr].reshape(rr, rr).cpu().numpy()
            _assert_close(u.T @ u, got, rel=1e-9)

    # ----------------------------------------------------------------- running
    def _sp(self):
        return int((self._cur or self.stream).cuda_stream)

    def set_cores(self, cores_host):
        """Upload C-order host cores and derive every layout + Gram (the 'prepare' of solvers.py:366-367)."""
        sp = self._sp()
        for j, g in enumerate(cores_host):
            t = torch.as_tensor(g, dtype=torch.float64)
            self.Gc[j].copy_(t, non_blocking=False)
        for j in range(self.N):
            self._derive(j, sp)

    def _derive(self, j, sp):
        ra, i, rb = self.R(j), self.dims[j], self.R(j + 1)
        L.check(self.lib.trals_core_relayout_f64(self.Gc[j].data_ptr(), L.LAYOUT_C, ra, i, rb,
                                                 self.Gs[j].data_ptr(), L.LAYOUT_SLICE, sp), "relayout")
        L.check(self.lib.trals_core_relayout_f64(self.Gc[j].data_ptr(), L.LAYOUT_C, ra, i, rb,
                                                 self.Gt[j].data_ptr(), L.LAYOUT_ZT, sp), "relayout")
        if self.s is not None and j == self.s:
            L.check(self.lib.trals_core_relayout_f64(self.core_zt(j).data_ptr(), L.LAYOUT_ZT, ra,
                                                     self.hi - self.lo, rb, self.Gc_loc.data_ptr(), L.LAYOUT_C,
                                                     sp), "relayout")
        self._gram(j, sp)

    def _env_kind(self, rows, k, rr):
        """Form of the int8 engine for one fp64 environment product (rows x k) . (k x rr)."""
        kind = "oz64"
        if (self.crt_min_k is not None and k >= self.crt_min_k and self.lib.trals_crt_supported(rows, k, rr)):
            # 16 residue bytes per element of this phase's copy of X must fit beside everything else
            free, _ = torch.cuda.mem_get_info(self.dev)
            if self.lib.trals_crt_planes_bytes(rows, k) * 1.05 < free:
                kind = "crt"
        self.env_kinds.add(kind)
        return kind

    def _sliced_api(self, kind):
        """(plane bytes, (split, split workspace), env workspace, env) of one sliced form."""
        lib = self.lib
        if kind == "oz32":
            return (lib.trals_oz_digits_bytes, (lib.trals_oz_split_f32, lib.trals_oz_split_ws_elems),
                    lib.trals_env_oz_ws_elems, lib.trals_env_oz)
        if kind == "crt":
            return (lib.trals_crt_planes_bytes, (lib.trals_crt_split_f64, lib.trals_crt_split_ws_elems),
                    lib.trals_env_crt_ws_elems, lib.trals_env_crt)
        return (lib.trals_oz64_digits_bytes, (lib.trals_oz64_split_f64, lib.trals_oz_split_ws_elems),
                lib.trals_env_oz64_ws_elems, lib.trals_env_oz64)

    def prepare_x(self):
        """Derive the per-X state after X (self.x) was (re)loaded: for the sliced
        environment products (fp32 variant, fp64 "ozaki"), X's int8 digit planes
        + row exponents, K-major for each X-streaming phase (phase L slices X as
        stored, phase R its transpose)."""
        if not self.sliced:
            return
        sp = self._sp()
        for (kind, side, pre, post), (xd, xe) in self._xsplit.items():
            _, (split, split_ws), _, _ = self._sliced_api(kind)
            need = split_ws(pre, post, side)
            ws = torch.empty(max(1, need), dtype=torch.float64, device=self.dev)
            L.check(split(self.x.data_ptr(), pre, post, side, xd.data_ptr(), xe.data_ptr(), ws.data_ptr(),
                          ws.numel(), sp), "oz_split")
        if self._x64 is not None:
            self._x64.copy_(self.x)

    def x_dynamic_range(self):
        """Largest rho = max|x| K / sum|x| over the K-major rows of X in every X-streaming phase of the
        int8 engine (trals_oz_range_f64): the accuracy guard of fp64_gemm="auto" (include/trals.h)."""
        if not self.oz64:
            return 0.0
        out = self._empty(len(self._xsplit))
        sp = self._sp()
        for i, (_, side, pre, post) in enumerate(self._xsplit):
            ws = self._empty(max(1, self.lib.trals_oz_range_ws_elems(pre, post, side)))
            L.check(self.lib.trals_oz_range_f64(self.x.data_ptr(), pre, post, side, out[i:].data_ptr(), ws.data_ptr(),
                                                ws.numel(), sp), "oz_range")
        return float(out.max().item())

    def ensure_x64(self):
        """fp32 variant with exact errors: the residual kernel reads an fp64 copy of X
        (made once per X, outside any graph capture; refreshed by prepare_x)."""
        if self.fp32 and self._x64 is None:
            self._x64 = self.x.to(torch.float64)

    def compute_xnorm2(self):
        """Device [|X|^2, #non-finite entries] (all-reduced over ranks)."""
        fn = self.lib.trals_sumsq_f32 if self.fp32 else self.lib.trals_sumsq_f64
        L.check(fn(self.x.data_ptr(), self.x.numel(), self.xnorm2.data_ptr(), self.sumsq_ws.data_ptr(), self._sp()),
                "sumsq")
        if self.world > 1:
            import torch.distributed as dist
            dist.all_reduce(self.xnorm2, group=self.group)
        return self.xnorm2

    def env_flops(self):
        """Flops of each X-streaming environment product (2*M*K*N), in step order."""
        return list(self._env_flops)

    def run_sweep(self, events=None, env_events=None, aux_events=None):
        """Launch one full sweep.

        events: list -> (bucket, event) pairs appended at bucket changes.
        env_events: list -> (start, end) event pairs around every X-streaming
        environment product (the dominant kernel, for the roofline).
        aux_events: dict -> the same for the CRT form's other stages ("bslice", "crt").
        """
        prev = None
        cuda = self.dev.type == "cuda"
        for st in self.steps:
            if st.kind == "fork":
                if cuda:
                    self._fork_ev.record(self.stream)
                    self.side.wait_event(self._fork_ev)
                continue
            if st.kind == "join":
                if cuda:
                    self._join_ev.record(self.side)
                    self.stream.wait_event(self._join_ev)
                continue
            self._cur = self.side if st.stream == "side" else None
            if events is not None and st.stream == "main" and st.bucket != prev:
                ev = torch.cuda.Event(enable_timing=True)
                ev.record(self.stream)
                events.append((st.bucket, ev))
                prev = st.bucket
            timed = None
            if env_events is not None and st.name.startswith("env"):
                timed = env_events
            elif aux_events is not None and st.name.startswith(("bslice", "crt[")):
                timed = aux_events.setdefault(st.name.split("[")[0], [])
            if timed is not None:
                e0 = torch.cuda.Event(enable_timing=True)
                e1 = torch.cuda.Event(enable_timing=True)
                e0.record(self.stream)
                st.fn()
                e1.record(self.stream)
                timed.append((e0, e1))
            else:
                st.fn()
        self._cur = None

    def error_step(self, out, exact=False):
        """Per-sweep relative error into `out` (3 doubles).

        exact=False: cheap identity from the last block (solvers.py:177-212): [e, <M,Z>, <S,Z^T Z>].
        exact=True : ||X - TR(G)|| / ||X|| (solvers.py:164-174) by the fused reconstruct-residual
                     GEMM: [e, sum (X - X_hat)^2, 0]."""
        if exact:
            self._exact_error(out)
            return
        N = self.N
        n = N - 1
        rr = self.R(n) * self.R(n + 1)
        L.check(self.lib.trals_error_terms_f64(self.M[n].data_ptr(), self.Gt[n].data_ptr(), self.S[n].data_ptr(),
                                               self.dims[n], rr, self.xnorm2.data_ptr(), out.data_ptr(),
                                               self.err_ws.data_ptr(), self.err_ws.numel(), self._sp()),
                "error_terms")

    def _exact_plan(self):
        if getattr(self, "_xp", None) is not None:
            return self._xp
        N = self.N
        h = max(1, N // 2)
        pre, post = _prod(self.dl[:h]), _prod(self.dl[h:])
        R0, Rh = self.R(0), self.R(h)
        need = 1

        def chain_need(lo, hi):
            bd = self.dl[lo:hi + 1]
            br = [self.R(j) for j in range(lo, hi + 2)]
            n = 1
            p = bd[0]
            for j in range(1, len(bd)):
                n = max(n, self.lib.trals_gemm_ws_elems(1, p * br[0], br[j], bd[j] * br[j + 1]))
                p *= bd[j]
            tmp = self.lib.trals_half_chain_tmp_elems(len(bd), L.i64_array(bd), L.i32_array(br))
            return n, tmp, L.i64_array(bd), L.i32_array(br)

        nl, tl, bdl, brl = chain_need(0, h - 1)
        nr, tr, bdr, brr = chain_need(h, N - 1)
        self._xp = {
            "h": h, "pre": pre, "post": post, "K": R0 * Rh,
            "HL": self._empty(pre * R0 * Rh), "HRt": self._empty(R0 * Rh * post),
            "tmp": self._empty(max(1, tl, tr)), "ws": self._empty(max(1, nl, nr)),
            # the int8 engines also form the exact error's product on the tensor cores
            "part": self._empty(max(1, self.lib.trals_residual_oz64_ws_elems(pre, post, R0 * Rh) if self.sliced
                                    else self.lib.trals_residual_ws_elems(pre, post))),
            "bdl": bdl, "brl": brl, "bdr": bdr, "brr": brr,
        }
        return self._xp

    def _exact_error(self, out):
        xp = self._exact_plan()
        N, h = self.N, xp["h"]
        sp = self._sp()
        for lo, hi, H, bd, br, tr in ((0, h - 1, xp["HL"], xp["bdl"], xp["brl"], 0),
                                      (h, N - 1, xp["HRt"], xp["bdr"], xp["brr"], 1)):
            blk = list(range(lo, hi + 1))
            cc = L.ptr_array([self.core_c(j).data_ptr() for j in blk])
            L.check(self.lib.trals_half_chain_f64(len(blk), bd, br, self.core_s(lo).data_ptr(), cc, H.data_ptr(),
                                                  xp["tmp"].data_ptr(), xp["ws"].data_ptr(), xp["ws"].numel(), tr, sp),
                    "half_chain")
        if self.fp32 and self._x64 is None:
            self.ensure_x64()
        xd = self._x64 if self.fp32 else self.x
        res = self.lib.trals_residual_oz64 if self.sliced else self.lib.trals_residual_f64
        L.check(res(xd.data_ptr(), xp["pre"], xp["post"], xp["HL"].data_ptr(), xp["HRt"].data_ptr(), xp["K"],
                    self.xnorm2.data_ptr(), out.data_ptr(), xp["part"].data_ptr(), xp["part"].numel(), sp), "residual")
        if self.world > 1:
            import torch.distributed as dist
            dist.all_reduce(out[1:2], group=self.group)
            x2 = self.xnorm2[0:1]
            out[0:1].copy_(torch.where(x2 > 0, torch.sqrt(out[1:2] / x2), torch.zeros_like(x2)))

    def cores_host(self):
        return [g.detach().cpu().numpy().copy() for g in self.Gc]

    # ------------------------------------------------------------ CUDA graphs
    def capture(self, with_error=True, exact=False):
        """Capture one sweep as a CUDA graph, and the error terms (into `err_cur`) as a second one.

        Every buffer is owned by the engine, so the graphs stay valid for the
        engine's lifetime; replaying re-launches the identical kernel list with a
        single host call (the small configs are launch-bound).  The error has its
        own graph so a caller can time the sweep alone (AlsReport.iter_seconds
        excludes the error, solvers.py:111-116).  A sharded sweep can be captured
        only over NCCL (its all-reduces become graph nodes); gloo collectives are
        host-side and stay eager."""
        if not self.x.is_cuda:
            raise RuntimeError("graphs need a CUDA engine")
        if self.world > 1:
            import torch.distributed as dist
            if dist.get_backend(self.group) != "nccl":
                raise RuntimeError("sharded sweeps capture only over NCCL (collectives between kernels)")
        old = self.stream
        cap = torch.cuda.Stream(device=self.dev)
        cap.wait_stream(old)
        g = torch.cuda.CUDAGraph()
        ge = torch.cuda.CUDAGraph() if with_error else None
        self.stream = cap
        try:
            with torch.cuda.stream(cap):
                # relaxed: first-use cudaFuncSetAttribute calls (dynamic shared memory opt-in) may
                # happen inside the capture when no eager sweep preceded it
                g.capture_begin(capture_error_mode="relaxed")
                self.run_sweep()
                g.capture_end()
                if with_error:
                    ge.capture_begin(capture_error_mode="relaxed")
                    self.error_step(self.err_cur, exact=exact)
                    ge.capture_end()
        finally:
            self.stream = old
        old.wait_stream(cap)
        self.graph = g
        self.graph_err = ge
        self.graph_exact = exact
        return g

    def replay(self, sweep=True, error=True):
        """Replay the captured sweep and/or its error graph on the engine's stream."""
        with torch.cuda.stream(self.stream):
            if sweep:
                self.graph.replay()
            if error and self.graph_err is not None:
                self.graph_err.replay()

    def mttsp_flops_per_sweep(self):
        """Algorithmic RHS flops of one sweep: sum_n 2 |X| R_n R_{n+1}."""
        tot = _prod(self.dims)
        return sum(2.0 * tot * self.R(n) * self.R(n + 1) for n in range(self.N))
