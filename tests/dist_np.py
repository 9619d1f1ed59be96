"""CPU (NumPy) stand-in for one rank of the distributed engine.

TEST INFRASTRUCTURE: implements the same interface as the GPU RankEngine in
distributed mode (exchange_sizes / pack / unpack / run_phase / run_level)
from the per-rank plans the native setup exposes (R<r>.* arrays) and the
oracle restatement's operators, so the multi-rank driver
(paper_2006_15367_b200/distributed.py) and the plans can be checked with
world_size > 1 over gloo on CPU.  Values this rank must not know are NaN:
charges of other ranks' particles, multipole rows of nodes it neither holds
nor receives, the rows of a plural node outside this rank's slice once the
reduce-scatter has run (they hold only partial sums), and local rows outside
this rank's observer slices until the all-gather -- a missing ghost, halo,
reduce-scatter or gather entry poisons the result.
"""
from __future__ import annotations

import numpy as np

from oracle import hfmm_np


class NumpyRankEngine:
    def __init__(self, setup, rank: int):
        self.s = setup
        self.r = rank
        meta = setup.array("meta_i64", np.int64)
        self.L, self.top, self.P = int(meta[0]), int(meta[1]), int(meta[5])
        mf = setup.array("meta_f64", np.float64)
        self.root_side, self.k = float(mf[0]), float(mf[5])
        parts = setup.array("particles", np.float64).reshape(-1, 5)
        self.pos = parts[:, :3].copy()
        self.q_all = parts[:, 3] + 1j * parts[:, 4]
        self.leaf_start = setup.array("leaf_start", np.uint64).astype(np.int64)
        rr = setup.array("rank_ranges", np.uint64).astype(np.int64).reshape(-1, 2)
        self.lb, self.le = int(rr[rank, 0]), int(rr[rank, 1])
        self.pb, self.pe = int(self.leaf_start[self.lb]), int(self.leaf_start[self.le])
        self.lv = {}
        for l in range(self.top, self.L + 1):
            tr, nt, nphi = (int(v) for v in setup.array(f"L{l}.sampling", np.int64))
            codes = setup.array(f"L{l}.codes", np.uint64)
            self.lv[l] = dict(
                trunc=tr, nt=nt, np=nphi, S=nt * nphi, codes=codes,
                centers=setup.array(f"L{l}.centers", np.float64).reshape(-1, 3),
                dirs=hfmm_np.directions(nt, nphi), quad=hfmm_np.quadrature(nt, nphi),
                far_off=setup.array(f"L{l}.far_off", np.uint64).astype(np.int64),
                far=np.searchsorted(codes, setup.array(f"L{l}.far", np.uint64)),
                held=setup.array(f"R{rank}.held.L{l}", np.int32),
                halo=setup.array(f"R{rank}.halo.L{l}", np.int32),
                cho=setup.array(f"R{rank}.child_off.L{l}", np.int32),
                ch=setup.array(f"R{rank}.children.L{l}", np.int32))
        self.mp = {l: np.full((d["codes"].size, d["S"]), np.nan, complex) for l, d in self.lv.items()}
        self.loc = {l: np.full((d["codes"].size, d["S"]), np.nan, complex) for l, d in self.lv.items()}
        self.q = np.full(self.pos.shape[0], np.nan, complex)
        self.pot = np.full(self.pos.shape[0], np.nan, complex)
        # this rank's slice [b, e) of every node it holds (empty: (0, 0))
        for l, d in self.lv.items():
            so = setup.array(f"L{l}.slices_off", np.uint64).astype(np.int64)
            sl = setup.array(f"L{l}.slices", np.int64).reshape(-1, 3)
            users = setup.array(f"L{l}.users", np.int64).reshape(-1, 3)
            d["plural"] = users[:, 2].astype(bool)
            mine = {}
            for n in d["held"]:
                b, e = 0, 0
                for z in range(so[n], so[n + 1]):
                    if sl[z, 0] == rank and sl[z, 2] > sl[z, 1]:
                        b, e = int(sl[z, 1]), int(sl[z, 2])
                mine[int(n)] = (b, e)
            d["mine"] = mine
        self.items = {}
        for q in range(self.P):
            if q == rank:
                continue
            for kind in (0, 2, 3):
                for dr in ("send", "recv"):
                    self.items[dr, kind, q] = setup.array(f"R{rank}.{dr}{kind}.{q}", np.int64).reshape(-1, 4)
        flat = setup.array("near_plan", np.int64)
        self.near_send = {}
        i = 0
        for qq in range(self.P):
            for w in range(self.P):
                c = int(flat[i])
                self.near_send[qq, w] = flat[i + 1:i + 1 + c]
                i += 1 + c
        self.near_off = setup.array("near_off", np.uint64).astype(np.int64)
        self.near = np.searchsorted(self.lv[self.L]["codes"], setup.array("near", np.uint64))

    # ---- charges
    def set_charges_sorted(self, q_sorted: np.ndarray) -> None:
        self.q[:] = np.nan
        self.q[self.pb:self.pe] = q_sorted[self.pb:self.pe]

    # ---- exchange interface (same as the GPU RankEngine)
    def _ghost_idx(self, leaves):
        if len(leaves) == 0:
            return np.zeros(0, np.int64)
        return np.concatenate([np.arange(self.leaf_start[li], self.leaf_start[li + 1]) for li in leaves])

    def _rows(self, dr, kind, peer, level):
        it = self.items[dr, kind, peer]
        return it if level < 0 else it[it[:, 0] == level]

    def exchange_sizes(self, kind, peer, level=-1):
        if kind == 1:
            return (5 * self._ghost_idx(self.near_send[self.r, peer]).size,
                    5 * self._ghost_idx(self.near_send[peer, self.r]).size)
        cnt = lambda it: int(2 * (it[:, 3] - it[:, 2]).sum())  # noqa: E731
        return cnt(self._rows("send", kind, peer, level)), cnt(self._rows("recv", kind, peer, level))

    def _arr(self, kind):
        return self.loc if kind == 3 else self.mp

    def pack(self, kind, peer, buf, level=-1):
        out = buf.numpy()
        if kind == 1:
            idx = self._ghost_idx(self.near_send[self.r, peer])
            out[:] = np.concatenate([self.pos[idx], self.q[idx].real[:, None], self.q[idx].imag[:, None]],
                                    axis=1).reshape(-1)
            return
        arr = self._arr(kind)
        vals = [arr[int(l)][int(n), b:e] for l, n, b, e in self._rows("send", kind, peer, level)]
        flat = np.concatenate(vals) if vals else np.zeros(0, complex)
        out[:] = np.stack([flat.real, flat.imag], -1).reshape(-1)

    def unpack(self, kind, peer, buf, level=-1):
        v = buf.numpy()
        if kind == 1:
            idx = self._ghost_idx(self.near_send[peer, self.r])
            g = v.reshape(-1, 5)
            self.pos[idx] = g[:, :3]
            self.q[idx] = g[:, 3] + 1j * g[:, 4]
            return
        arr = self._arr(kind)
        off = 0
        for l, n, b, e in self._rows("recv", kind, peer, level):
            seg = v[off:off + 2 * (e - b)]
            val = seg[0::2] + 1j * seg[1::2]
            if kind == 2:
                arr[int(l)][int(n), b:e] += val
            else:
                arr[int(l)][int(n), b:e] = val
            off += 2 * (e - b)

    def run_level(self, phase, level):
        self._phase(phase, level)

    # ---- phases (restatement of operators on held nodes only)
    def run_phase(self, phase):
        self._phase(phase, -1)

    def _phase(self, phase, level):
        k, L, top = self.k, self.L, self.top
        if phase == 1:  # C2M, own leaves
            d = self.lv[L]
            for li in range(self.lb, self.le):
                b, e = self.leaf_start[li], self.leaf_start[li + 1]
                rel = self.pos[b:e] - d["centers"][li]
                self.mp[L][li] = np.exp(1j * k * (d["dirs"] @ rel.T)) @ self.q[b:e]
        elif phase == 2:  # M2M partials over held children
            for l in range(L - 1, top - 1, -1):
                P, C = self.lv[l], self.lv[l + 1]
                for i, p in enumerate(P["held"]):
                    acc = np.zeros(P["S"], complex)
                    for c in P["ch"][P["cho"][i]:P["cho"][i + 1]]:
                        up = hfmm_np.fft_interpolate(self.mp[l + 1][c].reshape(C["nt"], C["np"]), P["nt"], P["np"])
                        acc += up.reshape(-1) * np.exp(1j * k * (P["dirs"] @ (C["centers"][c] - P["centers"][p])))
                    self.mp[l][p] = acc
            # after the reduce-scatter only the own slice of a plural node is
            # valid; poison the partial rows outside it right away
            self._poison_plural = True
        elif phase == 8:  # T build (nothing to precompute); the reduce-scatter is done
            self._poison_partials()
        elif phase == 3:  # M2L, held observers, own slice rows only
            self._poison_partials()
            for l in ([level] if level >= 0 else range(top, L + 1)):
                d = self.lv[l]
                side = self.root_side / 2 ** (l - 1)
                cells = hfmm_np._cells(d["codes"], l)
                cache = {}
                for o in d["held"]:
                    b, e = d["mine"][int(o)]
                    acc = np.full(d["S"], np.nan, complex)
                    acc[b:e] = 0.0
                    for src in d["far"][d["far_off"][o]:d["far_off"][o + 1]]:
                        off = tuple(cells[o] - cells[src])
                        if off not in cache:
                            cache[off] = hfmm_np.translation_operator(d["trunc"], d["dirs"], np.array(off, float) * side, k)
                        acc[b:e] += self.mp[l][src][b:e] * cache[off][b:e]
                    self.loc[l][o] = acc
        elif phase == 4:  # L2L, held parents -> held children
            for l in ([level] if level >= 0 else range(top, L)):
                P, C = self.lv[l], self.lv[l + 1]
                wp = np.repeat(P["quad"][0], P["np"]) * P["quad"][1]
                wc = np.repeat(C["quad"][0], C["np"]) * C["quad"][1]
                for i, p in enumerate(P["held"]):
                    for c in P["ch"][P["cho"][i]:P["cho"][i + 1]]:
                        z = self.loc[l][p] * np.exp(1j * k * (P["dirs"] @ (P["centers"][p] - C["centers"][c]))) * wp
                        down = hfmm_np.fft_anterpolate(z.reshape(P["nt"], P["np"]), C["nt"], C["np"]).reshape(-1)
                        self.loc[l + 1][c] += down * (P["S"] / C["S"]) / wc
        elif phase == 5:  # L2T, own leaves
            d = self.lv[L]
            w = np.repeat(d["quad"][0], d["np"]) * d["quad"][1]
            norm = -1j * k / (16.0 * np.pi ** 2)
            for li in range(self.lb, self.le):
                b, e = self.leaf_start[li], self.leaf_start[li + 1]
                rel = self.pos[b:e] - d["centers"][li]
                self.pot[b:e] = norm * (np.exp(-1j * k * (rel @ d["dirs"].T)) @ (w * self.loc[L][li]))
        elif phase == 6:  # near field with ghosts
            for li in range(self.lb, self.le):
                b, e = self.leaf_start[li], self.leaf_start[li + 1]
                nb = self.near[self.near_off[li]:self.near_off[li + 1]]
                srcs = np.concatenate([np.arange(self.leaf_start[j], self.leaf_start[j + 1]) for j in nb])
                dv = self.pos[b:e, None, :] - self.pos[None, srcs, :]
                r = np.sqrt((dv * dv).sum(-1))
                ok = r > 0
                g = np.where(ok, np.exp(-1j * k * r) / (4.0 * np.pi * np.where(ok, r, 1.0)), 0.0)
                self.pot[b:e] += g @ self.q[srcs]
        elif phase == 7:  # near-field start: the CPU stand-in evaluates it at the join
            pass
        else:
            raise ValueError(phase)

    def _poison_partials(self):
        """Rows of plural nodes outside this rank's slice hold partial sums
        after the reduce-scatter: nothing downstream may read them."""
        if not getattr(self, "_poison_plural", False):
            return
        self._poison_plural = False
        for l, d in self.lv.items():
            for n in d["held"]:
                if d["plural"][n]:
                    b, e = d["mine"][int(n)]
                    self.mp[l][n, :b] = np.nan
                    self.mp[l][n, e:] = np.nan

    def synchronize(self):
        pass

    def potentials_own(self):
        return self.pb, self.pot[self.pb:self.pe].copy()
