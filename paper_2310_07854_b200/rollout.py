"""Device-resident rollout runner over the C ABI (the call a user makes).

`Rollout` owns one libvapr context plus the device buffers of one batch of
trajectories (q, world_idx, the cost_grad workspace and the outputs), all
allocated once with PyTorch; `run()` enqueues `vapr_cost_grad` on the current
stream and returns without synchronising.  `run_host()` is the end-to-end
variant: pinned host q in, host grad_q / cost_traj out, copies included.
"""
import numpy as np
import torch

from . import binding as vb

SLOT_NAMES = ("out_spheres", "grad_out_spheres", "out_vec", "closest_pt", "closest_pt_swept")


class Context:
    """RAII wrapper of a vapr_ctx."""

    def __init__(self, device=0, robot=None, formats=None, cuboids=None, offsets=None,
                 goals=None):
        self.device = int(device)
        self.h = vb.vapr_create(self.device)
        if robot is not None:
            vb.vapr_set_robot(self.h, robot)
        if formats is not None:
            self.set_formats(formats)
        if cuboids is not None:
            vb.vapr_set_worlds(self.h, cuboids, offsets)
        if goals is not None:
            vb.vapr_set_goals(self.h, goals)

    def set_formats(self, formats):
        self.formats = tuple(tuple(f) for f in formats)
        vb.vapr_set_formats(self.h, self.formats)

    def set_cull(self, on):
        vb.vapr_set_option(self.h, vb.VAPR_OPT_CULL, int(on))

    def set_streams(self, n):
        vb.vapr_set_option(self.h, vb.VAPR_OPT_STREAMS, int(n))

    def set_sparse(self, on):
        """N3: grad_out_spheres in the sparse form inside vapr_cost_grad."""
        vb.vapr_set_option(self.h, vb.VAPR_OPT_SPARSE, int(on))

    def set_fused(self, on):
        """N4: the whole rollout in one kernel, no tensor materialised."""
        vb.vapr_set_option(self.h, vb.VAPR_OPT_FUSED, int(on))

    def close(self):
        if self.h is not None:
            vb.vapr_destroy(self.h)
            self.h = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass


class Rollout:
    """One batch [B, H] of trajectories resident in HBM."""

    def __init__(self, workload, device=0, formats=None, ctx=None, sparse=False, fused=False):
        self.wl = workload
        self.device = torch.device("cuda", device)
        self.ctx = ctx or Context(device, workload.robot, formats or workload.formats,
                                  workload.cuboids, workload.world_offsets,
                                  getattr(workload, "goals", None))
        if formats is not None and ctx is not None:
            self.ctx.set_formats(formats)
        self.sparse = bool(sparse)
        if sparse:
            self.ctx.set_sparse(True)
        self.fused = bool(fused)
        if fused:
            self.ctx.set_fused(True)
        self.B, self.H = workload.B, workload.H
        self.params = dict(workload.params)
        self._p = vb.cost_params(self.params)
        d = self.device
        self.q = torch.from_numpy(np.ascontiguousarray(workload.q)).to(d)
        self.world_idx = torch.from_numpy(np.ascontiguousarray(workload.world_idx, np.int32)).to(d)
        nbytes = vb.vapr_cost_grad_workspace_bytes(self.ctx.h, self.B, self.H)
        self.workspace = torch.zeros(nbytes, dtype=torch.uint8, device=d)
        self.cost_pose = torch.zeros(self.B * self.H, dtype=torch.float32, device=d)
        self.cost_traj = torch.zeros(self.B, dtype=torch.float32, device=d)
        self.grad_q = torch.zeros(self.B * self.H * 7, dtype=torch.float32, device=d)

    def set_formats(self, formats):
        self.ctx.set_formats(formats)
        need = vb.vapr_cost_grad_workspace_bytes(self.ctx.h, self.B, self.H)
        if need > self.workspace.numel():
            self.workspace = torch.zeros(need, dtype=torch.uint8, device=self.device)

    def run(self, stream=None):
        """Enqueue vapr_cost_grad on `stream` (default: the current stream of
        this rollout's device, not of the current device)."""
        if stream is None:
            stream = torch.cuda.current_stream(self.device).cuda_stream
        vb.vapr_cost_grad(self.ctx.h, self.q, self.world_idx, self.B, self.H, self.params,
                          self.workspace, self.cost_pose, self.cost_traj, self.grad_q,
                          stream=stream, _p=self._p)

    def capture_graph(self, warmup=2):
        """vapr_cost_grad captured in a CUDA graph (SURVEY.md §8(d) timing
        protocol; launch-bound small batches): replay() re-runs it on the
        buffers' current contents (update q in place between replays)."""
        import torch
        s = torch.cuda.Stream(self.device)
        s.wait_stream(torch.cuda.current_stream(self.device))
        with torch.cuda.stream(s):
            for _ in range(warmup):
                self.run()
        torch.cuda.current_stream(self.device).wait_stream(s)
        g = torch.cuda.CUDAGraph()
        with torch.cuda.graph(g):
            self.run()
        return g

    def run_host(self, q_host, grad_q_host, cost_traj_host=None, n_chunks=0, stream=None):
        """End to end from host buffers: q_host [B, H, 7] float32 in, grad_q_host
        [B, H, 7] (and cost_traj_host [B]) out, copies pipelined against the
        compute inside vapr_cost_grad_host; stream-ordered (synchronise the
        stream before reading the host outputs).  Pinned host tensors overlap."""
        vb.vapr_cost_grad_host(self.ctx.h, q_host, self.world_idx, self.B, self.H, self.params,
                               self.workspace, self.q, self.cost_pose, self.cost_traj,
                               self.grad_q, cost_traj_host, grad_q_host, n_chunks,
                               stream=stream, _p=self._p)

    def _rows_of_pool(self, mask, pool_t, base, wmax, pf):
        out = []
        for i, mi in enumerate(mask):
            n = -(-3 * bin(int(mi)).count("1") // pf)
            o = base + i * wmax
            out.append(pool_t[o:o + n].cpu().numpy().view(np.uint32))
        return out

    def sparse_gos(self, rows=None):
        """N3 (sparse mode): grad_out_spheres' mask [P] uint64, off [P], the
        pool (its whole capacity) and the count of words in use, as numpy
        arrays.  rows (a slice of poses): only those rows' masks / offsets,
        and `row_words` = each of those rows' pool words."""
        torch.cuda.synchronize(self.device)
        lay, pw = vb.vapr_cost_grad_sparse_layout(self.ctx.h, self.B, self.H)
        mo, oo, uo, po = lay[:4]
        P = self.B * self.H
        ws = self.workspace
        mask = ws[mo:mo + 8 * P].view(torch.int64)
        off = ws[oo:oo + 4 * P].view(torch.int32)
        used = int(ws[uo:uo + 4].view(torch.int32).cpu().numpy().view(np.uint32)[0])
        pool_t = ws[po:po + 4 * pw].view(torch.int32)
        if rows is None:
            return dict(mask=mask.cpu().numpy().view(np.uint64), off=off.cpu().numpy().view(np.uint32),
                        pool=pool_t.cpu().numpy().view(np.uint32), used=used)
        m = mask[rows].cpu().numpy().view(np.uint64)
        o = off[rows].cpu().numpy().view(np.uint32)
        fmt = self.ctx.formats[vb.VAPR_GRAD_OUT_SPHERES]
        pf = 32 // (1 + fmt[0] + (fmt[1] & 0xFF))
        rw = []
        for mi, oi in zip(m, o):
            n = -(-3 * bin(int(mi)).count("1") // pf)
            rw.append(pool_t[int(oi):int(oi) + n].cpu().numpy().view(np.uint32))
        return dict(mask=m, off=o, row_words=rw, used=used)

    def sparse_slot(self, slot, rows=None):
        """N3 (sparse mode): a collision output (closest_pt[_swept] or out_vec)
        in the sparse form -- its sphere bitmaps [P] (or of the poses in `rows`)
        and each row's packed codes (row p at pool word p * ceil(cols / pf))."""
        torch.cuda.synchronize(self.device)
        lay, _ = vb.vapr_cost_grad_sparse_layout(self.ctx.h, self.B, self.H)
        is_ov = slot == vb.VAPR_OUT_VEC
        mo, po = (lay[5], lay[7]) if is_ov else (lay[4], lay[6])
        P = self.B * self.H
        fmt = self.ctx.formats[slot]
        pf = 32 // (1 + fmt[0] + (fmt[1] & 0xFF))
        cols = 3 * len(self.wl.robot["sphere_link"])
        wmax = -(-cols // pf)
        ws = self.workspace
        rows = rows if rows is not None else slice(0, P)
        mask = ws[mo:mo + 8 * P].view(torch.int64)[rows].cpu().numpy().view(np.uint64)
        pool_t = ws[po:po + 4 * wmax * P].view(torch.int32)
        return dict(mask=mask, row_words=self._rows_of_pool(mask, pool_t, wmax * rows.start, wmax, pf))

    def packed_dense(self, slot, rows=None):
        """N3 (sparse mode): a collision output densified by the oracle's
        definition (oracle/sparse.py) into the dense packed rows."""
        from oracle import codec, sparse as osp
        sp = self.sparse_slot(slot, rows)
        fmt = self.ctx.formats[slot]
        cols = 3 * len(self.wl.robot["sphere_link"])
        return codec.pack(osp.densify(sp["mask"], sp["row_words"], fmt[0], fmt[1] & 0xFF, cols),
                          fmt[0], fmt[1] & 0xFF)

    def packed(self, slot, rows=None):
        """The packed tensor of `slot` inside the workspace, as uint32 [P, W]
        (or the poses in `rows`, a slice)."""
        lay = vb.vapr_cost_grad_workspace_layout(self.ctx.h, self.B, self.H, self.params["swept"])
        off = lay[slot]
        if off is None:
            return None
        fmt = self.ctx.formats[slot]
        W = vb.vapr_packed_row_words(fmt, 3 * len(self.wl.robot["sphere_link"]))
        P = self.B * self.H
        words = self.workspace[off:off + 4 * W * P].view(torch.int32).view(P, W)
        if rows is not None:
            words = words[rows]
        return words.cpu().numpy().view(np.uint32)

    def results(self):
        torch.cuda.synchronize(self.device)
        return dict(cost_pose=self.cost_pose.cpu().numpy().reshape(self.B, self.H),
                    cost_traj=self.cost_traj.cpu().numpy(),
                    grad_q=self.grad_q.cpu().numpy().reshape(self.B, self.H, 7))
