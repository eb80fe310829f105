"""pytest plugin (debug only): report non-finite values in backward workspaces."""
import threading
import torch


def pytest_configure(config):
    from paper_2403_09347_b200 import kernels as K
    o_fin = K.CudaKernels.bwd_finalize
    o_fin_q = K.CudaKernels.bwd_finalize_qtravel
    o_acc = K.CudaKernels.accumulate

    def nz(name, t):
        torch.cuda.current_stream().synchronize()
        bad = (~torch.isfinite(t)).sum().item()
        if bad:
            idx = (~torch.isfinite(t)).nonzero()[:4].flatten().tolist()
            print(f"\n[nanplug] {threading.current_thread().name} {name}: {bad} non-finite, first idx {idx}, numel {t.numel()}", flush=True)

    def fin(self, st, dk_parts, dv_parts, dq, dk, dv, stream=None):
        with torch.cuda.stream(stream):
            nz("dq_acc", st.dq_acc)
            for i, p in enumerate(dk_parts): nz(f"dk_part{i}", p)
            for i, p in enumerate(dv_parts): nz(f"dv_part{i}", p)
            nz("stats", st.stats)
        return o_fin(self, st, dk_parts, dv_parts, dq, dk, dv, stream)

    def finq(self, st, dq_parts, dk_acc, dv_acc, dq, dk, dv, stream=None):
        with torch.cuda.stream(stream):
            nz("dq_acc(q)", st.dq_acc)
            for i, p in enumerate(dq_parts): nz(f"dq_part{i}", p)
            nz("dk_acc(q)", dk_acc); nz("dv_acc(q)", dv_acc); nz("stats(q)", st.stats)
        return o_fin_q(self, st, dq_parts, dk_acc, dv_acc, dq, dk, dv, stream)

    def acc(self, acc_pair, part_pair, like, stream=None):
        with torch.cuda.stream(stream):
            for i, p in enumerate(part_pair): nz(f"fold_part{i}", p)
            for i, p in enumerate(acc_pair): nz(f"fold_acc{i}", p)
        return o_acc(self, acc_pair, part_pair, like, stream)

    K.CudaKernels.bwd_finalize = fin
    K.CudaKernels.bwd_finalize_qtravel = finq
    K.CudaKernels.accumulate = acc


def _patch_bwd():
    from paper_2403_09347_b200 import kernels as K
    o_bwd = K.CudaKernels.bwd

    def cnt(t):
        return int((~torch.isfinite(t)).sum().item())

    def bwd(self, plan, q, k, v, dout, scale, st, dk_part, dv_part, accumulate, stream=None):
        s = stream if stream is not None else torch.cuda.current_stream()
        s.synchronize()
        before = (cnt(dk_part), cnt(dv_part), cnt(st.stats), cnt(q), cnt(dout), cnt(k), cnt(v))
        o_bwd(self, plan, q, k, v, dout, scale, st, dk_part, dv_part, accumulate, stream)
        s.synchronize()
        after = (cnt(dk_part), cnt(dv_part), cnt(st.dq_acc))
        if any(before) or any(after):
            print(f"\n[nanplug-bwd] {threading.current_thread().name} q[{plan.q_begin},+{plan.q_len}) "
                  f"k[{plan.k_begin},+{plan.k_len}) causal={plan.causal} acc={accumulate} "
                  f"before(dk,dv,stats,q,do,k,v)={before} after(dk,dv,dq)={after}", flush=True)
    K.CudaKernels.bwd = bwd


_orig_cfg = pytest_configure


def pytest_configure(config):  # noqa: F811
    _orig_cfg(config)
    _patch_bwd()
