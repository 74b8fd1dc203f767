"""Helpers shared by the -m gpu parity tests: move a workloads.Problem onto the device,
read back column-major [A | b] rows, and the A14 scale-normalised entry metric."""
import numpy as np
import torch

from paper_2602_10541_b200 import fls

ENTRY_TOL = 1e-12      # north_star: <= 1e-12 relative per entry, read as |dA| <= 1e-12 * S_ij (A14)
U_TOL = 1e-6           # north_star: <= 1e-6 relative L2 of the fitted u at 10,000 held-out points


def dev_blocks(problem, device="cuda"):
    out = []
    for blk in problem.blocks:
        out.append(fls.Block(
            X=torch.from_numpy(blk.X).to(device),
            terms=[(tuple(a), float(c), int(f)) for a, c, f in blk.terms],
            weight=float(blk.weight),
            values=torch.from_numpy(blk.values).to(device),
            fields=torch.from_numpy(blk.fields).to(device) if blk.fields is not None else None))
    return out


def rows_from_colmajor(Ab, lda, F, rows_local):
    """(len(rows), F) A entries and (len(rows),) rhs from the flat column-major [A | b]."""
    M = Ab[: (F + 1) * lda].view(F + 1, lda)          # M[j, i] = A_ij
    idx = torch.as_tensor(np.asarray(rows_local), device=Ab.device, dtype=torch.long)
    sub = M.index_select(1, idx).cpu().numpy()        # (F+1, n)
    return np.ascontiguousarray(sub[:F].T), sub[F].copy()


def scaled_err(A_gpu, A_orc, S):
    """max and p99.9 of |A_gpu - A_orc| / S (S = sum of absolute term magnitudes, A14)."""
    e = np.abs(A_gpu - A_orc) / np.maximum(S, 1e-300)
    return float(e.max()), float(np.quantile(e, 0.999))
