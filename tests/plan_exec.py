"""Execute a qsim_plan_json plan on ONE numpy array in PHYSICAL index order
(test infrastructure).  Checks the planner's reordering, sigma bookkeeping,
relabels and exchanges (as index-bit interchanges, Eq. onequbitchange) on
the CPU, independently of the CUDA kernels."""
from __future__ import annotations

import json

import numpy as np


def _apply_u4(psi, idx, t, t2, m):
    """Fused 4x4 block: index j = bit_t + 2 bit_t2, m = 4 rows of 4 complex."""
    U = np.asarray(m, dtype=np.float64).reshape(4, 4, 2)
    U = U[..., 0] + 1j * U[..., 1]
    b0 = idx[(idx & ((1 << t) | (1 << t2))) == 0]
    ii = [b0, b0 | (1 << t), b0 | (1 << t2), b0 | (1 << t) | (1 << t2)]
    x = np.stack([psi[i] for i in ii])
    y = U @ x
    for r in range(4):
        psi[ii[r]] = y[r]


def _apply(psi, idx, code, t, cm, cv, m):
    if code in (6, 8):  # phase-run flush marker / U4 data rows
        return
    sel = (idx & cm) == cv
    if code in (3, 5):  # PHASE / PHASE_ACC
        psi[sel] *= complex(m[0], m[1])
        return
    tb = 1 << t
    i0 = idx[sel & ((idx & tb) == 0)]
    i1 = i0 | tb
    x, y = psi[i0].copy(), psi[i1].copy()
    if code == 2:  # exact swap
        psi[i0], psi[i1] = y, x
        return
    u00, u01 = complex(m[0], m[1]), complex(m[2], m[3])
    u10, u11 = complex(m[4], m[5]), complex(m[6], m[7])
    psi[i0] = u00 * x + u01 * y
    psi[i1] = u10 * x + u11 * y


def _apply_perm(psi, idx, perm, T, cm):
    w = np.zeros_like(idx)
    for b, p in enumerate(T):
        w |= ((idx >> p) & 1) << b
    pw = np.asarray(perm, dtype=np.int64)[w]
    dest = idx.copy()
    for b, p in enumerate(T):
        dest = (dest & ~(1 << p)) | (((pw >> b) & 1) << p)
    sel = (idx & cm) == cm
    new = psi.copy()
    new[dest[sel]] = psi[idx[sel]]
    return new


def _store_remap(psi, idx, tp, tp_out):
    """A pass stores tile bit t at physical bit tp_out[t] (was tp[t]): the
    amplitude at index i moves to the index with those bits permuted."""
    if list(tp) == list(tp_out):
        return psi
    j = idx.copy()
    for a, b in zip(tp, tp_out):
        j &= ~(1 << b)
    for a, b in zip(tp, tp_out):
        j |= ((idx >> a) & 1) << b
    new = np.empty_like(psi)
    new[j] = psi
    return new


def _swap_bits(idx, a, b):
    ba, bb = (idx >> a) & 1, (idx >> b) & 1
    return idx ^ ((ba ^ bb) << a) ^ ((ba ^ bb) << b)


def run_plan(js: str, n: int, init_index: int, gates) -> np.ndarray:
    d = json.loads(js)
    plan = d["plan"]
    phys0 = d["initial_phys_of"]
    idx = np.arange(1 << n, dtype=np.int64)
    psi = np.zeros(1 << n, dtype=np.complex128)
    p0 = sum(((init_index >> q) & 1) << phys0[q] for q in range(n))
    psi[p0] = 1.0
    for st in plan["steps"]:
        ty = st["type"]
        if ty == "pass":
            for op in st["ops"]:
                if op["code"] in (4, 6, 8):
                    continue
                if op["code"] == 7:
                    _apply_u4(psi, idx, op["t"], op["t2"], op["m"])
                    continue
                _apply(psi, idx, op["code"], op["t"], op["cm"], op["cv"], op["m"])
            psi = _store_remap(psi, idx, st["tp"], st.get("tp_out", st["tp"]))
        elif ty == "generic":
            _apply(psi, idx, st["code"], st["t"], st["cm"], st["cv"], st["m"])
        elif ty == "phase":
            _apply(psi, idx, 3, -1, st["cm"], st["cv"], st["m"])
        elif ty == "permrun":  # the run's perms in order, each with its own controls
            for gid, cm in zip(st["gates"], st["cms"]):
                psi = _apply_perm(psi, idx, gates[gid].perm, st["targets"], cm)
        elif ty == "perm":
            g = gates[st["gate"]]
            T = st["targets"]
            cm = st["cm"]
            new = psi.copy()
            w = np.zeros_like(idx)
            for b, p in enumerate(T):
                w |= ((idx >> p) & 1) << b
            pw = np.asarray(g.perm, dtype=np.int64)[w]
            dest = idx.copy()
            for b, p in enumerate(T):
                dest = (dest & ~(1 << p)) | (((pw >> b) & 1) << p)
            sel = (idx & cm) == cm
            new[dest[sel]] = psi[idx[sel]]
            psi = new
        elif ty == "exchange":
            j = idx
            for a, b in zip(st["lpos"], st["gpos"]):
                j = _swap_bits(j, a, b)
            new = np.empty_like(psi)
            new[j] = psi
            psi = new
        elif ty == "relabel":
            pass
        elif ty == "pairwise":  # a gate on a nonlocal bit: in one array it is just that bit
            _apply(psi, idx, st["code"], st["t"], st["cm"], st["cv"], st["m"])
        else:
            raise ValueError(ty)
    fin = plan["final_phys_of"]
    phys = np.zeros_like(idx)
    for q in range(n):
        phys |= ((idx >> q) & 1) << fin[q]
    return psi[phys]
