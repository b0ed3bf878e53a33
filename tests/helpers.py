"""Test-side helpers (no oracle arithmetic, no product code)."""
import numpy as np


def rel_frob(a, b):
    a = np.asarray(a, np.float64)
    b = np.asarray(b, np.float64)
    return float(np.linalg.norm(a - b) / max(np.linalg.norm(b), 1e-30))


def bf16_round(x):
    """float32 -> bf16 (round-to-nearest-even) -> float32, via integer arithmetic."""
    x = np.ascontiguousarray(x, np.float32)
    u = x.view(np.uint32).astype(np.uint64)
    u = (u + 0x7FFF + ((u >> 16) & 1)) & 0xFFFF0000
    return u.astype(np.uint32).view(np.float32)


def predict_from_state(W, m, v, k, s, lr, b1, b2, eps, bf16=True):
    """The north-star prediction W_hat = W - s*lr*m_hat/(sqrt(v_hat)+eps) evaluated from a
    stage's own (W, m, v, version k) in the fp32 op order of DESIGN.md section 4 -- used to
    check the GPU's materialised W_hat buffers against the GPU's own state (O8 item 4)."""
    W, m, v = (np.asarray(a, np.float32) for a in (W, m, v))
    if k == 0:
        return bf16_round(W) if bf16 else W.copy()
    b1d, b2d = float(np.float32(b1)), float(np.float32(b2))
    b1p = b2p = 1.0
    for _ in range(k):
        b1p *= b1d
        b2p *= b2d
    c1 = np.float32(float(np.float32(lr)) / (1.0 - b1p))
    r2 = np.float32(1.0 / np.sqrt(1.0 - b2p))
    den = np.sqrt(v) * r2 + np.float32(eps)
    d = (c1 * m) / den
    # fmaf(-s, d, W): -s*d is exact in double and the double sum is exact here -> one rounding
    p = (-(float(s)) * d.astype(np.float64) + W.astype(np.float64)).astype(np.float32)
    return bf16_round(p) if bf16 else p


def log_parity(name, **fields):
    """Append one parity record (relFrob curves, margins) as a JSON line to $XPIPE_PARITY_LOG
    when set, so GPU runs can bring the curves back for profiles/."""
    import json
    import os
    path = os.environ.get("XPIPE_PARITY_LOG")
    if not path:
        return
    os.makedirs(os.path.dirname(os.path.abspath(path)), exist_ok=True)
    with open(path, "a") as f:
        f.write(json.dumps(dict(test=name, **fields)) + "\n")
