"""attnkit/b200.py -- the reference-side binding a maintainer adds to attnkit (arXiv 2603.02188)
to route the latent branch of ``attend_local`` + ``reduce_contributions`` through the B200
library (include/mlra_b200.h, libmlra_b200.so), keeping attnkit's own data structures: its
``KvCache`` (numpy rows), ``Ownership`` / ``LatentUnit``, ``local_weights`` slices and
``token_queries`` dicts.

It imports nothing from this repo's Python package: only ctypes, numpy, torch (device memory
and the stream) and attnkit itself. The hook in attnkit is one branch at the top of
``absorbed_decode_step`` (attnkit/decode.py:290-306):

    if os.environ.get("ATTNKIT_BACKEND") == "b200" and cfg.variant in ("mla", "mlra"):
        from .b200 import absorbed_decode_step as _b200_step
        return _b200_step(cfg, w, cache, h_t)

Served ownerships: every unit serves the same heads (MLRA-4 and MLA, full ownership or a
tensor-parallel shard of them). Errors are attnkit's own classes (attnkit/errors.py).
"""

from __future__ import annotations

import ctypes
import math
import os

import numpy as np

LIB_ENV = "MLRA_B200_LIB"
_DEFAULT_LIB = os.path.join(os.path.dirname(os.path.abspath(__file__)), "..", "paper_2603_02188_b200",
                            "libmlra_b200.so")
_P, _I, _F = ctypes.c_void_p, ctypes.c_int, ctypes.c_float
#: the entry points this binding uses, with the header's signatures (include/mlra_b200.h)
SIGNATURES = {
    "mlra_last_error": (ctypes.c_char_p, []),
    "mlra_workspace_bytes": (ctypes.c_size_t, [_I] * 6),
    "mlra_default_splits": (_I, [_I] * 4),
    "mlra_check_status": (_I, [_P, _I, _P]),
    "mlra_decode_step": (_I, [_P] * 9 + [_I] * 11 + [_F, _F, _P]),
}
PAGE = 128  # tokens per page of the packed pool
_lib = None


def load_library(path: str | None = None):
    global _lib
    if _lib is None:
        lib = ctypes.CDLL(path or os.environ.get(LIB_ENV, _DEFAULT_LIB))
        for name, (res, args) in SIGNATURES.items():
            fn = getattr(lib, name)
            fn.restype, fn.argtypes = res, args
        _lib = lib
    return _lib


def _errors():
    from attnkit import errors  # attnkit's own classes: callers catch AttnKitError as before

    return errors


def _pad_latent(dl: int) -> int:  # unit width in the pool: 64, or a multiple of 128
    return 64 if dl <= 64 else -(-dl // 128) * 128


def _pad_rope(dr: int) -> int:
    return max(16, -(-dr // 16) * 16)


def attend_reduce_gpu(cfg, local_w, own, cache, queries, alpha: float) -> np.ndarray:
    """``reduce_contributions(cfg, attend_local(cfg, local_w, own, cache, queries))[0]`` rows of
    the owned heads (attnkit/decode.py:217-230, :264-285), on the B200 kernels (K1 absorb, K2
    split-KV decode, K3 merge + W^UV + ascending branch sum + alpha). Returns float64
    [len(own.heads), d_h]; charges ``cache.reads`` exactly like ``KvCache.read``."""
    import torch

    err = _errors()
    units = list(own.units)
    if not units:
        raise err.RoutingError("attend_reduce_gpu serves the latent family (ownership without latent units)")
    heads = list(units[0].heads)
    if any(list(u.heads) != heads for u in units) or list(own.heads) != heads:
        raise err.RoutingError("attend_reduce_gpu: every latent unit must serve the owned heads")
    n = cache.n
    if n == 0:
        raise err.ShapeMismatchError("attend on an empty cache")
    lib = load_library()
    dl = int(np.asarray(cache.peek(units[0].stream)).shape[1])
    dr = int(np.asarray(cache.peek("rope")).shape[1])
    dlp, drp = _pad_latent(dl), _pad_rope(dr)
    nb = len(units)
    width, pages = nb * dlp + drp, -(-n // PAGE)
    rows = np.zeros((pages * PAGE, width), np.float32)  # [unit 0 | ... | unit NB-1 | rope] per token
    for i, u in enumerate(units):
        rows[:n, i * dlp:i * dlp + dl] = cache.peek(u.stream)
    rows[:n, nb * dlp:nb * dlp + dr] = cache.peek("rope")
    dev = torch.device("cuda", torch.cuda.current_device())
    pool = torch.tensor(rows, device=dev).to(torch.bfloat16)
    bt = torch.arange(pages, dtype=torch.int32, device=dev)[None]
    lens = torch.tensor([n], dtype=torch.int32, device=dev)
    H, DH = len(heads), cfg.d_h
    uk = np.zeros((H, DH, nb * dlp), np.float32)
    uv = np.zeros((H, nb * dlp, DH), np.float32)
    for i, u in enumerate(units):  # local_w["uk:<stream>"] is (latent, heads, d_h) (decode.py:185-186)
        uk[:, :, i * dlp:i * dlp + dl] = np.asarray(local_w[f"uk:{u.stream}"]).transpose(1, 2, 0)
        uv[:, i * dlp:i * dlp + dl, :] = np.asarray(local_w[f"uv:{u.stream}"]).transpose(1, 0, 2)
    qn = torch.tensor(np.asarray(queries["q_nope"])[heads], device=dev).to(torch.bfloat16)[None].contiguous()
    qr = torch.zeros((1, H, drp), device=dev, dtype=torch.bfloat16)
    qr[0, :, :dr] = torch.tensor(np.asarray(queries["q_rope"])[heads], device=dev)
    w_uk = torch.tensor(uk, device=dev).to(torch.bfloat16)
    w_uv = torch.tensor(uv, device=dev).to(torch.bfloat16)
    sub, dls = (dlp // 128, 128) if dlp % 128 == 0 else (1, 64)
    nsplit = lib.mlra_default_splits(1, n, nb, sub)
    ws = torch.zeros(lib.mlra_workspace_bytes(1, H, nb, dlp, drp, nsplit), dtype=torch.uint8, device=dev)
    out = torch.empty((1, H, DH), dtype=torch.float32, device=dev)
    stream = torch.cuda.current_stream().cuda_stream
    rc = lib.mlra_decode_step(qn.data_ptr(), qr.data_ptr(), w_uk.data_ptr(), w_uv.data_ptr(), pool.data_ptr(),
                              bt.data_ptr(), lens.data_ptr(), out.data_ptr(), ws.data_ptr(), 1, H, DH, nb, sub, dls,
                              drp, PAGE, pages, pages, nsplit, float(cfg.tau) * math.log2(math.e), float(alpha), stream)
    if rc != 0:
        raise err.AttnKitError(f"mlra_decode_step: {lib.mlra_last_error().decode(errors='replace')}")
    if lib.mlra_check_status(ctypes.c_void_p(ws.data_ptr()), 1, stream) != 0:  # tensors.py:74-78
        raise err.NumericError("softmax_rows: NaN in logits or a row with no finite logit")
    cache.reads += n * cache.row_elements()  # the charge of reading every owned stream once
    return out[0].double().cpu().numpy()


def absorbed_decode_step(cfg, w, cache, h_t):
    """attnkit/decode.py:290-306 with attend_local + reduce_contributions on the B200: the
    cache append, projections and ownership stay attnkit's own code."""
    from attnkit.decode import append_owned, full_ownership, local_weights, token_cache_rows, token_queries
    from attnkit.latent import calib_factors

    if cfg.variant not in ("mla", "mlra") or (cfg.variant == "mlra" and cfg.branches != 4):
        raise _errors().RoutingError(f"the B200 binding serves MLA and MLRA-4; got {cfg.variant!r}")
    pos = cache.pos_offset + cache.n
    own = full_ownership(cfg)
    append_owned(cfg, own, cache, token_cache_rows(cfg, w, h_t, pos))
    queries = token_queries(cfg, w, h_t, pos)
    alpha = calib_factors(cfg).alpha_attn if cfg.variant == "mlra" else 1.0
    out = attend_reduce_gpu(cfg, local_weights(cfg, w, own), own, cache, queries, alpha)
    return out, cache
