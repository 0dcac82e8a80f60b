"""B200-native decode attention for Multi-Head Low-Rank Attention (MLRA-4), with the MLA and
GQA comparison variants, behind the reference kit's decode API (arXiv 2603.02188, "attnkit").

Drop-in names (attnkit/__init__.py:25-53 subset for the decode path):
``AttnConfig``, ``trained_config``, ``table_context``, ``Rng``, ``WeightSet``,
``build_weights``, ``weight_shapes``, ``calib_factors``, ``new_cache``, ``absorb_query``,
``attend_local``, ``reduce_contributions``, ``absorbed_decode_step``, ``decode_step``,
``make_shards``, ``sim_decode``, ``per_device_load``, ``latent_prefill`` and the error classes;
the output side (``OutputProjection``, ``TpComm``) and the host I/O loop (``MicroBatchLoop``).

Compute runs on hand-written sm_100a kernels (``csrc/``) through the C ABI declared in
``include/mlra_b200.h`` and loaded from the in-tree ``libmlra_b200.so``. Importing the
package does not need a GPU; every compute entry point does (no CPU fallback).
"""

from .config import (GPU_VARIANTS, LATENT_VARIANTS, TP_DEGREES, VARIANTS, AttnConfig, table_context, tiny_config,
                     trained_config)
from .costs import (ScaleFactors, algorithmic_bytes, calib_factors, calib_factors_squared, decode_flops_per_device,
                    kv_cache_per_token, per_device_load)
from .errors import (AttnKitError, ConfigError, CudaError, IntegrityError, NumericError, RoutingError,
                     ShapeMismatchError)
from .weights import Rng, WeightSet, build_weights, gaussian_init, weight_shapes

__version__ = "0.1.0"


def __getattr__(name):
    # torch-dependent modules load lazily so config/oracle-side code can import the package
    # without initialising CUDA.
    lazy = {
        "decode": ("decode", None), "tp": ("tp", None), "cache": ("cache", None), "ops": ("ops", None),
        "LatentUnit": ("decode", "LatentUnit"), "Ownership": ("decode", "Ownership"),
        "full_ownership": ("decode", "full_ownership"), "owned_stream_layout": ("decode", "owned_stream_layout"),
        "new_cache": ("decode", "new_cache"), "absorb_query": ("decode", "absorb_query"),
        "local_weights": ("decode", "local_weights"), "attend_local": ("decode", "attend_local"),
        "reduce_contributions": ("decode", "reduce_contributions"),
        "absorbed_decode_step": ("decode", "absorbed_decode_step"), "decode_step": ("decode", "decode_step"),
        "naive_decode_step": ("decode", "naive_decode_step"), "DecodeEngine": ("decode", "DecodeEngine"),
        "shard_ownership": ("tp", "shard_ownership"), "make_shards": ("tp", "make_shards"),
        "sim_decode": ("tp", "sim_decode"), "ShardSet": ("tp", "ShardSet"), "DeviceShard": ("tp", "DeviceShard"),
        "TrafficLedger": ("tp", "TrafficLedger"), "TPDecodeGroup": ("tp", "TPDecodeGroup"),
        "PagedCache": ("cache", "PagedCache"), "PagedLatentCache": ("cache", "PagedLatentCache"),
        "RowLayout": ("cache", "RowLayout"), "GqaLayout": ("cache", "GqaLayout"),
        "gqa": ("gqa", None), "GqaDecodeEngine": ("gqa", "GqaDecodeEngine"),
        "latent_prefill": ("decode", "latent_prefill"), "PrefillOutput": ("decode", "PrefillOutput"),
        "outproj": ("outproj", None), "OutputProjection": ("outproj", "OutputProjection"),
        "TpComm": ("outproj", "TpComm"), "host_loop": ("host_loop", None),
        "MicroBatchLoop": ("host_loop", "MicroBatchLoop"), "collective": ("collective", None),
        "PeerAllReduce": ("collective", "PeerAllReduce"),
    }
    if name in lazy:
        import importlib

        mod_name, attr = lazy[name]
        mod = importlib.import_module(f".{mod_name}", __name__)
        return mod if attr is None else getattr(mod, attr)
    raise AttributeError(name)
