"""pytest plugin (-p ref_shim): make ``import kvmix`` resolve its hot path to this package.

``kvmix.quant``, ``kvmix.pool``, ``kvmix.errors`` and the decode entry points of
``kvmix.attention`` (flash_decode, merge_partials, SplitPartial) plus the calibration
replay pieces this package runs on the GPU (apply_mixed_quantization, attention_full,
output_mse_per_head: SURVEY 8(f) rank 4) are paper_2605_17170_b200's; every other name --
the tagger, captures, the sensitivity tables, the allocator, the CLI, and the remaining
CPU helpers of attention.py (attention_selective_quant, output_mse, ...) -- is the
reference's own code from the vendored copy (tools/vendor_ref_suite.py), which stays on
the host per the north_star.  The reference's tests then run unmodified.
"""
import importlib.util
import os
import sys
import types

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(os.path.dirname(HERE))
SRC = os.path.join(HERE, "_vendored", "src")
sys.path.insert(0, ROOT)

import paper_2605_17170_b200 as ours  # noqa: E402
from paper_2605_17170_b200 import attention as ours_att  # noqa: E402
from paper_2605_17170_b200 import calib as ours_calib  # noqa: E402
from paper_2605_17170_b200 import errors as ours_err  # noqa: E402
from paper_2605_17170_b200 import pool as ours_pool  # noqa: E402
from paper_2605_17170_b200 import quant as ours_quant  # noqa: E402

# kvmix.report (plots; out of scope) imports matplotlib at module level, which this image
# lacks: a stub lets test_acceptance.py import kvmix.cli (criterion 10, the CLI run, is
# not among the hot-path criteria this suite selects).
try:
    import matplotlib  # noqa: F401
except ImportError:
    _mpl = types.ModuleType("matplotlib")
    _mpl.use = lambda *a, **k: None
    _mpl.pyplot = types.ModuleType("matplotlib.pyplot")
    sys.modules["matplotlib"] = _mpl
    sys.modules["matplotlib.pyplot"] = _mpl.pyplot

# the package object first (its __init__ runs last, after the submodules are in place)
spec = importlib.util.spec_from_file_location("kvmix", os.path.join(SRC, "kvmix", "__init__.py"),
                                              submodule_search_locations=[os.path.join(SRC, "kvmix")])
kvmix = importlib.util.module_from_spec(spec)
sys.modules["kvmix"] = kvmix
for name, mod in (("quant", ours_quant), ("pool", ours_pool), ("errors", ours_err)):
    sys.modules[f"kvmix.{name}"] = mod
    setattr(kvmix, name, mod)



def _load_ref(name):
    """A vendored reference module under a private name."""
    sp = importlib.util.spec_from_file_location(f"kvmix._ref_{name}", os.path.join(SRC, "kvmix", f"{name}.py"))
    mod = importlib.util.module_from_spec(sp)
    sys.modules[sp.name] = mod
    sp.loader.exec_module(mod)
    return mod


# The reference's attention.py for its CPU-only helpers; its fake-quant helpers import the
# reference codec's private functions (quant.py:27-50), so it is loaded against the
# reference quant module and then kvmix.quant points back at this package.
ref_quant = _load_ref("quant")
sys.modules["kvmix.quant"] = ref_quant
ref_att = _load_ref("attention")
sys.modules["kvmix.quant"] = ours_quant


def _np(x):
    return x.detach().cpu().numpy() if hasattr(x, "detach") else x


def apply_mixed_quantization(k, v, row_bits, group_len=ours_quant.GROUP_SIZE):
    kq, vq = ours_calib.apply_mixed_quantization(k, v, row_bits, group_len=group_len)
    return _np(kq), _np(vq)


def attention_full(q, k, v, scale=None, causal=False, return_probs=False):
    if return_probs:  # the probabilities are a reference debugging aid, not part of the replay
        return ref_att.attention_full(q, k, v, scale=scale, causal=causal, return_probs=True)
    import torch
    dev = torch.device("cuda", torch.cuda.current_device())
    t = [torch.as_tensor(np.asarray(x, np.float32), device=dev) for x in (q, k, v)]
    return _np(ours_calib.attention_full(*t, scale=scale, causal=causal))


def output_mse_per_head(o_ref, o_test):
    import torch
    return ours_calib.output_mse_per_head(torch.as_tensor(np.asarray(o_ref)), torch.as_tensor(np.asarray(o_test)))


att = types.ModuleType("kvmix.attention")
att.__dict__.update({k: v for k, v in vars(ref_att).items() if not k.startswith("__")})
att.__dict__.update(flash_decode=ours_att.flash_decode, merge_partials=ours_att.merge_partials,
                    SplitPartial=ours_att.SplitPartial, apply_mixed_quantization=apply_mixed_quantization,
                    attention_full=attention_full, output_mse_per_head=output_mse_per_head)
sys.modules["kvmix.attention"] = att
kvmix.attention = att
spec.loader.exec_module(kvmix)
assert kvmix.quant is ours_quant and kvmix.pool is ours_pool and kvmix.attention.flash_decode is ours.flash_decode
