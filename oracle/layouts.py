"""Table 2 of PAPER.md as data, and the spec row (TEST INFRASTRUCTURE).

Each layout is (shape in symbols of b, s, h, p; sharded dim or None; transposed).
Columns: activations (X_MHA, O, X_FFN, Z), W_qkv, W_proj, W_in, W_out.
The "Specification" row is normative (R-28).

Pins: tests/golden/table2.txt transcribes the paper's cells; the test checks
every cell and that all spec-row strategies are pairwise compatible
(SPEC.md:177, 565).
"""
from __future__ import annotations

ROLES = ("act", "w_qkv", "w_proj", "w_in", "w_out")

# cell strings exactly as the paper writes them (after removing LaTeX markup)
TABLE2 = {
    "Megatron-LM TP": ("bxsxh", "hx3h/p", "h/pxh", "hx4h/p", "4h/pxh"),
    "Megatron-LM TP+SP": ("bxs/pxh", "hx3h/p", "h/pxh", "hx4h/p", "4h/pxh"),
    "Megatron-LM CP": ("bxs/pxh", "hx3h", "hxh", "hx4h", "4hxh"),
    "DeepSpeed Ulysses": ("bxs/pxh", "hx3h", "hxh", "hx4h", "4hxh"),
    "DeepSpeed ZeRO3": ("b/pxsxh", "(h/px3h)^T", "h/pxh", "(h/px4h)^T", "4h/pxh"),
    "Colossal-AI SP": ("bxs/pxh", "hx3h", "hxh", "hx4h", "4hxh"),
    "METP": ("bxs/pxh", "hx3h/p", "h/pxh", "hx4h/p", "4h/pxh"),
    "Specification": ("bxs/pxh", "(3h/pxh)^T", "h/pxh", "(4h/pxh)^T", "4h/pxh"),
}


def spec_layout(role, h, p, s=None, b=1):
    """Concrete stored shard shape of `role` under the specification row."""
    if role == "act":
        if s % p:
            raise ValueError(f"s={s} not divisible by p={p}")
        return (b, s // p, h), "s", False
    if role == "w_qkv":
        if (3 * h) % p:
            raise ValueError("3h not divisible by p")
        return (3 * h // p, h), "rows", True
    if role == "w_proj":
        return (h // p, h), "rows", False
    if role == "w_in":
        return (4 * h // p, h), "rows", True
    if role == "w_out":
        return (4 * h // p, h), "rows", False
    raise KeyError(role)


def compatible(a, b):
    """No redistribution iff the two layout cells coincide."""
    return a == b


# strategies of the switchable set and the layout each presents at the boundary
STRATEGY_LAYOUT = {"MegatronTS": "Specification", "UlyssesZ": "Specification",
                   "METP": "Specification"}
