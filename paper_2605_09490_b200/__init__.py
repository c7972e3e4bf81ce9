"""B200-native tiered KV decode hot path (arXiv 2605.09490).

The product is the C-ABI library ``libkvtier.so`` (include/kv_tier.h); this
package holds its CUDA sources (csrc/), the thin ctypes binding (kvtier.py) and
the step driver used by the tests and bench.py (harness.py).
"""
