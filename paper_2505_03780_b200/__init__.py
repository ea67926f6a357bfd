"""B200-native (sm_100a) flash-attention forward — causal varlen prefill + paged-KV decode —
behind the ktune autotuner's config-space API and runner protocol (arXiv 2505.03780)."""

__version__ = "0.1.0"

from .attention import (  # noqa: E402,F401
    cache_append,
    combine,
    paged_decode,
    prefill_varlen,
)
