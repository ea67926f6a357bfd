"""ktune protocol-v1 benchmark runner for the sm_100a attention kernels.

Drop-in for the reference runner (ref/pkg/runner/src/ktune_triton_runner): same invocation
(``<runner> --binding F --protocol 1``, ref/SPEC.md:602), same wire messages and failure
mapping, so the unmodified ``ktune tune`` / ``ktune runner-check`` drive it.
"""

PROTOCOL_VERSION = 1
RUNNER_ID = "b200attn-runner"
