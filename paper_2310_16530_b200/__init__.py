"""hcnn-b200: B200-native RNS-CKKS engine for encrypted CNN inference.

Drop-in for the hot path of the reference package ``hcnn``
(/root/reference/pkg/src/hcnn): ``ring`` and ``ckks`` keep its API with
ciphertexts resident in HBM; ``packing`` and ``graph`` run the HyPHEN /
AESPA layers on top.  All integer arithmetic is CUDA (sm_100a) behind the C
ABI in include/hcnn_b200.h; there is no CPU fallback.
"""

import os as _os

# Large, long-lived HBM residents (keys, resident masks) next to a churning
# working set fragment the caching allocator's fixed segments; expandable
# segments avoid that (read when CUDA first allocates, so set it early).
_os.environ.setdefault("PYTORCH_CUDA_ALLOC_CONF", "expandable_segments:True")

__version__ = "0.1.0"
