"""B200-native (sm_100a) AttentionStore KV-reuse prefill path.

Host side: Python + PyTorch (device memory, streams, cuBLAS projections).
Hot path: hand-written CUDA in libaskv.so behind the C ABI of include/askv.h.

Modules
  rope      GPU mirror of kvsim.rope (KvRecord, rotate_matrix, attention_with_decoupled_cache)
  ops       torch wrappers over the C ABI
  model     ModelProfile / TierConfig mirror + LLaMA-2 shapes
  store     KvStore mirror with a pinned host block arena behind it
  overlap   Timeline + measured pre-load / save timelines
  runner    LLaMA-shaped prefill runner with layer-wise pre-load, re-embed, attention, save
  engine    multi-turn serving loop over the runner (reuse / recompute / HBM-resident)
"""

__version__ = "0.1.0"
