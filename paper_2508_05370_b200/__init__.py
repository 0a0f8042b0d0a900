"""B200-native batched evaluator of the heterogeneity-aware LLM-training
simulator of arXiv 2508.05370.

Public surface: :class:`Sim` (``hsim_create`` / ``eval_batch`` / ``topk`` /
``decode``) over the C ABI in include/hsim.h, and :func:`sweep` (multi-GPU
top-k over torch.distributed).
"""
from .hsim import (Sim, HsimError, hsim_create, hsim_destroy, hsim_space_size, hsim_decode,  # noqa: F401
                   hsim_eval_batch, hsim_topk, descriptors, lib, EXPORTS, LIB_PATH)
