"""Shared helpers for the test-suite."""
import functools


@functools.lru_cache(None)
def has_gpu() -> bool:
    try:
        import torch
        return torch.cuda.is_available()
    except Exception:
        return False
