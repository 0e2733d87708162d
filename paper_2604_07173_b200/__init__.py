"""B200-native multi-LoRA delta hot path of InfiniLoRA (arxiv 2604.07173).

The product is the C-ABI library ``liblora_server.so`` (include/lora_server.h,
kernels in csrc/); ``binding`` is its thin ctypes binding and ``server`` a
small convenience wrapper over torch tensors.  Importing the binding without
the built library raises -- there is no CPU fallback.
"""
__all__ = ["binding", "server"]
