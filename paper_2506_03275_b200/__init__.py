"""B200-native Chipmunk column-sparse-delta hot path (sm_100a).

The compute lives in ``libcsd_b200.so`` (hand-written CUDA, C ABI in
``include/csd_b200.h``); ``ops`` mirrors the reference's ``csd::`` operator API
over it.  Importing ``ops`` loads the library and fails loudly if it is absent.
"""
__all__ = ["ops", "errors", "build", "generation"]
