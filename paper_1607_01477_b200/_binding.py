"""ctypes binding for libmstrsm.so (filled in with the CUDA library)."""


def load():
    raise RuntimeError("libmstrsm.so not built yet")
