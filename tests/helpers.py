import base64
import hashlib

import numpy as np


def sha(b: bytes) -> str:
    return hashlib.sha256(bytes(b)).hexdigest()


def sha_samples(a) -> str:
    return sha(np.ascontiguousarray(a, dtype="<i8").tobytes())


def b64d(s: str) -> bytes:
    return base64.b64decode(s)
