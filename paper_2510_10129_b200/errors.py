"""Exception hierarchy of the reference, kept so callers' except-clauses work
unchanged (tensor_core.py:18, kv_store.py:36-52, model.py:43-56,
tokenizers.py:19-28). Everything is a ValueError subclass."""


class DimensionError(ValueError):
    """Operand shapes cannot be attended over / unsupported by the kernels."""


class CacheFormatError(ValueError):
    pass


class BadMagicError(CacheFormatError):
    pass


class VersionMismatchError(CacheFormatError):
    pass


class ChecksumError(CacheFormatError):
    pass


class CacheConsistencyError(ValueError):
    """Caches that cannot be merged or extended together."""


class WeightFormatError(ValueError):
    pass


class ManifestVersionError(WeightFormatError):
    pass


class MissingTensorError(WeightFormatError):
    pass


class TensorShapeError(WeightFormatError):
    pass


class UnknownCharacterError(ValueError):
    pass


class VocabFormatError(ValueError):
    pass


class SpanCoverageError(ValueError):
    pass
