"""Host-side tokenization and cross-tokenizer span alignment.

Same contract as pkg/src/cacheclip/tokenizers.py: greedy longest match with
character offsets (tokenizers.py:38-95) and character-overlap projection of
aux-token indices onto primary tokens (tokenizers.py:151-177). This is O(chars)
host work outside the device path; when both models share one tokenizer the
projection is the identity and the pipeline short-circuits it.
"""

from __future__ import annotations

from dataclasses import dataclass
from typing import Iterable, Sequence

import numpy as np

from .errors import SpanCoverageError, UnknownCharacterError, VocabFormatError


@dataclass(frozen=True)
class TokenSpan:
    token_id: int
    start: int
    end: int  # exclusive


class GreedyTokenizer:
    """Longest-match tokenizer; entries bucketed by length for the scan."""

    def __init__(self, vocab: Sequence[str], tokenizer_id: str = "") -> None:
        if not vocab:
            raise VocabFormatError("empty vocabulary")
        table: dict[str, int] = {}
        for i, tok in enumerate(vocab):
            if not tok:
                raise VocabFormatError(f"empty token at index {i}")
            if "\n" in tok:
                raise VocabFormatError(f"token at index {i} contains a newline")
            if tok in table:
                raise VocabFormatError(f"duplicate token {tok!r} at index {i}")
            table[tok] = i
        self._vocab = list(vocab)
        self._table = table
        self._lengths = sorted({len(t) for t in vocab}, reverse=True)
        self.tokenizer_id = tokenizer_id
        self._digest: str | None = None
        self._canonical: set[bytes] = set()  # id sequences (int64 bytes) known to re-encode to themselves

    @property
    def vocab_digest(self) -> str:
        """SHA-256 of the vocabulary contents (two tokenizers with equal
        digests tokenize every text identically)."""
        if self._digest is None:
            import hashlib
            h = hashlib.sha256()
            for tok in self._vocab:
                h.update(tok.encode("utf-8", "surrogatepass"))
                h.update(b"\n")  # tokens never contain a newline
            self._digest = h.hexdigest()
        return self._digest

    def is_canonical(self, ids: Sequence[int], key: bytes | None = None) -> bool:
        """True when decode(ids) re-encodes to exactly ids (memoised: a
        cached chunk's ids are checked once per tokenizer, not per request).
        ``key``: the ids as int64 bytes when the caller has them
        (``ChunkCache.chunk_key``), so a repeat check is one hash lookup."""
        if key is None:
            key = np.asarray([int(i) for i in ids], dtype=np.int64).tobytes()
        if key in self._canonical:
            return True
        seq = [int(i) for i in ids]
        ok = self.encode(self.decode(seq)) == seq
        if ok:
            self._canonical.add(key)
        return ok

    @property
    def vocab_size(self) -> int:
        return len(self._vocab)

    @property
    def vocab(self) -> list[str]:
        return list(self._vocab)

    def token(self, token_id: int) -> str:
        if not 0 <= token_id < len(self._vocab):
            raise ValueError(f"token id {token_id} out of range")
        return self._vocab[token_id]

    def encode_with_offsets(self, text: str) -> list[TokenSpan]:
        out: list[TokenSpan] = []
        pos, n = 0, len(text)
        table = self._table
        while pos < n:
            for ln in self._lengths:
                if pos + ln > n:
                    continue
                tid = table.get(text[pos:pos + ln])
                if tid is not None:
                    out.append(TokenSpan(tid, pos, pos + ln))
                    pos += ln
                    break
            else:
                raise UnknownCharacterError(f"no vocab entry matches at offset {pos}: {text[pos]!r}")
        return out

    def encode(self, text: str) -> list[int]:
        return [s.token_id for s in self.encode_with_offsets(text)]

    def decode(self, ids: Iterable[int]) -> str:
        return "".join(self.token(int(i)) for i in ids)


@dataclass(frozen=True)
class AlignmentMap:
    images: tuple[tuple[int, ...], ...]

    def image(self, src_index: int) -> tuple[int, ...]:
        return self.images[src_index]

    def project(self, src_indices: Iterable[int]) -> list[int]:
        out: set[int] = set()
        for i in src_indices:
            out.update(self.images[i])
        return sorted(out)


def _tiled_length(spans: Sequence[TokenSpan], label: str) -> int:
    cursor = 0
    for s in spans:
        if s.start != cursor or s.end <= s.start:
            raise SpanCoverageError(f"{label} spans do not tile the text at offset {cursor}")
        cursor = s.end
    return cursor


def align_spans(src: Sequence[TokenSpan], dst: Sequence[TokenSpan]) -> AlignmentMap:
    """Source token -> every destination token whose interval it overlaps."""
    a, b = _tiled_length(src, "source"), _tiled_length(dst, "destination")
    if a != b:
        raise SpanCoverageError(f"covered lengths differ: source {a}, destination {b}")
    images: list[tuple[int, ...]] = []
    j = 0
    for s in src:
        while j < len(dst) and dst[j].end <= s.start:
            j += 1
        t = j
        hit: list[int] = []
        while t < len(dst) and dst[t].start < s.end:
            hit.append(t)
            t += 1
        images.append(tuple(hit))
    return AlignmentMap(tuple(images))


def char_vocab(size: int, base: int = 0x4E00) -> list[str]:
    """`size` distinct single characters: greedy matching is the identity, so
    arbitrary id sequences round-trip through text (synthetic workloads).
    Code points skip the UTF-16 surrogate block."""
    out = []
    cp = base
    while len(out) < size:
        if 0xD800 <= cp <= 0xDFFF:
            cp = 0xE000
        out.append(chr(cp))
        cp += 1
    return out
