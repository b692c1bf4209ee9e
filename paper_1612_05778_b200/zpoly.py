"""The boundary type: dense integer polynomials as two's-complement limb arrays.

Same layout and semantics as the reference's IntPolynomial (tc/zpoly.py:32-100):
``words`` is a C-contiguous ``(d, ceil(bit_width/64))`` uint64 array, coefficient
i little-endian in row i, sign-extended across the row; equality compares
bit_width, shape and words.  Differences are internal only: construction-time
validation is vectorised over the limbs (the reference converts every
coefficient to a Python int, tc/zpoly.py:45-48), and products built by the
CUDA path use a trusted constructor.
"""

from __future__ import annotations

import numpy as np

from .errors import PolynomialParseError

WORD_BITS = 64
_WORD_MASK = (1 << WORD_BITS) - 1


def twos_complement_width(x: int) -> int:
    """Minimal two's-complement bit count for x, including the sign bit
    (tc/params.py:183-185)."""
    return x.bit_length() + 1 if x >= 0 else (-x - 1).bit_length() + 1


def _words_from_int(value: int, nwords: int) -> np.ndarray:
    enc = value & ((1 << (WORD_BITS * nwords)) - 1)
    return np.frombuffer(enc.to_bytes(8 * nwords, "little"), dtype=np.uint64).copy()


def _int_from_words(words: np.ndarray) -> int:
    u = int.from_bytes(words.tobytes(), "little")
    top = 1 << (WORD_BITS * len(words) - 1)
    return u - (top << 1) if u & top else u


def fits_width(words: np.ndarray, bit_width: int) -> np.ndarray:
    """Per-row: does the coefficient fit `bit_width` bits (two's complement)?

    Vectorised: the top limb must be the sign extension of bit bit_width-1."""
    r = (bit_width - 1) % WORD_BITS
    top = words[:, -1].view(np.int64) >> np.int64(r)
    return (top == 0) | (top == -1)


def row_widths(words: np.ndarray) -> np.ndarray:
    """Two's-complement width of every coefficient (numpy, host side)."""
    d, cw = words.shape
    sign = np.where((words[:, -1] >> np.uint64(63)).astype(bool), np.uint64(_WORD_MASK), np.uint64(0))
    x = words ^ sign[:, None]
    nz = x != 0
    any_nz = nz.any(axis=1)
    top = cw - 1 - np.argmax(nz[:, ::-1], axis=1)
    topw = x[np.arange(d), top]
    bl = np.zeros(d, dtype=np.int64)
    v = topw.copy()
    for s in (32, 16, 8, 4, 2, 1):
        m = v >= (np.uint64(1) << np.uint64(s))
        bl += np.where(m, s, 0)
        v = np.where(m, v >> np.uint64(s), v)
    bl += (v > 0).astype(np.int64)
    return np.where(any_nz, 64 * top + bl + 1, 1)


class IntPolynomial:
    """Dense polynomial over Z; index = degree, ascending (tc/zpoly.py:32)."""

    __slots__ = ("bit_width", "words")

    def __init__(self, words: np.ndarray, bit_width: int):
        if words.ndim != 2 or words.dtype != np.uint64 or words.shape[0] < 1:
            raise ValueError("words must be a (d, coeff_words) uint64 array")
        if bit_width < 1 or words.shape[1] != -(-bit_width // WORD_BITS):
            raise ValueError("coeff_words does not match the declared bit width")
        self.bit_width = int(bit_width)
        self.words = np.ascontiguousarray(words)
        ok = fits_width(self.words, self.bit_width)
        if not ok.all():
            i = int(np.argmin(ok))
            raise ValueError(f"coefficient {i} does not fit {bit_width} bits")

    @classmethod
    def _trusted(cls, words: np.ndarray, bit_width: int) -> "IntPolynomial":
        """Wrap words produced by the device path (already exact and in range)."""
        obj = cls.__new__(cls)
        obj.words = words
        obj.bit_width = int(bit_width)
        return obj

    @classmethod
    def from_coefficients(cls, coeffs, bit_width: int | None = None) -> "IntPolynomial":
        coeffs = [int(c) for c in coeffs]
        if not coeffs:
            raise ValueError("a polynomial needs at least one coefficient")
        if bit_width is None:
            bit_width = max(twos_complement_width(c) for c in coeffs)
        nwords = -(-bit_width // WORD_BITS)
        words = np.empty((len(coeffs), nwords), dtype=np.uint64)
        for i, c in enumerate(coeffs):
            words[i] = _words_from_int(c, nwords)
        return cls(words, bit_width)

    @property
    def degree_plus_one(self) -> int:
        return self.words.shape[0]

    @property
    def coeff_words(self) -> int:
        return self.words.shape[1]

    def coefficient(self, i: int) -> int:
        return _int_from_words(self.words[i])

    def coefficients(self) -> list:
        return [self.coefficient(i) for i in range(self.degree_plus_one)]

    def is_zero(self) -> bool:
        return not self.words.any()

    def min_coefficient(self) -> int:
        return min(self.coefficients())

    def max_coefficient(self) -> int:
        return max(self.coefficients())

    def max_width(self) -> int:
        """max over coefficients of twos_complement_width (vectorised)."""
        return int(row_widths(self.words).max())

    def __eq__(self, other) -> bool:
        if not isinstance(other, IntPolynomial):
            return NotImplemented
        return (self.bit_width == other.bit_width
                and self.words.shape == other.words.shape
                and bool(np.array_equal(self.words, other.words)))

    def __hash__(self):
        return hash((self.bit_width, self.words.tobytes()))

    def __repr__(self):
        return f"IntPolynomial(d={self.degree_plus_one}, bits={self.bit_width})"


def output_bit_width(d: int, n_in: int) -> int:
    """Width of the product from the tight bound |c_i| <= d 2^(2 n_in - 2)."""
    return d.bit_length() + max(2 * n_in - 2, 0) + 1      # bit_length(d << (2 n_in - 2)) + 1


def product_bit_width(a: IntPolynomial, b: IntPolynomial) -> int:
    """tc/zpoly.py:103-114, with the width scan vectorised."""
    n_in = max(a.max_width(), b.max_width())
    return output_bit_width(max(a.degree_plus_one, b.degree_plus_one), n_in)


def parse_polynomial(text) -> IntPolynomial:
    """The reference's text format (tc/zpoly.py:117-142): ``d=<count>`` then one
    signed decimal coefficient per line."""
    if isinstance(text, bytes):
        text = text.decode("ascii")
    lines = text.splitlines()
    if not lines or not lines[0].startswith("d="):
        raise PolynomialParseError("expected header 'd=<count>'", line=1)
    try:
        d = int(lines[0][2:])
    except ValueError:
        raise PolynomialParseError("malformed degree count", line=1) from None
    if d < 1:
        raise PolynomialParseError("degree count must be positive", line=1)
    body = lines[1:]
    if len(body) < d:
        raise PolynomialParseError(f"expected {d} coefficient lines, found {len(body)}")
    if any(s.strip() for s in body[d:]):
        raise PolynomialParseError("trailing data after last coefficient", line=d + 2)
    coeffs = []
    for idx, raw in enumerate(body[:d]):
        try:
            coeffs.append(int(raw.strip()))
        except ValueError:
            raise PolynomialParseError(f"not an integer: {raw.strip()!r}", line=idx + 2) from None
    return IntPolynomial.from_coefficients(coeffs)


def format_polynomial(poly: IntPolynomial) -> str:
    return "\n".join([f"d={poly.degree_plus_one}"] + [str(c) for c in poly.coefficients()]) + "\n"
