"""Bitshift trellis: edge rule, windows, logical pack/unpack.  (oracle; test infrastructure only)

Paper passages:
  P:121-123  (L,k,V) trellis: 2^L nodes, 2^{kV} in/out edges, walk of T/V nodes.
  P:208-210  bitshift edge rule  j = (i 2^{kV} mod 2^L) + c ; group t reads bit
             positions (t-1)kV+1 ... (t-1)kV+L (1-indexed).
  P:203      Fig. 2: L=2,k=1,V=1, walk stored as 0010110; tail-biting drops the
             last L-kV bits -> 001011.
  P:325-328  tail-biting: start and end state share L-kV bits, kT bits per sequence.

Readings: the logical stream is MSB-first (bit 0 of the stream is
the most significant bit of the first state, Fig. 2 read left to right), and a
window that runs past bit kT-1 of a tail-biting stream wraps to bit 0.
Bits are represented as numpy uint8 arrays of 0/1 -- deliberately plain.
"""
import numpy as np


def next_states(i, L, k, V):
    """All successors of node i: {(i * 2^{kV} mod 2^L) + c : 0 <= c < 2^{kV}}."""
    kv = k * V
    return [((i * (1 << kv)) % (1 << L)) + c for c in range(1 << kv)]


def is_edge(i, j, L, k, V):
    """the top L-kV bits of j equal the bottom L-kV bits of i."""
    kv = k * V
    return (j >> kv) == (i % (1 << (L - kv)))


def is_walk(states, L, k, V, tail_biting=False):
    ok = all(is_edge(states[t], states[t + 1], L, k, V) for t in range(len(states) - 1))
    if tail_biting and len(states) > 0:
        ok = ok and is_edge(states[-1], states[0], L, k, V)
    return ok


def int_to_bits(v, width):
    """MSB-first bit list of an unsigned integer."""
    return [(v >> (width - 1 - i)) & 1 for i in range(width)]


def bits_to_int(bits):
    v = 0
    for b in bits:
        v = (v << 1) | int(b)
    return v


def pack(states, L, k, V, tail_biting):
    """Walk -> stored bit string (Fig. 2).

    The first state's L bits, then the kV new (low) bits of each later state.
    Tail-biting drops the final L-kV bits (they repeat the first state's top bits).
    """
    kv = k * V
    if not is_walk(states, L, k, V, tail_biting):
        raise ValueError("not a valid (tail-biting) walk")
    bits = int_to_bits(states[0], L)
    for s in states[1:]:
        bits += int_to_bits(s % (1 << kv), kv)
    if tail_biting:
        drop = L - kv
        bits = bits[: len(bits) - drop] if drop else bits
    return np.array(bits, dtype=np.uint8)


def window(bits, t, L, k, V, tail_biting):
    """State of group t (0-indexed): the L-bit window starting at bit t*kV,
    indices taken mod len(bits) when tail-biting."""
    n = len(bits)
    start = t * k * V
    if tail_biting:
        idx = [(start + i) % n for i in range(L)]
    else:
        idx = [start + i for i in range(L)]
    return bits_to_int([bits[i] for i in idx])


def unpack(bits, L, k, V, n_groups, tail_biting):
    """Stored bits -> walk: one window per group."""
    return [window(bits, t, L, k, V, tail_biting) for t in range(n_groups)]


def bits_from_bytes(byte_arr, nbits=None):
    """Byte buffer -> MSB-first bit array (bit 0 = MSB of byte 0)."""
    b = np.unpackbits(np.asarray(byte_arr, dtype=np.uint8), bitorder="big")
    return b if nbits is None else b[:nbits]


def bytes_from_bits(bits):
    return np.packbits(np.asarray(bits, dtype=np.uint8), bitorder="big")


def tile_states(tile_bytes, L, k, V, T):
    """All T/V states of one tail-biting tile stream (kT bits = 32k bytes for T=256),
    vectorised over tiles: tile_bytes has shape (..., kT/8); returns int64 (..., T/V).

    Same definition as `window` (bits [t kV, t kV + L) mod kT, MSB-first), written
    with array indexing so whole matrices can be decoded in seconds."""
    tile_bytes = np.asarray(tile_bytes, dtype=np.uint8)
    nbits = k * T
    bits = np.unpackbits(tile_bytes, axis=-1, bitorder="big")[..., :nbits].astype(np.int64)
    kv = k * V
    n_groups = T // V
    out = np.zeros(bits.shape[:-1] + (n_groups,), dtype=np.int64)
    for i in range(L):
        pos = (np.arange(n_groups) * kv + i) % nbits
        out = (out << 1) | bits[..., pos]
    return out
