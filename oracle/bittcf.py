"""Reference BitTCF encoder / decoder and byte formulas (TEST INFRASTRUCTURE ONLY).

Format (§3.3): a sparse M x K matrix is cut into
RowWindows of 8 rows; each window's non-empty columns are condensed and cut
into 8x8 TC blocks ("we choose the shape of 8x8 tile in reality",
P:266 "we partition the sparse matrix A into 8x8 tiles").  Four arrays:

  1. RowWindowOffset  u32[ceil(M/8)+1]  offset of the first TC block of each window
  2. TCOffset         u32[NB+1]         offset of the first nnz of each TC block
  3. SparseAToB       u32[8*NB]         original column index of each condensed lane
  4. TCLocalBit       u64[NB]           1 = nnz at a local position of the block
  (+ values[nnz], ordered per block by ascending bit -- implied by P:273's popcount offset)

Readings where the paper is silent: bit k = r*8 + c, LSB = 0,
row-major, c = condensed lane (Q3); condensed columns ascending (Q4); padding
lanes store 0 (Q5); values by ascending bit (Q6); blocks may hold 1..64 nnz
(Q8); a ragged last window contributes no bits for missing rows (Q22).

Window height ``wh`` (reading R20; default 8 = the paper's format): the
same construction with windows of wh = 16 or 32 rows, i.e. wh x 8 tiles.  A block's
occupancy is wh/8 u64 words, word j covering tile rows 8j..8j+7 with the paper's bit rule
inside (bit (r mod 8)*8 + c); TCLocalBit holds the words block-major (NB*wh/8 entries);
values ascend by tile position p = r*8 + c, so a value's index is TCOffset[b] + the
popcount of the block's occupancy below p -- P:273 over the concatenated words.
"""
from __future__ import annotations

import numpy as np

WINDOW = 8  # P:250 "8 x 8 TC blocks", "ceil(M/8)+1 elements"


def encode(M: int, K: int, rowptr, colidx, vals=None, wh: int = WINDOW) -> dict:
    """Steps 1-7 of SURVEY §8(c) C-2 "BitTCF (independent Python encoder)", vectorised;
    ``wh`` = rows per window (8 = the paper's; 16 / 32 = reading R20)."""
    if wh not in (8, 16, 32):
        raise ValueError("window height must be 8, 16 or 32")
    nw = wh // WINDOW
    rowptr = np.asarray(rowptr, dtype=np.int64)
    colidx = np.asarray(colidx, dtype=np.int64)
    nnz = int(rowptr[-1]) if M > 0 else 0
    # 1. W = ceil(M/wh)
    W = (M + wh - 1) // wh
    # 2. window rows [wh*w, min(wh*w+wh, M)): window and local row of every nnz
    rows = np.repeat(np.arange(M, dtype=np.int64), np.diff(rowptr))
    w_of = rows // wh
    r_of = rows % wh
    # 3. U_w = sorted unique columns of the window's rows
    keys = w_of * np.int64(max(K, 1)) + colidx
    uniq, inverse = np.unique(keys, return_inverse=True)
    uw = uniq // np.int64(max(K, 1))
    ucol = uniq - uw * np.int64(max(K, 1))
    U = np.bincount(uw, minlength=W).astype(np.int64) if W > 0 else np.zeros(0, np.int64)
    ustart = np.zeros(W, dtype=np.int64)
    if W > 1:
        np.cumsum(U[:-1], out=ustart[1:])
    rank = np.arange(uniq.size, dtype=np.int64) - ustart[uw]
    # 4. blocks_w = ceil(|U_w|/8); block t owns U_w[8t:8t+8]; lanes beyond |U_w| pad with 0
    blocks = (U + WINDOW - 1) // WINDOW
    rwo = np.zeros(W + 1, dtype=np.int64)
    np.cumsum(blocks, out=rwo[1:])
    NB = int(rwo[-1])
    gblock = rwo[uw] + rank // WINDOW
    lane = rank % WINDOW
    a2b = np.zeros(WINDOW * NB, dtype=np.uint32)
    a2b[WINDOW * gblock + lane] = ucol.astype(np.uint32)
    # 5. tile position p = r*8 + lane of every nnz, in block gblock: word p // 64, bit p % 64
    nb_of = gblock[inverse]
    pos_of = r_of * WINDOW + lane[inverse]
    # 6. values of a block in ascending tile position
    order = np.lexsort((pos_of, nb_of))
    sb, sp = nb_of[order], pos_of[order]
    bits = np.zeros(NB * nw, dtype=np.uint64)
    counts = np.bincount(sb, minlength=NB).astype(np.int64) if NB > 0 else np.zeros(0, np.int64)
    tco = np.zeros(NB + 1, dtype=np.int64)
    np.cumsum(counts, out=tco[1:])
    if nnz > 0:
        onehot = np.left_shift(np.uint64(1), (sp % 64).astype(np.uint64))
        np.bitwise_or.at(bits, sb * nw + sp // 64, onehot)
    out = {
        "M": M, "K": K, "nnz": nnz, "W": W, "NB": NB, "wh": wh,
        "RowWindowOffset": rwo.astype(np.uint32),
        "TCOffset": tco.astype(np.uint32),       # 7. popcount prefix sums
        "SparseAToB": a2b,
        "TCLocalBit": bits,
        "U": U,                                   # |U_w| = valid lanes per window (bytes model)
    }
    if vals is not None:
        out["values"] = np.asarray(vals)[order]
    return out


def decode(fmt: dict):
    """Inverse of encode via P:273's popcount offset: idx(b,k) = TCOffset[b] + popc(mask & (2^k - 1)).

    Returns canonical CSR (rowptr int64, colidx int32, values or None)."""
    M, K = fmt["M"], fmt["K"]
    wh = fmt.get("wh", WINDOW)
    nw = wh // WINDOW
    rwo = fmt["RowWindowOffset"].astype(np.int64)
    tco = fmt["TCOffset"].astype(np.int64)
    a2b = fmt["SparseAToB"].astype(np.int64)
    words = fmt["TCLocalBit"].astype(np.uint64).reshape(-1, nw)   # [NB][wh/8]
    NB = words.shape[0]
    if np.any(tco[1:] - tco[:-1] != np.bitwise_count(words).sum(axis=1)):
        raise ValueError("BitTCF corruption: TCOffset step != popcount(TCLocalBit)")
    win_of_block = np.searchsorted(rwo, np.arange(NB), side="right") - 1
    ks = np.arange(64, dtype=np.uint64)
    # present[b, p] for tile positions p = 64*word + bit
    present = ((words[:, :, None] >> ks[None, None, :]) & np.uint64(1)).astype(bool).reshape(NB, 64 * nw)
    b_idx, p_idx = np.nonzero(present)
    # index = TCOffset[b] + occupancy of block b below position p
    before = np.cumsum(present, axis=1) - present
    vidx = tco[b_idx] + before[b_idx, p_idx].astype(np.int64)
    r = p_idx // WINDOW
    lane = p_idx % WINDOW
    row = win_of_block[b_idx] * wh + r
    col = a2b[WINDOW * b_idx + lane]
    if np.any(row >= M) or np.any(col >= K):
        raise ValueError("BitTCF corruption: position out of range")
    order = np.lexsort((col, row))
    row, col, vidx = row[order], col[order], vidx[order]
    rowptr = np.zeros(M + 1, dtype=np.int64)
    np.cumsum(np.bincount(row, minlength=M), out=rowptr[1:])
    vals = fmt["values"][vidx] if "values" in fmt else None
    return rowptr, col.astype(np.int32), vals


def value_index(mask: int, k: int, tco_b: int = 0) -> int:
    """P:273 decode of one position: TCOffset[b] + popc(mask & ((1<<k)-1))."""
    return tco_b + bin(mask & ((1 << k) - 1)).count("1")


# ----------------------------------------------------------------------- byte formulas

def bittcf_index_bytes(M: int, NB: int) -> int:
    """(ceil(M/8) + NumTCBlock*11 + 2) * 4 bytes (index structure only, Q7)."""
    return ((M + 7) // 8 + NB * 11 + 2) * 4


def metcf_index_bytes(M: int, NB: int, nnz: int) -> int:
    """ME-TCF skeleton with an int8 TCLocalId per nnz."""
    return ((M + 7) // 8 + 1 + NB + 1 + 8 * NB) * 4 + nnz


def csr_index_bytes(M: int, nnz: int) -> int:
    """CSR with 32-bit row pointers and column indices."""
    return (M + 1) * 4 + nnz * 4


def array_bytes(fmt: dict) -> int:
    """Sum of the four index arrays' sizes (must equal bittcf_index_bytes)."""
    return sum(int(fmt[k].nbytes) for k in ("RowWindowOffset", "TCOffset", "SparseAToB", "TCLocalBit"))


def mean_nnz_tc(fmt: dict) -> float:
    """MeanNNZTC = nnz / NB."""
    return fmt["nnz"] / fmt["NB"] if fmt["NB"] else 0.0


def permute_rows(M: int, rowptr, colidx, vals, perm_new2old):
    """Row relabelling A'[r] = A[perm[r]] (the reading of Q12: rows only, B untouched)."""
    rowptr = np.asarray(rowptr, dtype=np.int64)
    perm = np.asarray(perm_new2old, dtype=np.int64)
    lens = np.diff(rowptr)[perm]
    newptr = np.zeros(M + 1, dtype=np.int64)
    np.cumsum(lens, out=newptr[1:])
    total = int(newptr[-1]) if M else 0
    src = np.repeat(rowptr[perm] if M else np.zeros(0, np.int64), lens) \
        + (np.arange(total, dtype=np.int64) - np.repeat(newptr[:-1], lens))
    return newptr, np.asarray(colidx)[src], (np.asarray(vals)[src] if vals is not None else None)
