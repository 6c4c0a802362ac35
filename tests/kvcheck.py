"""Element-by-element checks of a K/V cache after one window step (shared by the GPU parity tests).

The north star's bar for the KV refresh: pure copies bit-exact (V reuse; refreshed rows of ANCHOR / NEW /
prompt tokens), rotated keys (Eq. 5) within 1e-2 abs (bf16) / 1e-5 (fp32).  These
helpers split every element of the cache into exactly those classes, using the oracle's dispositions and slot map:

  * REUSE key rows, rotated columns          -> tolerance (and the count of non-bit-exact elements);
  * REUSE key rows, columns Eq. 5 leaves     -> bits (M-RoPE h / w sections, reading NEXT-3);
  * V rows of REUSE tokens                   -> bits (paged: untouched; copy mode: copied from the old cache);
  * K and V rows of every non-REUSE token    -> bits, and equal to row r of the recompute buffer (the r-th non-REUSE
                                                token in p_new order, reading Q18), checked against the buffer itself;
  * every row no token of the window wrote   -> bits, equal to its content before the step.

Nothing here computes a rotation: the expected values are the oracle's pool and the step's own inputs.
"""
import numpy as np

DISP_REUSE = 2


def _bits(a):
    a = np.ascontiguousarray(a)
    return a.view(np.uint16) if a.dtype == np.uint16 else a.view(np.uint32)


def rot_cols(kv):
    """(rotated, kept) column indices of a key row [H][D] under kv's RoPE: with M-RoPE only the temporal pairs
    (i, i + D/2), i < s_t, are rotated; the h / w sections keep their bits (reading NEXT-3)."""
    D = kv["head_dim"]
    st = kv["mrope_section"][0] if kv.get("rope_mode", 0) == 1 else D // 2
    rot = np.array([i for i in range(D) if (i % (D // 2)) < st], dtype=np.int64)
    keep = np.array([i for i in range(D) if (i % (D // 2)) >= st], dtype=np.int64)
    return rot, keep


def _rotated_stats(ka, kb, kv, stats, tag):
    if kv["dtype"] == 0:
        fa = (ka.astype(np.uint32) << 16).view(np.float32)
        fb = (kb.astype(np.uint32) << 16).view(np.float32)
        tol = 1e-2
    else:
        fa, fb, tol = ka, kb, 1e-5
    d = float(np.abs(fa.astype(np.float64) - fb).max()) if fa.size else 0.0
    assert d <= tol, (tag, d)
    if stats is not None:
        stats["max_diff"] = max(stats.get("max_diff", 0.0), d)
        stats["not_bit_exact"] = stats.get("not_bit_exact", 0) + int((_bits(ka) != _bits(kb)).sum())
        stats["rotated"] = stats.get("rotated", 0) + int(ka.size)


def refreshed_rows(disp, n_tok):
    """Row r of the recompute buffer for every token p < n_tok that is not REUSE (r counts them in p_new order)."""
    r = np.cumsum(disp[:n_tok] != DISP_REUSE) - 1
    return np.where(disp[:n_tok] != DISP_REUSE, r, -1)


def check_pool_step(got, pre, exp, disp, slots, n_tok, kv, refr=None, stats=None, tag=""):
    """Paged (in-place) step of one stream: pool `got` (GPU, after), `pre` (before), `exp` (oracle, after); the
    oracle's disposition / slot map of the window's first n_tok tokens; refr = the recompute buffer or None."""
    L, _, cap = got.shape[:3]
    rot, keep = rot_cols(kv)
    disp = disp[:n_tok]
    slots = slots[:n_tok]
    r_of = refreshed_rows(disp, n_tok)
    valid = (slots >= 0) & (slots < cap)
    reuse_rows = np.unique(slots[valid & (disp == DISP_REUSE)])
    ref_cap = kv["refresh_capacity"]
    wr = valid & (disp != DISP_REUSE) & (refr is not None) & (r_of < ref_cap)
    written = slots[wr]
    assert np.intersect1d(reuse_rows, written).size == 0, tag      # a row holds one token
    # 1. everything except the rotated columns of REUSE key rows: bit-identical to the oracle
    other = np.setdiff1d(np.arange(cap), reuse_rows)
    assert (_bits(got[:, 1]) == _bits(exp[:, 1])).all(), tag
    assert (_bits(got[:, 0, other]) == _bits(exp[:, 0, other])).all(), tag
    ga, ea = got[:, 0, reuse_rows], exp[:, 0, reuse_rows]
    assert (_bits(ga[..., keep]) == _bits(ea[..., keep])).all(), tag
    _rotated_stats(ga[..., rot], ea[..., rot], kv, stats, tag)
    # 2. rows nobody wrote this step: as before the step (values of REUSE tokens included: never touched)
    untouched = np.setdiff1d(np.arange(cap), written)
    assert (_bits(got[:, 1, untouched]) == _bits(pre[:, 1, untouched])).all(), tag
    still = np.setdiff1d(untouched, reuse_rows)
    assert (_bits(got[:, 0, still]) == _bits(pre[:, 0, still])).all(), tag
    if reuse_rows.size:
        assert (_bits(got[:, 0, reuse_rows][..., keep]) == _bits(pre[:, 0, reuse_rows][..., keep])).all(), tag
    # 3. refreshed rows (ANCHOR / NEW / prompt): bit copies of the recompute buffer's row r, K and V
    if written.size:
        assert (_bits(got[:, :, written]) == _bits(refr[:, :, r_of[wr]])).all(), tag
    if stats is not None:
        stats["bit_checked_rows"] = stats.get("bit_checked_rows", 0) + int(cap - reuse_rows.size)
        stats["refreshed_rows"] = stats.get("refreshed_rows", 0) + int(written.size)


def check_copy_step(got, pre, exp, disp, p_old, n_tok, kv, old=None, refr=None, stats=None, tag=""):
    """Out-of-place step of one stream: new cache `got` (GPU, after), `pre` (its content before), `exp` (oracle);
    rows p < n_tok are the window's tokens at p_new = p; old = the window-(k-1) cache (V reuse source)."""
    L, _, cap = got.shape[:3]
    rot, keep = rot_cols(kv)
    rows = min(n_tok, cap)
    disp = disp[:rows]
    re = np.flatnonzero(disp == DISP_REUSE)
    nonre = np.flatnonzero(disp != DISP_REUSE)
    # oracle, bit for bit, except the rotated key columns of REUSE rows
    assert (_bits(got[:, 1]) == _bits(exp[:, 1])).all(), tag
    assert (_bits(got[:, 0, nonre]) == _bits(exp[:, 0, nonre])).all(), tag
    assert (_bits(got[:, :, rows:]) == _bits(exp[:, :, rows:])).all(), tag
    assert (_bits(got[:, 0, re][..., keep]) == _bits(exp[:, 0, re][..., keep])).all(), tag
    _rotated_stats(got[:, 0, re][..., rot], exp[:, 0, re][..., rot], kv, stats, tag)
    # rows past the window's tokens: untouched
    assert (_bits(got[:, :, rows:]) == _bits(pre[:, :, rows:])).all(), tag
    # V reuse: bit copies of the old cache's row p_old, checked against the old cache itself
    if old is not None and re.size:
        po = p_old[:rows][re]
        ok = po < old.shape[2]
        assert (_bits(got[:, 1, re[ok]]) == _bits(old[:, 1, po[ok]])).all(), tag
    # refreshed rows: row r of the recompute buffer
    if refr is not None and nonre.size:
        r_of = refreshed_rows(disp, rows)[nonre]
        ok = r_of < kv["refresh_capacity"]
        assert (_bits(got[:, :, nonre[ok]]) == _bits(refr[:, :, r_of[ok]])).all(), tag
    if stats is not None:
        stats["bit_checked_rows"] = stats.get("bit_checked_rows", 0) + int(cap - re.size)


def assert_rotation_bits(stats, frac=1e-3):
    """Report the non-bit-exact rotated elements; the rotation is specified to the last bit (Q20), so more than a
    trace of them (cos / sin of the fp64 angle landing on an fp32 rounding boundary, DESIGN Q19-Q21 note) is a bug."""
    n, tot = stats.get("not_bit_exact", 0), stats.get("rotated", 0)
    print("rotated elements:", tot, "not bit-exact:", n, "max |diff|:", stats.get("max_diff", 0.0))
    assert n <= frac * max(tot, 1), (n, tot)
