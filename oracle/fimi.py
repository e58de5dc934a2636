"""oracle/fimi.py -- TEST INFRASTRUCTURE ONLY (see oracle/__init__.py for who may import it).

Plain-Python reference for the NEXT-3 row: reading a FIMI-repository
transaction file ("taken from the Frequent Itemset Mining Dataset Repository")
into the vertical layout the method starts from (for each item the set S_i of
transactions containing it), and the frequent-item pre-filter the paper assumes
("we have preprocessed the data set to remove items with support below the
threshold").  Character-by-character, one line at a time, no blocking or reordering;
shares no code with the CUDA path (paper_1102_1003_b200/csrc/ingest.cu).

Semantics (readings in DESIGN.md §3, #21-#25):
  * a line is one transaction; transaction ids are 0-based line indices (reading #2);
  * tokens are runs of decimal digits separated by spaces, tabs or '\\r'; any other byte
    is a parse error reported with its 1-based line number; a token > 2^32 - 1 is
    an error too;
  * duplicate items within a line are collapsed (set semantics);
  * blank lines are empty transactions; the text after the last '\\n' is a
    transaction iff it is non-empty, so m = #'\\n' + (1 if the text does not end in '\\n');
  * item labels are re-densified in ascending label order; the map dense -> label is kept.
"""
from __future__ import annotations

import numpy as np

_WS = (ord(" "), ord("\t"), ord("\r"))


class FimiParseError(ValueError):
    def __init__(self, line: int, msg: str):
        super().__init__(f"line {line}: {msg}")
        self.line = line


def parse_fimi(text: bytes):
    """FIMI text -> (offsets int64[n+1], tids int32[nnz], labels uint32[n], m)."""
    transactions: list[set[int]] = []
    cur: set[int] = set()
    tok = None  # value of the token being read
    line = 1
    for byte in text:
        if 48 <= byte <= 57:  # digit
            tok = (0 if tok is None else tok) * 10 + (byte - 48)
            if tok > 0xFFFFFFFF:
                raise FimiParseError(line, "item id exceeds 2^32 - 1")
            continue
        if tok is not None:
            cur.add(tok)
            tok = None
        if byte == 10:  # '\n' ends the transaction
            transactions.append(cur)
            cur = set()
            line += 1
        elif byte not in _WS:
            raise FimiParseError(line, f"invalid byte 0x{byte:02X}")
    if tok is not None:
        cur.add(tok)
    if len(text) and text[-1] != 10:
        transactions.append(cur)
    m = len(transactions)
    labels = sorted(set().union(*transactions)) if transactions else []
    dense = {lab: k for k, lab in enumerate(labels)}
    lists: list[list[int]] = [[] for _ in labels]
    for t, items in enumerate(transactions):  # ascending t => every S_i comes out sorted
        for lab in items:
            lists[dense[lab]].append(t)
    offsets = np.zeros(len(labels) + 1, np.int64)
    offsets[1:] = np.cumsum([len(s) for s in lists])
    tids = np.array([t for s in lists for t in s], dtype=np.int32)
    return offsets, tids, np.array(labels, dtype=np.uint32), m


def frequent_items(offsets: np.ndarray, min_support: int) -> np.ndarray:
    """Items whose support |S_i| (a singleton's support) is at least min_support,
    ascending.  min_support 0 keeps every item."""
    sizes = np.diff(np.asarray(offsets, dtype=np.int64))
    return np.array([i for i, s in enumerate(sizes.tolist()) if s >= min_support], dtype=np.int32)


def filter_csr(offsets: np.ndarray, tids: np.ndarray, items: np.ndarray):
    """The vertical database restricted to `items` (kept in the given order)."""
    rows = [tids[offsets[i]:offsets[i + 1]] for i in items.tolist()]
    off = np.zeros(len(rows) + 1, np.int64)
    off[1:] = np.cumsum([len(r) for r in rows])
    return off, (np.concatenate(rows).astype(np.int32) if rows else np.zeros(0, np.int32))
