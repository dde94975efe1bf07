"""Rank AUROC used to show ranking parity (restates reference metrics.py:44-59;
test helper, not product)."""

import numpy as np


def auroc(scores, mask):
    s = np.asarray(scores, np.float64).ravel()
    labels = np.asarray(mask, bool).ravel()
    pos = int(labels.sum())
    neg = labels.size - pos
    order = np.argsort(s, kind="stable")
    ss = s[order]
    ranks = np.empty(ss.size, np.float64)
    starts = np.flatnonzero(np.r_[True, ss[1:] != ss[:-1]])
    ends = np.r_[starts[1:], ss.size]
    avg = (starts + ends - 1) / 2.0 + 1.0
    ranks[order] = np.repeat(avg, ends - starts)
    return float((ranks[labels].sum() - pos * (pos + 1) / 2) / (pos * neg))
