"""Pins for the oracle's step segmentation (a1): PAPER.md:119."""
import itertools
import json
import os

import numpy as np
import pytest

import oracle
from synth import traces

GOLD = os.path.join(os.path.dirname(__file__), "golden")
DELIM = 1


def seg1(tokens, final=1, gen_start=0, delims=(DELIM,)):
    t = np.asarray(tokens, np.int32)
    r = oracle.segment_steps(t, [0, t.size], [gen_start], [final], list(delims))
    return [[int(a), int(b)] for a, b in zip(r["step_start"], r["step_end"])], r


@pytest.mark.parametrize("ex", json.load(open(os.path.join(GOLD, "spec_examples.json")))["segment"],
                         ids=lambda e: e["cite"][:40])
def test_spec_worked_examples(ex):
    steps, _ = seg1(ex["tokens"], ex["final"])
    assert steps == ex["steps"], ex["cite"]


def test_tiny_t0_golden():
    g = json.load(open(os.path.join(GOLD, "tiny_t0.json")))
    b = traces.tiny_t0()
    r = oracle.segment_steps(b.tokens, b.seq_tok_off, b.gen_start, b.final, b.delim_ids)
    assert r["step_start"].tolist() == g["step_start"]
    assert r["step_end"].tolist() == g["step_end"]
    assert r["step_nbag"].tolist() == g["step_nbag"]
    assert r["seq_step_off"].tolist() == [0, 8]


def test_prompt_never_a_step_and_leading_delims_form_void_step():
    # prompt [5, D, 6] (gen_start 3) then D D a D b
    steps, r = seg1([5, DELIM, 6, DELIM, DELIM, 7, DELIM, 8], final=1, gen_start=3)
    assert steps == [[3, 5], [5, 7], [7, 8]]
    assert r["step_nbag"].tolist() == [0, 1, 1]      # first step is void (reading R5)


def test_multiple_delimiter_ids_and_empty_sequence():
    t = np.asarray([10, 1, 2, 11, 2, 12], np.int32)
    r = oracle.segment_steps(np.concatenate([t, t]), [0, 0, 6, 12], [0, 0, 0], [1, 1, 0], [1, 2])
    assert r["seq_step_off"].tolist() == [0, 0, 3, 5]
    assert list(zip(r["step_start"], r["step_end"])) == [(0, 3), (3, 5), (5, 6), (0, 3), (3, 5)]


def _brute_segment(tokens, gen_start, final, delims):
    """Independent construction: group the generated tokens into maximal runs of
    (delimiter / non-delimiter) and glue each delimiter run onto the step it closes."""
    gen = list(tokens[gen_start:])
    runs, pos = [], gen_start
    for isd, grp in itertools.groupby(gen, key=lambda x: x in delims):
        n = len(list(grp))
        runs.append((isd, pos, pos + n))
        pos += n
    steps, cur = [], None
    for idx, (isd, a, b) in enumerate(runs):
        if cur is None:
            cur = a
        if isd:
            last = idx == len(runs) - 1
            if not last or final:
                steps.append((cur, b))
                cur = None
    if cur is not None and final:
        steps.append((cur, len(tokens)))
    return steps


@pytest.mark.parametrize("seed", range(30))
def test_brute_force_random(seed):
    rng = np.random.default_rng(seed)
    n = int(rng.integers(0, 60))
    delims = [1, 2]
    toks = rng.choice([1, 2, 3, 4, 5, 6], size=n, p=[0.2, 0.1, 0.2, 0.2, 0.2, 0.1]).astype(np.int32)
    gs = int(rng.integers(0, n + 1))
    fin = int(rng.integers(0, 2))
    got, r = seg1(toks, fin, gs, delims)
    exp = _brute_segment(toks.tolist(), gs, fin, set(delims))
    assert [tuple(x) for x in got] == exp
    for (a, b), nb in zip(got, r["step_nbag"]):
        assert nb == sum(1 for x in toks[a:b] if x not in delims)


def test_steps_tile_generated_region_of_synthetic_trace():
    b = traces.make_batch(7, 3, 3000, 128, 16)
    r = oracle.segment_steps(b.tokens, b.seq_tok_off, b.gen_start, b.final, b.delim_ids)
    for s in range(3):
        lo, hi = r["seq_step_off"][s], r["seq_step_off"][s + 1]
        st, en = r["step_start"][lo:hi], r["step_end"][lo:hi]
        assert st[0] == 128 and en[-1] == 3000            # final sequence: tiles [gen_start, n)
        assert np.all(st[1:] == en[:-1])
        # every ground-truth step start of the generator is a segment start
        assert set(b.step_starts[s].tolist()) <= set(st.tolist())
