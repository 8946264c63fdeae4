"""Property-based checks of the host rules against the reference itself
(oracle/_ref, compiled from its sources) and the oracle restatement, over
random and extreme arguments: the planner (chunk.cpp:27-81), pad/unpad
(chunk.cpp:83-100), the sweep generator (bench.cpp:109-125) and the key
schedule (aes.cpp:151-180).  CPU only; no compute kernels are called."""
import pytest
from hypothesis import HealthCheck, given, settings
from hypothesis import strategies as st

SETTINGS = settings(max_examples=300, deadline=None, suppress_health_check=[HealthCheck.function_scoped_fixture])

lengths = st.one_of(st.integers(0, 5000), st.integers(0, 1 << 40), st.sampled_from([0, 15, 16, 17, (1 << 36), (1 << 36) + 7]))
workers = st.one_of(st.integers(1, 40), st.sampled_from([1, 2, 4, 8, 64, 1000]))


def _ours(paes, direction, n, w):
    fn = paes.plan_chunks if direction == 0 else paes.plan_decrypt_chunks
    try:
        return [(c["offset"], c["raw_len"], c["padded_len"], c["is_final"]) for c in fn(n, w)]
    except paes.PaddingError:
        return "PaddingError"
    except ValueError:
        return "ValueError"


def _theirs(ref, direction, n, w):
    r = ref.plan(direction, n, w)
    if r == -74:
        return "PaddingError"
    if r == -22:
        return "ValueError"
    return r


@SETTINGS
@given(n=lengths, w=workers)
def test_plan_chunks_equals_reference(paes, ref, n, w):
    assert _ours(paes, 0, n, w) == _theirs(ref, 0, n, w)


@SETTINGS
@given(n=lengths, w=workers)
def test_plan_decrypt_chunks_equals_reference(paes, ref, n, w):
    assert _ours(paes, 1, n, w) == _theirs(ref, 1, n, w)


@SETTINGS
@given(n=lengths, w=workers)
def test_plan_invariants(paes, n, w):
    """Contiguous, disjoint, covering; only the last chunk is final; non-final
    chunks are whole blocks; output length is the always-pad length."""
    plan = paes.plan_chunks(n, w)
    assert 1 <= len(plan) <= w
    pos = 0
    for i, c in enumerate(plan):
        assert c["offset"] == pos
        assert c["is_final"] == (i == len(plan) - 1)
        if not c["is_final"]:
            assert c["raw_len"] % 16 == 0 and c["padded_len"] == c["raw_len"]
        pos += c["raw_len"]
    assert pos == n
    assert sum(c["padded_len"] for c in plan) == (n // 16 + 1) * 16


@SETTINGS
@given(data=st.binary(max_size=200))
def test_pad_unpad_round_trip(paes, orc, data):
    padded = paes.pkcs7_pad(data)
    k = 16 - len(data) % 16
    assert padded == data + bytes([k]) * k
    assert paes.pkcs7_unpad(padded) == data
    assert orc.unpad(padded) == len(data)


@SETTINGS
@given(body=st.binary(min_size=0, max_size=64), tail=st.binary(min_size=16, max_size=16))
def test_unpad_agrees_with_oracle_on_arbitrary_trailers(paes, orc, body, tail):
    blob = body[: len(body) - len(body) % 16] + tail
    want = orc.unpad(blob)
    if want < 0:
        with pytest.raises(paes.PaddingError):
            paes.pkcs7_unpad(blob)
    else:
        assert paes.pkcs7_unpad(blob) == blob[:want]


@settings(max_examples=60, deadline=None, suppress_health_check=[HealthCheck.function_scoped_fixture])
@given(seed=st.integers(0, (1 << 32) - 1), size=st.integers(0, 3000))
def test_sweep_generator_equals_reference(paes, ref, seed, size):
    assert paes.sweep(seed, size) == ref.sweep(seed, size)


@SETTINGS
@given(key=st.binary(min_size=16, max_size=16))
def test_key_schedule_equals_reference(paes, ref, key):
    assert paes.round_keys(key) == ref.expand_key(key)
