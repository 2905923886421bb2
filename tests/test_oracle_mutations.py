"""Every one-line misreading listed in tools/mutate_oracle.py must fail an oracle pin
("every pin fails under a deliberate one-line mutation of the oracle")."""
import os
import sys

sys.path.insert(0, os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))), "tools"))


def test_every_oracle_mutation_is_killed():
    import mutate_oracle as M
    res = M.run_all(jobs=min(12, os.cpu_count() or 4))
    assert res[0][2] == "pass", res[0]
    survivors = [r for r in res[1:] if r[2] != "killed"]
    assert not survivors, survivors
