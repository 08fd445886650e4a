"""The oracle mutation list (scripts/oracle_mutants.py) still applies.

Each mutant is a plausible mistake in oracle/ that some oracle pin must
catch; the script runs the pins against every mutant (results in
profiles/r02_oracle_mutants.json).  This fast check only makes sure every
mutant's text still occurs in the oracle as the list says, so the list
cannot silently go stale when the oracle changes."""
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, os.path.join(ROOT, "scripts"))

import oracle_mutants  # noqa: E402


def test_every_mutant_applies_to_the_current_oracle():
    oracle_mutants.check_all_apply()
    assert len(oracle_mutants.MUTANTS) >= 78
    files = {m[1] for m in oracle_mutants.MUTANTS}
    assert files == {"kvpool.py", "cfs.py", "sim.py", "pattern.py", "bwfit.py"}


def test_every_product_mutant_applies_to_the_current_sources():
    """scripts/product_mutants.py: one-line edits of libaqua's kernels, host
    library and native scheduler that the parity tests must catch (results
    in profiles/r02_product_mutants_{cpu,gpu}.json)."""
    import product_mutants
    product_mutants.check_all_apply()
    kinds = {m[3] for m in product_mutants.MUTANTS}
    assert kinds == {"cpu", "gpu"}


def test_a_sample_of_oracle_mutants_is_killed():
    """Run four mutants for real (one per oracle module with arithmetic):
    each must fail an oracle pin.  The whole list runs with
    `python scripts/oracle_mutants.py` (results in profiles/)."""
    names = {"U counts K or V only (U = L*S)", "decode order: most tokens generated first (P:833)",
             "reschedule every k+1 iterations (P:836)", "splitmix64 (vectorised): wrong second shift"}
    idx = [i for i, m in enumerate(oracle_mutants.MUTANTS) if m[0] in names]
    assert len(idx) == len(names)
    for i in idx:
        r = oracle_mutants.run_one(i)
        assert r["killed"], r
