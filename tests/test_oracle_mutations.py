"""Mutation check of the convention pins: build deliberately broken copies of the oracle
(plausible alternative readings of the paper, plus the mutations the round-1 review ran) and
require that tests/test_oracle_conventions.py FAILS on every one of them.  A mutation that
survives would mean the corresponding reading is not pinned.  CPU only (gcc).

Not listed because it is equivalent, not an alternative reading: dropping the keep() test on a
relaxation's RESULT inside the closure (`if (!keep(k, c)) continue;`).  A result that fails keep
can never beat a kept entry, and an entry touched only by failing results never survives
make_layer's filter, so the survivors are identical for every input."""
import os
import subprocess
import sys

import pytest

HERE = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(HERE)
SRC = os.path.join(ROOT, "oracle", "wfst_oracle.c")

# (name, reading it breaks, exact text in wfst_oracle.c, replacement)
MUTATIONS = [
    ("tie_break_reversed", "R9",
     "return (uint32_t)a1 < (uint32_t)a2;", "return (uint32_t)a1 > (uint32_t)a2;"),
    ("beam_keep_le", "R5 strict <",
     "return c < k->beam_cut &&", "return c <= k->beam_cut &&"),
    ("no_initial_cutoff", "R3",
     "Keep k0 = {0.0f + beam, INFINITY, 0};", "Keep k0 = {INFINITY, INFINITY, 0};"),
    ("alpha_after_closure", "R6 order (Fig. 1 P:77, P:86)",
     "    Keep k = {best + beam, INFINITY, 0};\n    int32_t n_in = 0;",
     "    Keep k = {best + beam, INFINITY, 0};\n    relax_total += eps_closure(&w, &k);\n    int32_t n_in = 0;"),
    ("alpha_keep_strict", "R6 ties survive",
     "(!k->use_alpha || c <= k->kalpha)", "(!k->use_alpha || c < k->kalpha)"),
    ("alpha_plus_one", "R6 alpha-th smallest",
     "k.kalpha = w.tmp[max_active - 1];", "k.kalpha = w.tmp[max_active];"),
    ("emit_sum_order", "R1 order",
     "float c = (cp + g->weight[a]) - row[g->ilabel[a] - 1];",
     "float c = cp + (g->weight[a] - row[g->ilabel[a] - 1]);"),
]


@pytest.mark.parametrize("name,reading,old,new", MUTATIONS, ids=[m[0] for m in MUTATIONS])
def test_mutation_is_caught(tmp_path, name, reading, old, new):
    src = open(SRC).read()
    assert src.count(old) == 1, f"mutation site for {name} not found exactly once"
    mut = tmp_path / "wfst_oracle_mut.c"
    mut.write_text(src.replace(old, new))
    lib = tmp_path / "libwfst_oracle_mut.so"
    subprocess.check_call(["gcc", "-O2", "-std=c11", "-ffp-contract=off", "-fno-fast-math", "-fPIC", "-shared",
                           "-pthread", "-o", str(lib), str(mut), "-lm"])
    env = dict(os.environ, WFST_ORACLE_LIB=str(lib))
    targets = [os.path.join(HERE, "test_oracle_conventions.py")]
    r = subprocess.run([sys.executable, "-m", "pytest", "-q", "-x", "-p", "no:cacheprovider", *targets],
                       cwd=ROOT, env=env, capture_output=True, text=True, timeout=600)
    assert r.returncode != 0, f"mutation {name} ({reading}) survived the pins:\n{r.stdout[-2000:]}"
