"""Static check of the built library (CPU, cuobjdump): no kernel issues a
non-coherent (LDG...CONSTANT) load before its first griddepcontrol.wait
(SASS ACQBULK). A programmatic dependent starts while its predecessor still
runs, so anything loaded before the wait may be the predecessor's stale data;
an invariant (const __restrict__) load hoisted above the wait caused exactly
that in round 2 (k4_route_verify_raw read a stale split). Plan tables that no
kernel writes are loaded before the wait on purpose -- with coherent loads."""
import os
import re
import shutil
import subprocess

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
LIB = os.path.join(ROOT, "paper_2604_08075_b200", "lib", "libfleetplan.so")


@pytest.mark.skipif(not shutil.which("cuobjdump"), reason="cuobjdump not available")
def test_no_noncoherent_load_before_griddepcontrol_wait():
    if not os.path.exists(LIB):
        import buildsys
        buildsys.build_product()
    sass = subprocess.run(["cuobjdump", "-sass", LIB], check=True, capture_output=True, text=True).stdout
    # per kernel: the non-coherent loads before its first wait -- only kernels
    # that wait at all are programmatic dependents (the others launch plainly)
    bad, n_wait, name, waited, pre = [], 0, None, False, []

    def close():
        if name is not None and waited:
            bad.extend((name, p) for p in pre)

    for line in sass.splitlines():
        if "Function :" in line:
            close()
            name, waited, pre = line.split("Function :")[1].strip(), False, []
            continue
        if name is None:
            continue
        if "ACQBULK" in line:
            if not waited:
                n_wait += 1
            waited = True
        elif not waited and re.search(r"\bLDG\S*CONSTANT", line):
            pre.append(line.strip()[:80])
    close()
    assert n_wait > 0, "no griddepcontrol.wait found: the SASS mnemonic changed?"
    assert not bad, "non-coherent loads before griddepcontrol.wait:\n" + "\n".join(f"{n}: {l}" for n, l in bad[:10])
