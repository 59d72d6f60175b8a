"""The sweep count the GPU must report for a converged step (R13,
R19): the GPU tests Algorithm 1's stopping criterion (line 8) after every
launch of F sweeps, so it stops at the first multiple of F at or after the
oracle's stopping sweep k whose norm ||V^(j) - V^(j-1)|| is below tol.  The
norms come from the oracle's stopping record (nodal.c oracle_transient
dtrace: sweeps k-1, k and four sweeps continued on a copy).  A step is
"in the rounding band" when a norm that decides it lies within BAND * tol of
tol: fp64 summation order (GPU vs oracle) may flip that decision."""
BAND = 1e-6


def expected_gpu_sweeps(k, dtrace, tol, F):
    """(expected count, flagged) for one step; expected None if the record
    does not reach the decision (flagged then)."""
    k = int(k)
    norm = {k - 1: dtrace[0], k: dtrace[1]}
    for e in range(4):
        norm[k + 1 + e] = dtrace[2 + e]
    flagged = False
    if (k - 1) % F == 0 and k - 1 >= 1 and abs(norm[k - 1] - tol) <= BAND * tol:
        flagged = True
    j = -(-k // F) * F
    while j in norm:
        if abs(norm[j] - tol) <= BAND * tol:
            flagged = True
        if norm[j] < tol:
            return j, flagged
        j += F
    return None, True


def check_counts(gpu_sweeps, oracle_sweeps, dtrace, tol, F, max_flag_frac=0.1):
    """Assert equality at every step outside the rounding band (those are
    allowed +-2F); returns the flagged steps."""
    flagged = []
    steps = len(oracle_sweeps) - 1
    for s in range(1, steps + 1):
        want, fl = expected_gpu_sweeps(oracle_sweeps[s], dtrace[s], tol, F)
        if fl or want is None:
            flagged.append(s)
            assert abs(int(gpu_sweeps[s]) - int(oracle_sweeps[s])) <= 2 * F, (s, gpu_sweeps[s], oracle_sweeps[s])
        else:
            assert int(gpu_sweeps[s]) == want, (s, int(gpu_sweeps[s]), want, int(oracle_sweeps[s]))
    assert len(flagged) <= max(1, int(max_flag_frac * steps)), flagged
    return flagged


def check_counts_same_stopping(gpu_sweeps, oracle_sweeps, dtrace, tol, F):
    """GPU counts against an oracle run with the GPU's stopping semantics
    (nodal transient check_every = F): the same iteration, so the same counts
    except where the deciding norm lies within BAND * tol of tol (+-F)."""
    flagged = []
    for s in range(1, len(oracle_sweeps)):
        if abs(dtrace[s, 1] - tol) <= BAND * tol:
            flagged.append(s)
            assert abs(int(gpu_sweeps[s]) - int(oracle_sweeps[s])) <= F, s
        else:
            assert int(gpu_sweeps[s]) == int(oracle_sweeps[s]), (s, int(gpu_sweeps[s]), int(oracle_sweeps[s]))
    return flagged
