"""Newton power flow on the bus admittance matrix -- TEST INFRASTRUCTURE ONLY.

Used by tests/ as an independent physical check on the ACOPF constraint
tape: a converged power-flow point mapped onto the ACOPF variable vector
must satisfy every equality row (the reference suite's power-flow point
check, pkg/tests/test_autodiff.py:76-83 with its helper in
pkg/tests/oracles.py:119-215).  Restated here from the textbook polar
formulation: complex Ybus, mismatch S_spec - V conj(Y V), and the analytic
Jacobian dS/dVa = j diag(V) conj(diag(I) - Y diag(V)),
dS/dVm = diag(V) conj(Y diag(V/|V|)) + conj(diag(I)) diag(V/|V|).
Never imported by the product package.
"""
import numpy as np

PQ, PV, REF = 1, 2, 3


def branch_pi(br):
    """(yff, yft, ytf, ytt) of the tap/phase-shift pi model."""
    ys = 1.0 / complex(br.r, br.x)
    bc = 0.5j * br.b_charge
    tc = br.tap * np.exp(1j * br.shift)
    return (ys + bc) / (tc * np.conj(tc)), -ys / np.conj(tc), -ys / tc, ys + bc


def ybus(net):
    idx = net.bus_index()
    Y = np.zeros((len(net.buses),) * 2, complex)
    for br in net.branches:
        f, t = idx[br.from_bus], idx[br.to_bus]
        yff, yft, ytf, ytt = branch_pi(br)
        Y[f, f] += yff
        Y[f, t] += yft
        Y[t, f] += ytf
        Y[t, t] += ytt
    for k, u in enumerate(net.buses):
        Y[k, k] += complex(u.gs, u.bs)
    return Y


def newton_power_flow(net, tol=1e-12, max_iter=30):
    """(vm, va) solving the PV/PQ mismatch equations; raises if not converged."""
    idx = net.bus_index()
    Y = ybus(net)
    nb = len(net.buses)
    types = np.array([u.type for u in net.buses])
    vm = np.array([u.vm for u in net.buses], float)
    va = np.zeros(nb)
    pg = np.zeros(nb)
    for g in net.generators:
        pg[idx[g.bus]] += g.pg
        vm[idx[g.bus]] = g.vg
    sspec = pg - np.array([u.pd for u in net.buses]) - 1j * np.array([u.qd for u in net.buses])
    pvpq = np.flatnonzero(types != REF)
    pq = np.flatnonzero(types == PQ)
    for _ in range(max_iter):
        V = vm * np.exp(1j * va)
        I = Y @ V
        mis = sspec - V * np.conj(I)
        F = np.concatenate([mis.real[pvpq], mis.imag[pq]])
        if np.max(np.abs(F), initial=0.0) < tol:
            return vm, va
        dVa = 1j * np.diag(V) @ np.conj(np.diag(I) - Y @ np.diag(V))
        Vn = V / np.abs(V)
        dVm = np.diag(V) @ np.conj(Y @ np.diag(Vn)) + np.conj(np.diag(I)) @ np.diag(Vn)
        J = np.block([[dVa.real[np.ix_(pvpq, pvpq)], dVm.real[np.ix_(pvpq, pq)]],
                      [dVa.imag[np.ix_(pq, pvpq)], dVm.imag[np.ix_(pq, pq)]]])
        dx = np.linalg.solve(J, F)
        va[pvpq] += dx[:pvpq.size]
        vm[pq] += dx[pvpq.size:]
    raise RuntimeError("power flow did not converge")


def power_flow_point(net, variables, n_var):
    """Map a converged power flow onto the ACOPF variable vector: voltages,
    generator injections (shared evenly between generators on one bus) and
    the four branch flows."""
    idx = net.bus_index()
    vm, va = newton_power_flow(net)
    V = vm * np.exp(1j * va)
    S = V * np.conj(ybus(net) @ V)
    x = np.zeros(n_var)
    x[variables.va] = va
    x[variables.vm] = vm
    sg = S + np.array([complex(u.pd, u.qd) for u in net.buses])
    count = np.zeros(len(net.buses))
    for g in net.generators:
        count[idx[g.bus]] += 1
    for gi, g in enumerate(net.generators):
        k = idx[g.bus]
        x[variables.pg[gi]] = sg[k].real / count[k]
        x[variables.qg[gi]] = sg[k].imag / count[k]
    for bi, br in enumerate(net.branches):
        f, t = idx[br.from_bus], idx[br.to_bus]
        yff, yft, ytf, ytt = branch_pi(br)
        sf = V[f] * np.conj(yff * V[f] + yft * V[t])
        st = V[t] * np.conj(ytf * V[f] + ytt * V[t])
        x[variables.p_from[bi]], x[variables.q_from[bi]] = sf.real, sf.imag
        x[variables.p_to[bi]], x[variables.q_to[bi]] = st.real, st.imag
    return x
