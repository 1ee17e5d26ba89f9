"""CPU emulator of ``mgp_sweep`` / ``mgp_sum_partials`` (TEST ONLY).

Implements the semantics documented in include/mgrit_phi.h on CPU torch
tensors, with the oracle propagator (oracle/phi_oracle.c) for every Phi
application, so that the host-side bookkeeping of the hierarchy and of the
distributed (gloo) hierarchy can be tested on a machine without a GPU.  The
product never installs it (see paper_2104_09404_b200/device.py)."""
import numpy as np
import torch

import oracle

_MODEL = {0: "burgers", 1: "advection", 2: "shallow-water", 3: "euler"}


def _rows(t, stride, n, nx, off=0):
    return torch.as_strided(t, size=(n, nx), stride=(stride, 1),
                            storage_offset=t.storage_offset() + off)


def _params(phi, regime):
    return oracle.make_params(model=_MODEL[phi.model], k=phi.weno_k, rk_order=phi.rk_order,
                              dt=phi.dt, dx=phi.dx, eps=phi.epsilon, speed=phi.speed,
                              regime=regime, scheme=phi.scheme, lf_order=phi.lf_order,
                              m_eff=phi.m_eff, repeats=phi.repeats, gravity=phi.gravity,
                              gamma=phi.gamma, characteristic=phi.characteristic)


def _apply(p, x, n, D, nx, status):
    try:
        return oracle.phi_apply(p, x.reshape(n, D, nx)).reshape(n, D * nx)
    except oracle.PhysicalStateOracleError as e:
        # the kernel flags the status word and completes the sweep
        if status is not None:
            status.view(-1)[0] |= e.bits
        return np.full((n, D * nx), np.nan)


def _add_g(y, mode, g):
    if mode == 1:
        return y + 0.0
    if mode == 2:
        return y + g
    return y


def emulate_sweep(phi, *, n_chunks, start, start_stride, n_steps, g_mode, g, g_cs, g_ss,
                  store, st_cs, st_ss, tail, tail_regime, tail_g_mode, guess, tail_g, tg_s,
                  tail_out, to_s, tail_out2, to2_s, aux, aux_s, aux2, aux2_s, ref, ref_cs,
                  ref_ss, ref_last_next, count_nonfinite, partials, status, what):
    D = {2: 2, 3: 3}.get(phi.model, 1)
    n, cells = int(n_chunks), int(phi.nx)
    nx = D * cells   # row length
    if n == 0:
        return
    with np.errstate(all="ignore"):
        x = _rows(start, start_stride, n, nx).numpy().copy()
        acc_r = np.zeros(n)
        acc_e = np.zeros(n)
        acc_n = np.zeros(n)

        def account(v, s):
            if ref is not None:
                rr = _rows(ref, ref_cs, n, nx, s * ref_ss).numpy()
                acc_e[:] += ((v - rr) ** 2).sum(axis=1)
            if count_nonfinite:
                acc_n[:] += (~np.isfinite(v)).sum(axis=1)

        account(x, 0)
        p = _params(phi, phi.regime)
        for s in range(1, n_steps + 1):
            y = _apply(p, x, n, D, cells, status)
            gr = _rows(g, g_cs, n, nx, (s - 1) * g_ss).numpy() if g is not None else None
            x = _add_g(y, g_mode, gr)
            if store is not None:
                _rows(store, st_cs, n, nx, (s - 1) * st_ss).copy_(torch.from_numpy(x))
            account(x, s)
        if tail:
            y = _apply(_params(phi, tail_regime), x, n, D, cells, status)
            tg = _rows(tail_g, tg_s, n, nx).numpy() if tail_g is not None else None
            if tail == 1:
                _rows(tail_out, to_s, n, nx).copy_(torch.from_numpy(_add_g(y, tail_g_mode, tg)))
            elif tail == 2:
                ph = _rows(aux, aux_s, n, nx).numpy().copy()
                gf = tg if tail_g_mode == 2 else 0.0
                left = ph if tail_g_mode == 0 else gf + ph
                gc = left - y
                if guess == 0:
                    uc = _add_g(ph, tail_g_mode, tg)
                else:
                    uc = _rows(aux2, aux2_s, n, nx).numpy().copy()
                _rows(tail_out, to_s, n, nx).copy_(torch.from_numpy(gc))
                _rows(tail_out2, to2_s, n, nx).copy_(torch.from_numpy(uc))
            else:
                tgt = _rows(aux, aux_s, n, nx).numpy()
                pred = y if tail_g_mode == 0 else (tg if tail_g_mode == 2 else 0.0) + y
                acc_r[:] = ((pred - tgt) ** 2).sum(axis=1)
                if tail_out is not None:     # the kept g + Phi(x) (mgp_sweep, MGP_TAIL_RESID)
                    _rows(tail_out, to_s, n, nx).copy_(torch.from_numpy(np.ascontiguousarray(pred)))
                if ref_last_next:
                    last = tgt[n - 1]
                    if ref is not None:
                        rn = _rows(ref, ref_cs, 1, nx, n * ref_cs).numpy()[0]
                        acc_e[n - 1] += ((last - rn) ** 2).sum()
                    if count_nonfinite:
                        acc_n[n - 1] += (~np.isfinite(last)).sum()
        if partials is not None:
            pv = partials.view(-1)
            pv[0:3 * n:3] = torch.from_numpy(acc_r)
            pv[1:3 * n:3] = torch.from_numpy(acc_e)
            pv[2:3 * n:3] = torch.from_numpy(acc_n)


def emulate_sum(partials, n, width, out):
    pv = partials.view(-1)[: width * n].reshape(n, width)
    out.view(-1)[:width] = pv.sum(dim=0)


def install():
    from paper_2104_09404_b200 import device
    device.install_emulator(emulate_sweep, emulate_sum, "cpu")


def remove():
    from paper_2104_09404_b200 import device
    device.remove_emulator()
