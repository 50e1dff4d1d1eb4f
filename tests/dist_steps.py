"""CPU stand-in for the two steps of the distributed reverse sweep (test infrastructure, SURVEY §4
"fake backends"): the same block arithmetic as cd_dist_rev_panel / cd_dist_rev_update written with
numpy on the storage tensors, the diagonal block by the oracle's unblocked sweep.
Lets the gloo tests check the host loop, ownership and broadcast of paper_1602_07527_b200/dist.py."""
import numpy as np

import oracle


class NumpySteps:
    def panel(self, n, j, w, Lk, Ak, X):
        k = j + w
        Lm = Lk.numpy().T  # (n, w) column block, logical orientation (views share memory)
        Am = Ak.numpy().T
        Xm = X.numpy().reshape(w, n - j).T  # (n - j, w), ld = n - j
        D = np.tril(Lm[j:k, :])
        if k < n:
            Am[k:n, :] = Am[k:n, :] @ np.linalg.inv(D)  # Cbar <- Cbar D^{-1}
            Am[j:k, :] = np.tril(Am[j:k, :]) - np.tril(Am[k:n, :].T @ Lm[k:n, :])
        Db = oracle.chol_rev(D, np.tril(Am[j:k, :]))
        Am[j:k, :] = Db
        Xm[:w, :] = Db + Db.T  # S = Dbar + Dbar^T (diagonal doubled)
        Xm[w:, :] = Am[k:n, :]

    def update(self, n, j, w, X, q, Lq, Aq):
        if q == 0:
            return
        k = j + w
        Lm = Lq.numpy().T  # (n, q)
        Am = Aq.numpy().T
        Xm = X.numpy().reshape(w, n - j).T
        Am[k:n, :] -= Xm[w:, :] @ Lm[j:k, :]  # Bbar <- Bbar - Cbar R
        Am[j:k, :] -= Xm.T @ Lm[j:n, :]  # Rbar <- Rbar - [S; Cbar]^T [R; B]

    def fwd_partial(self, n, j, w, q, Lq, Aq, Z):
        Zm = Z.numpy().reshape(w, n - j).T
        if q == 0:
            Zm[:] = 0.0
            return
        k = j + w
        Lm = Lq.numpy().T
        Am = Aq.numpy().T
        Zm[:] = Am[j:n, :] @ Lm[j:k, :].T + Lm[j:n, :] @ Am[j:k, :].T

    def fwd_panel(self, n, j, w, Lk, Ak, Z):
        k = j + w
        Lm = Lk.numpy().T
        Am = Ak.numpy().T
        Zm = Z.numpy().reshape(w, n - j).T
        D = np.tril(Lm[j:k, :])
        Dd = np.tril(Am[j:k, :]) - np.tril(Zm[:w, :])
        Dd = np.tril(oracle.chol_fwd(D, Dd + np.tril(Dd, -1).T))  # chol_unblocked_fwd on the block
        Am[j:k, :] = Dd
        if k < n:
            Cd = Am[k:n, :] - Zm[w:, :]
            Am[k:n, :] = (Cd - Lm[k:n, :] @ Dd.T) @ np.linalg.inv(D).T
