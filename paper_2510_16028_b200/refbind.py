"""The drop-in binding of libnao_b200.so into the UNMODIFIED reference package
(`fpverify`, /root/reference/pkg/src/fpverify): INTEGRATION.md section 1 as
code.  `install()` rebinds the reference's hot-path names to this package so
every caller inside the reference -- co_execute (bounds.py:221-262),
observed_p_max / screen (dispute.py:130-150), the leaf route of
Challenger.leaf_payload (dispute.py:605-671), calibration and the Merkle
commitments -- runs on the B200 kernels, while arguments and results keep
the reference's own types (numpy arrays, fpverify BoundTensor / MerkleTree /
Tensor).

    import fpverify, paper_2510_16028_b200.refbind as rb
    rb.install()          # idempotent; rb.CALLS counts the rebound calls

tests/test_reference_suite_gpu.py runs the reference's own test files with
this binding installed (tests/ref_plugin.py) on the B200.
"""

from __future__ import annotations

import collections

import numpy as np

CALLS: collections.Counter = collections.Counter()
_INSTALLED = False


def _counted(name, fn):
    def wrapper(*a, **k):
        CALLS[name] += 1
        return fn(*a, **k)
    wrapper.__name__ = getattr(fn, "__name__", name)
    wrapper.__doc__ = getattr(fn, "__doc__", None)
    wrapper.__wrapped__ = fn
    return wrapper


def install() -> None:
    """Rebind the reference's hot-path functions (see module docstring)."""
    global _INSTALLED
    if _INSTALLED:
        return
    from fpverify import bounds as rb, calibration as rc, commitments as rcm, dispute as rd

    from . import bounds as B, calibration as C, commitments as M, dispute as D

    def op_bound(node, arrays, model, profile=None):
        """bounds.py:176-218 -> (y float32, eps float64) numpy."""
        y, eps = B.op_bound(node, [np.asarray(a) for a in arrays], model, profile)
        return y, eps

    def matmul_bound(a, b, model, fma=False, transpose_b=False):
        """bounds.py:100-111 -> fpverify BoundTensor."""
        return rb.BoundTensor.from_array(
            B.matmul_bound(np.asarray(a), np.asarray(b), model, fma, transpose_b).array)

    def softmax_bound_parts(x, axis, model, profile=None):
        return B.softmax_bound_parts(np.asarray(x), axis, model, profile)

    def softmax_bound(x, axis, model, profile=None):
        _, eps = B.softmax_bound_parts(np.asarray(x), axis, model, profile)
        return rb.BoundTensor.from_array(eps)

    def layernorm_bound_parts(x, axis, eps_attr, model, profile=None):
        return B.layernorm_bound_parts(np.asarray(x), axis, eps_attr, model, profile)

    def percentile_profile(values, grid=rc.PERCENTILE_GRID):
        return C.percentile_profile(np.asarray(values), grid)

    def percentile(values, p):
        return C.percentile(np.asarray(values), p)

    def build_tree(leaves):
        """commitments.py:141-142 on the GPU -> an fpverify MerkleTree (levels
        hashed by nao_merkle_hash_leaves / nao_merkle_root_of)."""
        ours = M.build_tree(list(leaves))
        t = rcm.MerkleTree.__new__(rcm.MerkleTree)
        t.levels = [list(level) for level in ours.levels]
        return t

    def leaf_payload(self, state, part_payload, committee_pool, commit_payload=None):
        """Challenger.leaf_payload (dispute.py:605-671): the reference's own
        argument decoding, then the leaf route on the GPU (dispute.leaf_route:
        exact bound check with the certified band settled, FP64 oracle
        recheck, committee of emulated profiles)."""
        leaf = state.leaf_index
        node = self.graph.nodes[leaf]
        if part_payload is None:
            claimed = rd.decode_tensor(commit_payload["outputs"][0])
            args = []
            for ref in node.inputs:
                cat, key = rd.parse_ref(ref)
                args.append(self.graph.weights[key].array if cat == "weight"
                            else self.inputs[key].array)
        else:
            doc = None
            for child_doc in part_payload["children"]:
                if child_doc["start"] == leaf and child_doc["end"] == leaf + 1:
                    doc = child_doc
                    break
            if doc is None:
                raise rd.ProtocolError("leaf slice missing from final partition round")
            claimed = rd.decode_tensor(doc["out_tensors"][str(leaf)])
            args = []
            for ref in node.inputs:
                cat, key = rd.parse_ref(ref)
                args.append(self.graph.weights[key].array if cat == "weight"
                            else rd.decode_tensor(doc["in_tensors"][ref]).array)
        res = D.leaf_route(node, args, claimed.array, self.thresholds, committee_pool,
                           self.config.committee_size, self.config.committee_seed,
                           model=self.config.fp_model, profile=self.profile, leaf=leaf)
        ev = res["evidence"]
        evidence = {"leaf": leaf, "leaf_name": node.name,
                    "claimed_digest": rcm.tensor_digest(claimed)}
        for key in ("max_excess", "votes_within", "committee"):
            if key in ev:
                evidence[key] = ev[key]
        for key in ("undecided_bound_elements", "undecided_oracle_elements"):
            if ev.get(key):  # only when the reference's FP64 order could matter
                evidence[key] = ev[key]
        flops = rd.node_flops(node, tuple(np.asarray(claimed.array).shape),
                              [np.asarray(a).shape for a in args])
        return {"path": res["path"], "winner": res["winner"], "evidence": evidence,
                "flops": flops}

    def calibrate(g, dataset, profiles, grid=rc.PERCENTILE_GRID, epsilon=rc.DEFAULT_EPSILON):
        """calibration.py:70-114 on the GPU (every profile emulated bit-exactly,
        exact percentiles) -> an fpverify EnvelopeSet."""
        if len(profiles) < 2:
            raise ValueError("calibration requires at least 2 device profiles")
        if not dataset:
            raise ValueError("calibration requires at least 1 input")
        feed = [{k: np.asarray(v.array) for k, v in sample.items()} for sample in dataset]
        env = C.calibrate(g, feed, profiles, grid, epsilon)
        return rc.EnvelopeSet(grid=tuple(env.grid), abs_env=list(env.abs_env),
                              rel_env=list(env.rel_env), node_names=list(env.node_names),
                              per_sample_abs=[list(r) for r in env.per_sample_abs])

    def sample_committee(pool, size, seed):
        return D.sample_committee(pool, size, seed)

    rb.op_bound = _counted("op_bound", op_bound)
    rb.matmul_bound = _counted("matmul_bound", matmul_bound)
    rb.softmax_bound_parts = _counted("softmax_bound_parts", softmax_bound_parts)
    rb.softmax_bound = _counted("softmax_bound", softmax_bound)
    rb.layernorm_bound_parts = _counted("layernorm_bound_parts", layernorm_bound_parts)
    rc.percentile_profile = _counted("percentile_profile", percentile_profile)
    rc.percentile = _counted("percentile", percentile)
    rd.op_bound = rb.op_bound                        # imported by name, dispute.py:19
    rd.percentile_profile = rc.percentile_profile   # dispute.py:20
    rc.calibrate = _counted("calibrate", calibrate)
    rcm.build_tree = _counted("build_tree", build_tree)
    rd.Challenger.leaf_payload = _counted("leaf_payload", leaf_payload)
    rd.sample_committee = _counted("sample_committee", sample_committee)
    _INSTALLED = True
