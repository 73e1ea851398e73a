"""Seeded synthetic inputs for the Crius Cell-estimation hot path.

This module is the ONLY code shared by the CUDA path and the CPU oracle. It
draws clusters, jobs and per-layer profile tables ("Synthetic
inputs") and holds none of the method's arithmetic: no stage split, no plan
cost, no argmin, no scheduling.  Every array it returns is plain numpy in the
layout of the C-ABI (`include/crius.h`):

  types  t : cap, gpn, mem, alpha_in, beta_in, alpha_x, beta_x
  jobs   j : job_id, submit, ng, gb, kst, n_layers, layer_off
  layers l : w, act, bnd, tpv (int64 bytes), tpn (int32 calls)
  compute  : c[t][k][l] int32 ns per sample (fwd+bwd) at tp = 2^k

The paper profiles these quantities on real GPUs ("Single-
device distributed profiling"; communication "obtained offline", :372).  No
real profile is available here, so they are synthesised from layer templates
shaped like the paper's models (Table `models`) and GPU types
shaped like Table `sim_cluster`.  The recipe is stated in
DESIGN.md §"Input recipe".
"""
from __future__ import annotations

import math
from dataclasses import dataclass, field

import numpy as np

MiB = 1 << 20
GiB = 1 << 30
K_MAX = 6  # compute profiled up to tp = 2^6 = 64

# name: (peak TF, efficiency, memory GiB, gpus per node, intra alpha ns, intra GB/s,
#        inter alpha ns, inter GB/s)                      -- SURVEY §8(d) "GPU types"
GPU_TYPES = {
    "A100-NVLink-like": (312.0, 0.45, 40, 4, 3000, 300.0, 10000, 12.5),
    "A100-PCIe-like": (312.0, 0.45, 40, 4, 8000, 24.0, 10000, 12.5),
    "V100-like": (125.0, 0.40, 32, 16, 3000, 150.0, 10000, 12.5),
    "H100-like": (989.0, 0.40, 80, 8, 2500, 450.0, 8000, 50.0),
    "A10-like": (125.0, 0.35, 24, 2, 8000, 24.0, 10000, 25.0),
    "A40-like": (150.0, 0.40, 48, 2, 8000, 24.0, 10000, 12.5),
}


def beta_ns_per_mib(gbps: float) -> int:
    """beta in integer ns per MiB: 1 MiB / (GB/s = bytes/ns)."""
    return int(round(MiB / gbps))


@dataclass
class Problem:
    """One synthetic instance: cluster + jobs + profiles + round config."""
    name: str
    type_names: list
    cap: np.ndarray          # int32 [T]
    gpn: np.ndarray          # int32 [T]
    mem: np.ndarray          # int64 [T] bytes
    alpha_in: np.ndarray     # int64 [T] ns
    beta_in: np.ndarray      # int64 [T] ns per MiB
    alpha_x: np.ndarray      # int64 [T]
    beta_x: np.ndarray       # int64 [T]
    job_id: np.ndarray       # int64 [J]
    submit: np.ndarray       # int64 [J]
    ng: np.ndarray           # int32 [J]
    gb: np.ndarray           # int32 [J]
    kst: np.ndarray          # int32 [J]
    n_layers: np.ndarray     # int32 [J]
    layer_off: np.ndarray    # int64 [J+1]
    c: np.ndarray            # int32 [T][K+1][sum L]
    w: np.ndarray            # int64 [sum L]
    act: np.ndarray          # int64 [sum L]
    bnd: np.ndarray          # int64 [sum L]
    tpv: np.ndarray          # int64 [sum L]
    tpn: np.ndarray          # int32 [sum L]
    k_max: int = K_MAX
    gpu_set: int = 0         # 0 = paper3 {NG/2, NG, 2NG}; 1 = all powers of two <= cap
    s_max: int = 16
    g_max: int = 64
    b_mode: int = 0          # 0 = B = 4S (GPipe); 1 = list
    b_values: np.ndarray = field(default_factory=lambda: np.zeros(0, np.int32))
    depth: int = 3           # search depth (default 3 at :737)
    model_names: list = field(default_factory=list)

    @property
    def n_types(self) -> int:
        return int(self.cap.shape[0])

    @property
    def n_jobs(self) -> int:
        return int(self.ng.shape[0])

    @property
    def total_layers(self) -> int:
        return int(self.layer_off[-1])


# ----------------------------------------------------------------------------
# Layer templates (SURVEY §8(d) "Layer templates"; per-sample quantities,
# 2-byte parameters and activations).  Each returns a dict of per-layer arrays:
# flops (float64, fwd+bwd per sample), w, act, bnd, tpv (int64 bytes), tpn.
# ----------------------------------------------------------------------------

def _layers(rows):
    flops, w, act, bnd, tpv, tpn = zip(*rows)
    return dict(flops=np.array(flops, np.float64), w=np.array(w, np.int64),
                act=np.array(act, np.int64), bnd=np.array(bnd, np.int64),
                tpv=np.array(tpv, np.int64), tpn=np.array(tpn, np.int32))


def _gpt_block(h, s, heads):
    # fwd = 24 s h^2 + 4 s^2 h ; fwd+bwd = 3x.  act = the block's input (2 s h
    # bytes): GPipe re-materialisation keeps only layer inputs.
    return (3.0 * (24.0 * s * h * h + 4.0 * s * s * h), 24 * h * h, 2 * s * h,
            4 * s * h, 8 * s * h, 4)


def gpt_layers(h, blocks, seq=1024, vocab=51200, emb_head=True):
    heads = max(1, h // 128)
    rows = []
    if emb_head:
        rows.append((3.0 * 2.0 * seq * h, 2 * vocab * h, 2 * seq * h, 4 * seq * h, 2 * seq * h, 1))
    rows += [_gpt_block(h, seq, heads)] * blocks
    if emb_head:
        rows.append((3.0 * 2.0 * seq * h * vocab, 2 * vocab * h, 2 * seq * h, 4 * seq * h,
                     2 * seq * h, 1))
    return _layers(rows)


def moe_layers(h, blocks, experts, seq=1024, vocab=51200):
    rows = [(3.0 * 2.0 * seq * h, 2 * vocab * h, 2 * seq * h, 4 * seq * h, 2 * seq * h, 1)]
    for b in range(blocks):
        if b % 2 == 1:  # every other block is MoE (GShard): top-2 experts
            rows.append((3.0 * (40.0 * seq * h * h + 4.0 * seq * seq * h),
                         experts * 16 * h * h + 8 * h * h, 2 * seq * h, 4 * seq * h,
                         16 * seq * h, 4))  # tpv doubled: stands in for all-to-all
        else:
            rows.append(_gpt_block(h, seq, max(1, h // 64)))
    rows.append((3.0 * 2.0 * seq * h * vocab, 2 * vocab * h, 2 * seq * h, 4 * seq * h, 2 * seq * h, 1))
    return _layers(rows)


def wres_layers(params_b):
    """Wide-ResNet-style: stem, 16 bottleneck blocks (3/4/6/3), head; image 224.
    Per group channels x2 and spatial /2: flat FLOPs, params x4, act /2."""
    wf = math.sqrt(params_b * 1e9 / (212992.0 * 307.0))
    rows = []
    c0 = 64 * wf
    rows.append((3.0 * 2.0 * 9408 * wf * 112 * 112, int(2 * 9408 * wf), int(2 * 2 * c0 * 112 * 112),
                 int(4 * c0 * 56 * 56), int(8 * c0 * 56 * 56), 1))
    for g, n in enumerate((3, 4, 6, 3)):
        params = wf * wf * (4 ** g) * 212992.0
        hw = (56 // (2 ** g)) ** 2
        C = 256 * wf * 2 ** g
        B = 128 * wf * 2 ** g
        for _ in range(n):
            rows.append((3.0 * 2.0 * params * hw, int(2 * params), int(2 * C * hw),
                         int(4 * C * hw), int(8 * C * hw), 2))
    C3 = 256 * wf * 8
    rows.append((3.0 * 2.0 * C3 * 1000, int(2 * C3 * 1000), int(2 * C3), int(4 * 1000), int(2 * 1000), 1))
    return _layers(rows)


GPT_SIZES = {"GPT-0.76B": (1536, 24), "GPT-1.3B": (2048, 24), "GPT-2.6B": (2560, 32),
             "GPT-6.7B": (4096, 32)}
MOE_SIZES = {"MoE-0.69B": (768, 8, 8), "MoE-1.3B": (768, 16, 16), "MoE-2.4B": (1024, 16, 16),
             "MoE-10B": (1536, 16, 32), "MoE-27B": (2048, 16, 48)}
WRES_SIZES = {"WRes-0.5B": 0.5, "WRes-1B": 1.0, "WRes-2B": 2.0, "WRes-4B": 4.0, "WRes-6.8B": 6.8}
FAMILY_GB = {"GPT": (128, 256, 512), "MoE": (256, 512, 1024), "WRes": (256, 512, 1024)}


def model_layers(name):
    if name in GPT_SIZES:
        h, b = GPT_SIZES[name]
        return gpt_layers(h, b)
    if name in MOE_SIZES:
        h, b, e = MOE_SIZES[name]
        return moe_layers(h, b, e)
    if name in WRES_SIZES:
        return wres_layers(WRES_SIZES[name])
    if name == "GPT96":
        return gpt_layers(4096, 96, seq=2048, emb_head=False)
    if name.startswith("GPTtiny"):  # cfg1: L identical blocks
        L = int(name[len("GPTtiny"):])
        return gpt_layers(1024, L, seq=1024, emb_head=False)
    raise KeyError(name)


def family(name):
    return name.split("-")[0] if "-" in name else "GPT"


# ----------------------------------------------------------------------------
# Assembly
# ----------------------------------------------------------------------------

def _cluster(spec):
    """spec: list of (type name, capacity, gpn override or None)."""
    names, cap, gpn, mem, ai, bi, ax, bx, peak = [], [], [], [], [], [], [], [], []
    for name, capacity, gpn_over in spec:
        pk, eff, mem_gib, g, a_in, gbps_in, a_x, gbps_x = GPU_TYPES[name]
        names.append(name)
        cap.append(capacity)
        gpn.append(gpn_over if gpn_over else g)
        mem.append(mem_gib * GiB)
        ai.append(a_in)
        bi.append(beta_ns_per_mib(gbps_in))
        ax.append(a_x)
        bx.append(beta_ns_per_mib(gbps_x))
        peak.append(pk * eff)
    return (names, np.array(cap, np.int32), np.array(gpn, np.int32), np.array(mem, np.int64),
            np.array(ai, np.int64), np.array(bi, np.int64), np.array(ax, np.int64),
            np.array(bx, np.int64), np.array(peak, np.float64))


def _compute_table(flops, eff_peak_tf, k_max, rng, jitter):
    """c[t][k][l] = max(1, ceil(FLOPs_l / (peak_t eff_t 2^k 0.85^k) * u)) ns
    (SURVEY §8(d) "Compute table"; TP efficiency 0.85^log2(tp) follows SPEC)."""
    T = eff_peak_tf.shape[0]
    K1 = k_max + 1
    ks = np.arange(K1, dtype=np.float64)
    denom = eff_peak_tf[:, None] * 1e3 * (2.0 ** ks)[None, :] * (0.85 ** ks)[None, :]  # FLOP per ns
    base = flops[None, None, :] / denom[:, :, None]
    if jitter:
        u = rng.uniform(0.95, 1.05, size=base.shape)
        base = base * u
    c = np.maximum(1.0, np.ceil(base))
    assert c.max() < 2 ** 31
    return c.astype(np.int32)


def assemble(name, cluster_spec, models, ng, gb, rng, *, jitter=True, submit=None, job_id=None,
             **cfg):
    names, cap, gpn, mem, ai, bi, ax, bx, peak = _cluster(cluster_spec)
    J = len(models)
    per = [model_layers(m) for m in models]
    nl = np.array([p["flops"].shape[0] for p in per], np.int32)
    off = np.zeros(J + 1, np.int64)
    off[1:] = np.cumsum(nl)
    cat = {k: np.concatenate([p[k] for p in per]) for k in ("flops", "w", "act", "bnd", "tpv", "tpn")}
    c = _compute_table(cat["flops"], peak, K_MAX, rng, jitter)
    if submit is None:
        submit = np.arange(J, dtype=np.int64)
    if job_id is None:
        job_id = np.arange(J, dtype=np.int64)
    return Problem(name=name, type_names=names, cap=cap, gpn=gpn, mem=mem, alpha_in=ai, beta_in=bi,
                   alpha_x=ax, beta_x=bx, job_id=np.asarray(job_id, np.int64),
                   submit=np.asarray(submit, np.int64), ng=np.asarray(ng, np.int32),
                   gb=np.asarray(gb, np.int32), kst=np.full(J, 8, np.int32), n_layers=nl,
                   layer_off=off, c=c, w=cat["w"], act=cat["act"], bnd=cat["bnd"], tpv=cat["tpv"],
                   tpn=cat["tpn"], model_names=list(models), **cfg)


NG_CHOICES = np.array([1, 2, 4, 8, 16, 32, 64], np.int32)
NG_WEIGHTS = np.array([.25, .20, .20, .18, .10, .05, .02])


def _trace(rng, J, model_pool):
    """Philly-like job mix: skewed N_G (PAPER.md:584 randomises it), family
    uniform, size uniform in family, Poisson submits (integer s, ties allowed),
    unique ids in random order so (submit, id) priority != input order on ties."""
    fams = sorted(model_pool)
    ng = rng.choice(NG_CHOICES, size=J, p=NG_WEIGHTS / NG_WEIGHTS.sum()).astype(np.int32)
    models, gb = [], []
    for _ in range(J):
        f = fams[rng.integers(len(fams))]
        m = model_pool[f][rng.integers(len(model_pool[f]))]
        models.append(m)
        gbs = FAMILY_GB.get(family(m), (512, 1024))
        gb.append(gbs[rng.integers(len(gbs))])
    submit = np.cumsum(rng.exponential(20.0, size=J)).astype(np.int64)
    job_id = rng.permutation(J).astype(np.int64) + 1000
    return models, ng, np.array(gb, np.int32), submit, job_id


POOL = {"GPT": list(GPT_SIZES), "MoE": list(MOE_SIZES), "WRes": list(WRES_SIZES)}
CFG4_CLUSTER = [("A100-NVLink-like", 512, None), ("V100-like", 512, None), ("H100-like", 512, None),
                ("A10-like", 512, None)]
B_SWEEP = np.array([1, 2, 4, 8, 16, 32, 64], np.int32)


def make_config(cfg, seed=None, variant=None, scale=1, jitter=True):
    """BASELINE.json configs 1-5 (SURVEY §8(d) "Configs").  seed defaults to
    the config id (headline run); variants: cfg1 'sweep'; cfg4 'pow2';
    `scale` multiplies the job count (cfg '5x' steady-state runs)."""
    cfg = int(cfg)
    seed = cfg if seed is None else seed
    rng = np.random.default_rng(seed)
    if cfg == 1:
        kw = dict(gpu_set=1, s_max=4, g_max=4, depth=3)
        if variant == "sweep":
            kw.update(b_mode=1, b_values=np.array([1, 2, 4, 8, 16], np.int32))
        return assemble("cfg1" + (f"-{variant}" if variant else ""),
                        [("A100-NVLink-like", 4, 4), ("V100-like", 4, 4)], ["GPTtiny8"], [2], [32],
                        rng, jitter=jitter, **kw)
    if cfg == 2:
        models = ["GPT-1.3B", "GPT-2.6B", "MoE-1.3B", "MoE-2.4B", "WRes-1B", "WRes-2B", "GPT-0.76B",
                  "MoE-0.69B"]
        ng = rng.choice(np.array([2, 4, 8, 16], np.int32), size=8)
        gb = [FAMILY_GB[family(m)][rng.integers(3)] for m in models]
        return assemble("cfg2", [("A100-NVLink-like", 16, None), ("A100-PCIe-like", 16, None),
                                 ("V100-like", 32, None)], models, ng, gb, rng, jitter=jitter,
                        gpu_set=0, s_max=16, g_max=64, depth=3)
    if cfg == 3:
        models, ng, gb, submit, jid = _trace(rng, 1000 * scale, POOL)
        return assemble("cfg3", [("A100-NVLink-like", 128, None), ("V100-like", 128, None),
                                 ("A40-like", 256, None)], models, ng, gb, rng, jitter=jitter,
                        submit=submit, job_id=jid, gpu_set=0, s_max=16, g_max=64, b_mode=1,
                        b_values=B_SWEEP.copy(), depth=3)
    if cfg == 4:
        models, ng, gb, submit, jid = _trace(rng, 10000 * scale, POOL)
        return assemble("cfg4" + ("-pow2" if variant == "pow2" else ""), CFG4_CLUSTER, models, ng, gb,
                        rng, jitter=jitter, submit=submit, job_id=jid,
                        gpu_set=1 if variant == "pow2" else 0, s_max=16, g_max=64, depth=3)
    if cfg == 5:
        J = 10000 * scale
        _, ng, _, submit, jid = _trace(rng, J, {"GPT": ["GPT96"]})
        gb = rng.choice(np.array([512, 1024], np.int32), size=J)
        return assemble("cfg5" + (f"x{scale}" if scale != 1 else ""), CFG4_CLUSTER, ["GPT96"] * J, ng,
                        gb, rng, jitter=jitter, submit=submit, job_id=jid, gpu_set=1, s_max=32,
                        g_max=64, b_mode=1, b_values=B_SWEEP.copy(), depth=3)
    raise ValueError(f"unknown config {cfg}")


def random_tiny(seed, *, max_layers=8, n_types=2, n_jobs=3, b_mode=None, gpu_set=None):
    """Tiny random instance for brute-force pins: random per-layer tables drawn
    directly (not from templates), small caps, random B sets; values kept
    small so ties are frequent."""
    rng = np.random.default_rng(seed)
    T, J = n_types, n_jobs
    cap = rng.choice(np.array([1, 2, 4, 8, 16], np.int32), size=T)
    gpn = rng.choice(np.array([1, 2, 4, 8], np.int32), size=T)
    mem = rng.integers(50, 4000, size=T).astype(np.int64)
    ai = rng.integers(1, 50, size=T).astype(np.int64)
    ax = rng.integers(1, 200, size=T).astype(np.int64)
    bi = rng.integers(1, 4 * MiB, size=T).astype(np.int64)
    bx = rng.integers(1, 16 * MiB, size=T).astype(np.int64)
    nl = rng.integers(1, max_layers + 1, size=J).astype(np.int32)
    off = np.zeros(J + 1, np.int64)
    off[1:] = np.cumsum(nl)
    L = int(off[-1])
    c = rng.integers(1, 12, size=(T, 4, L)).astype(np.int32)
    k_max = 3
    ng = rng.choice(np.array([1, 2, 4, 8], np.int32), size=J)
    gb = rng.choice(np.array([1, 2, 4, 8, 16, 32, 64], np.int32), size=J)
    bm = int(rng.integers(2)) if b_mode is None else b_mode
    bv = np.sort(rng.choice(np.array([1, 2, 4, 8, 16, 32], np.int32), size=int(rng.integers(1, 4)),
                            replace=False)).astype(np.int32)
    return Problem(name=f"tiny{seed}", type_names=[f"T{i}" for i in range(T)], cap=cap, gpn=gpn,
                   mem=mem, alpha_in=ai, beta_in=bi, alpha_x=ax, beta_x=bx,
                   job_id=rng.permutation(J).astype(np.int64),
                   submit=rng.integers(0, 3, size=J).astype(np.int64), ng=ng, gb=gb,
                   kst=rng.integers(1, 9, size=J).astype(np.int32), n_layers=nl, layer_off=off, c=c,
                   w=rng.integers(0, 100, size=L).astype(np.int64),
                   act=rng.integers(0, 20, size=L).astype(np.int64),
                   bnd=rng.integers(0, 64, size=L).astype(np.int64),
                   tpv=rng.integers(0, 64, size=L).astype(np.int64),
                   tpn=rng.integers(0, 5, size=L).astype(np.int32), k_max=k_max,
                   gpu_set=int(rng.integers(2)) if gpu_set is None else gpu_set,
                   s_max=int(rng.choice([1, 2, 4, 8])), g_max=int(rng.choice([1, 2, 4, 8])),
                   b_mode=bm, b_values=bv, depth=int(rng.integers(0, 4)),
                   model_names=[f"rand{j}" for j in range(J)])


def iterations_for(pr, seed=0, lo=100, hi=5000):
    """Training length of every job (iterations), log-uniform in [lo, hi]
    (SPEC.md workload module's reading of the paper's trace adaptation)."""
    rng = np.random.default_rng(10_000 + seed)
    return np.exp(rng.uniform(np.log(lo), np.log(hi), size=pr.n_jobs)).astype(np.int64)


def subset(pr, n_jobs):
    """The first n_jobs jobs of a Problem (same cluster, tables sliced)."""
    import copy
    q = copy.copy(pr)
    L = int(pr.layer_off[n_jobs])
    for k in ("job_id", "submit", "ng", "gb", "kst", "n_layers"):
        setattr(q, k, getattr(pr, k)[:n_jobs].copy())
    q.layer_off = pr.layer_off[:n_jobs + 1].copy()
    for k in ("w", "act", "bnd", "tpv", "tpn"):
        setattr(q, k, getattr(pr, k)[:L].copy())
    q.c = np.ascontiguousarray(pr.c[:, :, :L])
    q.model_names = pr.model_names[:n_jobs]
    q.name = f"{pr.name}[:{n_jobs}]"
    return q
