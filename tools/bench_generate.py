#!/usr/bin/env python
"""Integrated verify loop at BASELINE config 1: draft
2L/4H, target 4L/8H, d_head 64, 4K prompt, 90% sparsity, gamma 4, 40 new
tokens — the device-resident ``paper_2605_15508_b200.generate`` vs the
reference's own ``specsparse.specdec.generate`` on the host cores (from
baseline/_ref when installed), same weights / mappings / prompt; tokens must
match.  Also the self-speculating c1 target.  One JSON line per case."""
import io
import json
import sys
import tempfile
import time
from pathlib import Path

ROOT = Path(__file__).resolve().parent.parent
sys.path.insert(0, str(ROOT))
import torch  # noqa: E402

import paper_2605_15508_b200 as P  # noqa: E402
from oracle import sts_oracle as O  # noqa: E402

REF = ROOT / "baseline" / "_ref"
for name in ("c1", "c1_self"):
    doc = json.loads((ROOT / "tests" / "golden" / "generate" / f"{name}.json").read_text())
    target = O.init_model(O.OracleModelConfig(**doc["target_config"]))
    draft = target if doc["draft_config"] is None else O.init_model(O.OracleModelConfig(**doc["draft_config"]))
    with tempfile.TemporaryDirectory() as td:
        paths = []
        for i, m in enumerate(doc["mappings"]):
            p = Path(td) / f"m{i}.json"
            p.write_text(json.dumps(m))
            paths.append(p)
        ms = P.MappingSet.from_paths(paths)
    cfg = P.SpecConfig(gamma=doc["gamma"], sparsity=P.SparsityConfig(**doc["sparsity"]), mappings=ms)
    P.generate(draft, target, doc["prompt"], doc["max_new"], cfg)  # warm-up (weights upload, kernels)
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    log = io.StringIO()
    res = P.generate(draft, target, doc["prompt"], doc["max_new"], cfg, event_log=log)
    torch.cuda.synchronize()
    t_gpu = time.perf_counter() - t0
    line = {"case": name, "prompt": len(doc["prompt"]), "new_tokens": len(res.new_tokens),
            "rounds": res.stats.rounds, "acceptance": round(res.stats.acceptance_rate, 3),
            "device_generate_s": round(t_gpu, 3), "tokens_match_reference": res.tokens == doc["expected"]["tokens"],
            "what": "wall time of paper_2605_15508_b200.generate (prefill + every round), one host sync per round"}
    if (REF / "specsparse").is_dir():
        sys.path.insert(0, str(REF))
        import specsparse.headmap as RH
        import specsparse.sparsity as RSP
        import specsparse.specdec as RS
        import specsparse.toymodel as RT

        rt = RT.init_model(RT.ModelConfig(**doc["target_config"]))
        rd = rt if doc["draft_config"] is None else RT.init_model(RT.ModelConfig(**doc["draft_config"]))
        with tempfile.TemporaryDirectory() as td:
            rp = []
            for i, m in enumerate(doc["mappings"]):
                p = Path(td) / f"m{i}.json"
                p.write_text(json.dumps(m))
                rp.append(p)
            rms = RH.MappingSet([RH.load_mapping(p) for p in rp])
        rcfg = RS.SpecConfig(gamma=doc["gamma"], sparsity=RSP.SparsityConfig(**doc["sparsity"]), mappings=rms)
        t0 = time.perf_counter()
        rres = RS.generate(rd, rt, doc["prompt"], doc["max_new"], rcfg)
        t_ref = time.perf_counter() - t0
        line.update({"reference_generate_s": round(t_ref, 3), "speedup_vs_reference": round(t_ref / t_gpu, 1),
                     "reference_tokens_equal": rres.tokens == res.tokens})
    print(json.dumps(line), flush=True)
