"""Write tests/golden/configs_oracle.json: the CPU ORACLE's counts for the five
BASELINE.json configs, with the input checksum (synth.checksum) they belong to.

Calls only synth/ (inputs) and oracle/ (counts) -- never the CUDA path -- so the
stored values are oracle values (task rule: "a stored value is ... written by a
committed script that calls only oracle/").  Usage:
    python tools/write_oracle_goldens.py C1 C2 C3 C4 C5
Existing entries for other configs are kept.  With --next1, also the NEXT-1
values: Lollipop / Barbell COUNT(*) and the sha256 of the
per-vertex triangle counts t(v) (uint64, in ascending original-id order).
With --k4, the 4-clique count of every named config (BASELINE.json north star:
"triangle and 4-clique counts bit-exact with the CPU oracle on all five
configs"), not only of the 4-clique config C4.  Values already stored for a
config (four_cliques, next1) are kept unless recomputed.
"""
import hashlib
import json
import os
import sys
import time

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import oracle  # noqa: E402
import synth  # noqa: E402

OUT = os.path.join(ROOT, "tests", "golden", "configs_oracle.json")


def main(names, next1=False, k4=False):
    data = json.load(open(OUT)) if os.path.exists(OUT) else {
        "citation": "BASELINE.json configs (SURVEY.md §8 C1..C5); values computed by oracle/eh_oracle.c "
                    "via tools/write_oracle_goldens.py on synthetic inputs from synth/ (DESIGN.md §4)",
        "configs": {}}
    for name in names:
        cfg = synth.CONFIGS[name]
        t0 = time.time()
        src, dst = cfg.generate()
        ck = synth.checksum(src, dst)
        t1 = time.time()
        g = oracle.Graph(src, dst)
        del src, dst
        t2 = time.time()
        entry = {"n_input": g.n_input, "m_undirected": g.m, "n_active": g.n_vertices,
                 "max_out_degree": g.max_out_degree, "checksum": str(ck)}
        entry["triangles"] = g.count_triangles()
        t3 = time.time()
        if cfg.query == "4cliques" or k4:
            entry["four_cliques"] = g.count_4cliques()
        t4 = time.time()
        entry["oracle_seconds"] = {"generate": round(t1 - t0, 1), "ingest": round(t2 - t1, 1),
                                   "triangles": round(t3 - t2, 1), "four_cliques": round(t4 - t3, 1),
                                   "threads": oracle.default_threads()}
        if next1:
            tv = g.triangles_per_vertex()
            entry["next1"] = {"sum_t": int(tv.sum(dtype="uint64")),
                              "t_sha256": hashlib.sha256(tv.astype("<u8").tobytes()).hexdigest(),
                              "lollipop": str(g.count_lollipop()), "barbell": str(g.count_barbell()),
                              "seconds": round(time.time() - t4, 1)}
        g.close()
        old = data["configs"].get(name, {})
        if old.get("checksum") == entry["checksum"]:
            if "four_cliques" in old and "four_cliques" not in entry:
                entry["four_cliques"] = old["four_cliques"]
                entry["oracle_seconds"]["four_cliques"] = old.get("oracle_seconds", {}).get("four_cliques", 0.0)
            if "next1" in old and "next1" not in entry:
                entry["next1"] = old["next1"]
        data["configs"][name] = entry
        json.dump(data, open(OUT, "w"), indent=1)
        print(name, entry, flush=True)


if __name__ == "__main__":
    args = [a for a in sys.argv[1:] if not a.startswith("--")]
    main(args or ["C1", "C2", "C3", "C4"], next1="--next1" in sys.argv, k4="--k4" in sys.argv)
