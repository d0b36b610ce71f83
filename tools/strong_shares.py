"""Strong-scaling projection of C4 from single-GPU runs: each rank's query
block (1,024,000 / P queries) is timed alone on one B200 with bench.py --nq; the projected
efficiency at P GPUs is T(N=1) / (P * T(share)), excluding the one 8-byte allreduce per
step.  usage: python tools/strong_shares.py BENCH_N1.json SHARE_1.json [SHARE_2.json ...]"""
import json
import sys


def line(path):
    return json.loads(open(path).read().strip().splitlines()[-1])


def main():
    n1 = line(sys.argv[1])
    out = {"n1_ms_per_step": n1["ms_per_step"], "n1_phases_ms": n1["phases_ms"], "shares": {}, "projected_efficiency": {}}
    nq_total = n1["config"].get("nq_total", 1024000)
    for p in sys.argv[2:]:
        d = line(p)
        nq = d["config"].get("nq_total")
        P = round(nq_total / nq)
        out["shares"][str(nq)] = {"ms_per_step": d["ms_per_step"], "phases_ms": d["phases_ms"], "clocks": d.get("clocks")}
        out["projected_efficiency"][str(P)] = n1["ms_per_step"] / (P * d["ms_per_step"])
    out["note"] = ("C4 strong scaling: each rank block (1,024,000/P queries) timed alone on one B200 "
                   "(bench.py --nq share); efficiency T1/(P T_share) excludes the 8-byte NCCL allreduce per step")
    print(json.dumps(out, indent=1))


if __name__ == "__main__":
    main()
