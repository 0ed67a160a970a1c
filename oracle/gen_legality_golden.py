"""TEST INFRASTRUCTURE: golden verdicts of check_semantic_legality
(I/transforms.hpp:598-663), computed by the reference's own host function
(compiled unmodified into integration/_build/libnb200_nestopt.so), for
tests/test_legality.py to hold the GPU check (nb_semantic_legality) to.

Cases, each an (original, transformed) pair of nest JSON (nbi_nest_json):
  * the reference tests' hand-injected rewrites, rebuilt from their
    descriptions (P/tests/test_transforms.cpp:311-435): init after its
    accumulations, swapped halves, producer/consumer swapped, forward-shifted
    consumer fused, write-after-write swap, reversed recurrence, duplicated
    instance, reversed accumulation chain, bottleneck (not applicable);
  * random semantic runs (interchange / strip_mine / tile / unroll / fuse /
    split, the moves of random_semantic, P/tests/acceptance.cpp:53-83) over
    conv nests of several shapes;
  * the same injections on nests near the 1e6-instance cap, where the first
    reordered pair (and so the reason string) depends on the full sort order.
Run: python oracle/gen_legality_golden.py (needs /root/reference built into
integration/_build)."""
import copy, json, os, random, sys

HERE = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, os.path.dirname(HERE))
from paper_2102_06599_b200 import search as S  # noqa: E402

OUT = os.path.join(os.path.dirname(HERE), "tests", "golden", "legality_cases.json")


def spec(ci, co, h, w, kh=1, kw=1, pad=0, groups=1, stride=1):
    return {"ci": ci, "co": co, "h": h, "w": w, "kh": kh, "kw": kw, "pad": pad,
            "groups": groups, "stride": stride}


def v(n):
    return ["v", n]


def stmt(id_, kind, domain, accesses, coord=None):
    return {"id": id_, "kind": kind, "domain": domain,
            "coord": coord or {d: v(d) for d in domain}, "accesses": accesses}


def acc(t, mode, idx):
    return {"tensor": t, "mode": mode, "indices": idx, "zero_pad": False}


def producer_consumer(n, off):
    a = stmt("A", "mac", ["i"], [acc("T", "rmw", [v("i")]), acc("X", "r", [v("i")])])
    b = stmt("B", "mac", ["i"], [acc("U", "rmw", [v("i")]),
                                 acc("T", "r", [["add", v("i"), ["c", off]]])])
    return {"parts": [{"spine": [["i", n, 1, False]], "stmts": [a]},
                      {"spine": [["i", n, 1, False]], "stmts": [b]}]}


def inits_last(nest):
    bad = copy.deepcopy(nest)
    p0 = bad["parts"][0]
    inits = {"spine": copy.deepcopy(p0["spine"]), "stmts": [p0["stmts"].pop(0)]}
    bad["parts"].append(inits)
    return bad


def dup_ci(nest):
    bad = copy.deepcopy(nest)
    bad["parts"][0]["stmts"][1]["coord"]["ci"] = ["div", v("ci"), 2]
    return bad


def reverse(nest, var, ext, stmts=None):
    out = copy.deepcopy(nest)
    for p in out["parts"]:
        for i, st in enumerate(p["stmts"]):
            if stmts is not None and i not in stmts:
                continue
            if var in st["coord"]:
                st["coord"][var] = ["add", ["mul", v(var), -1], ["c", ext - 1]]
    return out


def hand_cases():
    cases = []
    nest = S.nest_json(spec(2, 2, 2, 2))
    cases.append(("init_after_accumulations", nest, inits_last(nest)))
    halves = S.nest_json(spec(2, 2, 2, 2), "split(co,1,1)")
    swapped = copy.deepcopy(halves)
    swapped["parts"].reverse()
    cases.append(("split_halves_swapped", nest, swapped))
    pc = producer_consumer(4, 0)
    sw = copy.deepcopy(pc)
    sw["parts"].reverse()
    cases.append(("producer_consumer_swapped", pc, sw))
    pc1 = producer_consumer(4, 1)
    fused1 = {"parts": [{"spine": pc1["parts"][0]["spine"],
                         "stmts": [pc1["parts"][0]["stmts"][0], pc1["parts"][1]["stmts"][0]]}]}
    cases.append(("shifted_consumer_fused", pc1, fused1))
    fused0 = {"parts": [{"spine": pc["parts"][0]["spine"],
                         "stmts": [pc["parts"][0]["stmts"][0], pc["parts"][1]["stmts"][0]]}]}
    cases.append(("aligned_consumer_fused", pc, fused0))
    waw = {"parts": [{"spine": [["i", 4, 1, False]],
                      "stmts": [stmt(x, "init", ["i"], [acc("T", "w", [v("i")])]) for x in "AC"]}]}
    waw_bad = copy.deepcopy(waw)
    waw_bad["parts"][0]["stmts"].reverse()
    cases.append(("write_after_write_swapped", waw, waw_bad))
    rec = {"parts": [{"spine": [["i", 4, 1, False]], "stmts": [
        stmt("S", "mac", ["i"], [acc("T", "rmw", [v("i")]),
                                 acc("T", "r", [["add", v("i"), ["c", -1]]])])]}]}
    cases.append(("recurrence_reversed", rec, reverse(rec, "i", 4)))
    n4 = S.nest_json(spec(4, 2, 1, 1))
    cases.append(("duplicated_instance", n4, dup_ci(n4)))
    cases.append(("accumulation_chain_reversed", n4, reverse(n4, "ci", 4)))
    n8 = S.nest_json(spec(4, 8, 2, 2))
    cases.append(("bottleneck_not_applicable", n8, S.nest_json(spec(4, 8, 2, 2), "bottleneck(co,2)")))
    return [dict(name=n, original=o, transformed=t, cap=1_000_000) for n, o, t in cases] + [
        dict(name="cap_exceeded", original=S.nest_json(spec(8, 8, 8, 8, 3, 3, 1)),
             transformed=S.nest_json(spec(8, 8, 8, 8, 3, 3, 1)), cap=100)]


def random_run(sp, rng, max_len=4):
    dsl = []
    for _ in range(rng.randint(1, max_len)):
        cur = S.nest_json(sp, " | ".join(dsl))
        for _attempt in range(25):
            p = rng.randrange(len(cur["parts"]))
            spine = [iv[0] for iv in cur["parts"][p]["spine"]]
            if not spine:
                break
            tgt = f"@{p}" if p else ""
            k = rng.randrange(6)
            a, b = rng.choice(spine), rng.choice(spine)
            f = rng.choice([2, 2, 4])
            if k == 0:
                step = f"interchange{tgt}({a},{b})"
            elif k == 1:
                step = f"strip_mine{tgt}({a},{f})"
            elif k == 2:
                step = f"tile{tgt}({a},{f})"
            elif k == 3:
                step = f"unroll{tgt}({a},{f})"
            elif k == 4:
                i = rng.randrange(len(spine))
                if i + 1 >= len(spine):
                    continue
                step = f"fuse{tgt}({spine[i]},{spine[i + 1]})"
            else:
                ext = dict((iv[0], iv[1]) for iv in cur["parts"][p]["spine"])[a]
                if ext < 2:
                    continue
                cut = rng.randrange(1, ext)
                step = f"split{tgt}({a},{cut},{ext - cut})"
            try:
                S.nest_json(sp, " | ".join(dsl + [step]))
            except Exception:
                continue
            dsl.append(step)
            break
    return " | ".join(dsl)


def main():
    out = hand_cases()
    rng = random.Random(2)
    shapes = [spec(4, 8, 4, 4, 3, 3, 1), spec(2, 4, 5, 5, 3, 3, 1, stride=2), spec(6, 4, 3, 3),
              spec(4, 4, 6, 6, 3, 3, 1, groups=2), spec(3, 5, 7, 7, 5, 5, 2)]
    for si, sp in enumerate(shapes):
        base = S.nest_json(sp)
        for t in range(12):
            dsl = random_run(sp, rng)
            out.append(dict(name=f"random_{si}_{t}", dsl=dsl, original=base,
                            transformed=S.nest_json(sp, dsl), cap=1_000_000))
    # near the cap: 8x16 3x3 over 28x28 (903,168 MACs + 12,544 inits)
    big = spec(8, 16, 28, 28, 3, 3, 1)
    bn = S.nest_json(big)
    for dsl in ["tile(h,4) | interchange(ci,w) | unroll(kw,3)",
                "fuse(h,w) | strip_mine(ci,2) | interchange(co,ci_o)",
                "split(co,5,11) | interchange@1(ci,kh) | tile@0(w,7)"]:
        out.append(dict(name="big_" + dsl.split("(")[0], dsl=dsl, original=bn,
                        transformed=S.nest_json(big, dsl), cap=1_000_000))
    out.append(dict(name="big_init_after_accumulations", original=bn, transformed=inits_last(bn),
                    cap=1_000_000))
    out.append(dict(name="big_duplicated_instance", original=bn, transformed=dup_ci(bn),
                    cap=1_000_000))
    # only the init block reversed in co: inits of co=15 run first, still
    # before all accumulations -- legal; reversing the MACs' h against a
    # shifted init is not
    out.append(dict(name="big_inits_reversed", original=bn, transformed=reverse(bn, "co", 16, [0]),
                    cap=1_000_000))
    tr = S.nest_json(big, "split(h,14,14)")
    bad = copy.deepcopy(tr)
    bad["parts"][1]["stmts"] = [bad["parts"][1]["stmts"][1], bad["parts"][1]["stmts"][0]]
    out.append(dict(name="big_half_inits_after_macs", original=bn, transformed=bad, cap=1_000_000))
    # MACs of rows h >= 14 now run before their init: the first reordered
    # pair sits in the middle of the sorted touch order
    out.append(dict(name="big_macs_h_reversed", original=bn, transformed=reverse(bn, "h", 28, [1]),
                    cap=1_000_000))
    big_pc = producer_consumer(400_000, 1)
    fused_pc = {"parts": [{"spine": big_pc["parts"][0]["spine"],
                           "stmts": [big_pc["parts"][0]["stmts"][0], big_pc["parts"][1]["stmts"][0]]}]}
    out.append(dict(name="big_shifted_consumer_fused", original=big_pc, transformed=fused_pc,
                    cap=1_000_000))
    big_pc0 = producer_consumer(400_000, 0)
    fused_pc0 = {"parts": [{"spine": big_pc0["parts"][0]["spine"],
                            "stmts": [big_pc0["parts"][0]["stmts"][0], big_pc0["parts"][1]["stmts"][0]]}]}
    out.append(dict(name="big_aligned_consumer_fused", original=big_pc0, transformed=fused_pc0,
                    cap=1_000_000))
    out.append(dict(name="big_over_cap", original=S.nest_json(spec(16, 16, 28, 28, 3, 3, 1)),
                    transformed=S.nest_json(spec(16, 16, 28, 28, 3, 3, 1), "interchange(ci,kh)"),
                    cap=1_000_000))
    for c in out:
        res, ms = S.legality_nests(c["original"], c["transformed"], c["cap"], device=-1)
        c["expected"] = res
        c["host_ms"] = round(ms, 3)
        print(f'{c["name"]:36s} {ms:9.1f} ms  {res}', flush=True)
    with open(OUT, "w") as f:
        json.dump(out, f, separators=(",", ":"))
    print("wrote", OUT, len(out), "cases")


if __name__ == "__main__":
    main()
