"""Randomised campaign over the GPU sort: sizes, key types, payloads, input
patterns, scratch modes and the test hooks (minrun, fused-subtree / tile /
block sizes, one or two tree levels per pass), each case checked bit-exact
against the plain definition of the result: the
stable sort of (key, position) under the key order -- numpy's stable argsort
of the order image (u32 / u64 as is; f32 bits b -> b ^ (sign ? ~0 : 2^31),
every NaN -> the maximum image).  The payload is the input position, so the
output payload must be exactly that permutation and the output keys the
input keys gathered by it.

usage: python scripts/fuzz_gpu.py [CASES] [SEED] [MAXLOG]   (MAXLOG > 23: 60% of
the cases have 2^21 <= n < 2^MAXLOG; prints one JSON line per
failure and a summary line; exit 1 on any failure)"""
import json, math, os, sys, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import torch
import paper_2605_27147_b200 as vm


def order_image(keys: np.ndarray, kt: str) -> np.ndarray:
    if kt == "f32":
        b = keys.view(np.uint32).astype(np.uint64)
        img = np.where(b >> 31, b ^ 0xFFFFFFFF, b ^ 0x80000000)
        nan = np.isnan(keys)
        img[nan] = 0xFFFFFFFF
        return img
    return keys.astype(np.uint64)


def gen(rng: np.random.Generator, n: int, kt: str, pat: str) -> np.ndarray:
    if kt == "u64":
        base = rng.integers(0, 2**63, size=n, dtype=np.uint64) * np.uint64(2) + rng.integers(0, 2, size=n, dtype=np.uint64)
    elif kt == "u32":
        base = rng.integers(0, 2**32, size=n, dtype=np.uint64).astype(np.uint32)
    else:
        base = rng.standard_normal(n).astype(np.float32) * np.float32(rng.choice([1e-3, 1.0, 1e6]))
    if pat == "uniform":
        k = base
    elif pat == "few":
        vals = base[: max(1, int(rng.integers(1, 17)))] if n else base
        k = vals[rng.integers(0, len(vals), size=n)] if n else base
    elif pat == "equal":
        k = np.full(n, base[0] if n else 0, dtype=base.dtype)
    elif pat in ("segments", "segments_rev", "mixed"):
        k = base.copy()
        pos = 0
        mean = float(rng.choice([8, 40, 300, 5000, 70000]))
        while pos < n:
            ln = int(min(n - pos, 1 + rng.geometric(1.0 / mean)))
            kind = rng.integers(0, 3) if pat == "mixed" else (1 if pat == "segments" else 2)
            if kind == 1:
                k[pos:pos + ln] = np.sort(k[pos:pos + ln], kind="stable")
            elif kind == 2:
                k[pos:pos + ln] = np.sort(k[pos:pos + ln], kind="stable")[::-1]
            pos += ln
    elif pat == "sawtooth":
        per = int(rng.integers(2, 5000))
        idx = np.arange(n) % per
        k = np.sort(base[:per])[idx] if n else base
    elif pat == "sorted":
        k = np.sort(base, kind="stable")
    else:  # reversed
        k = np.sort(base, kind="stable")[::-1].copy()
    k = np.ascontiguousarray(k)
    if kt == "f32" and n and rng.random() < 0.5:  # specials: +-0, +-inf, NaNs with payloads
        m = int(rng.integers(1, max(2, n // 50)))
        at = rng.integers(0, n, size=m)
        sp = np.array([0.0, -0.0, np.inf, -np.inf, np.nan], dtype=np.float32)
        k[at] = sp[rng.integers(0, len(sp), size=m)]
        nanp = rng.integers(0, n, size=max(1, m // 4))
        k.view(np.uint32)[nanp] = (rng.integers(0, 2, size=len(nanp)) << 31 | 0x7FC00000
                                   | rng.integers(1, 1 << 22, size=len(nanp))).astype(np.uint32)
    return k


def to_dev(k: np.ndarray, kt: str) -> torch.Tensor:
    if kt == "u64":
        return torch.from_numpy(k.view(np.int64).copy()).view(torch.uint64).cuda()
    if kt == "u32":
        return torch.from_numpy(k.view(np.int32).copy()).view(torch.uint32).cuda()
    return torch.from_numpy(k.copy()).cuda()


def to_host_bits(t: torch.Tensor, kt: str) -> np.ndarray:
    if kt == "u64":
        return t.view(torch.int64).cpu().numpy().view(np.uint64)
    return t.view(torch.int32).cpu().numpy().view(np.uint32)


def run(cases: int, seed: int, maxlog: int = 23):
    """Run `cases` random cases from `seed`; returns (failed case dicts,
    cases skipped for a refused scratch budget, elements sorted)."""
    rng = np.random.default_rng(seed)
    pats = ["uniform", "few", "equal", "segments", "segments_rev", "mixed", "sawtooth", "sorted", "reversed"]
    failed, skipped, tot = [], 0, 0
    try:
        for c in range(cases):
            kt = str(rng.choice(["u32", "u32", "u64", "f32"]))
            r = rng.random()
            if r < 0.05:
                n = int(rng.integers(0, 8))
            elif r < (0.9 if maxlog <= 23 else 0.4):
                n = int(math.exp(rng.uniform(math.log(8), math.log(1 << 21))))
            else:
                n = int(rng.integers(1 << 21, 1 << maxlog))
            pat = str(rng.choice(pats))
            hv = bool(rng.random() < 0.75)
            minrun = int(rng.choice([0, 0, 0, 1, 2, 4, 7, 16, 33])) if n < (1 << 20) else 0
            hooks = rng.random() < 0.35 and n < (1 << 20)
            fz = int(rng.choice([64, 128, 512])) if hooks else 0
            mt = int(rng.choice([16, 64, 256])) if hooks else 0
            mode = int(rng.choice([1, 2, 2, 2]))
            bounded = rng.random() < 0.2 and n >= 64
            scratch = None
            blk = 0
            if bounded:
                scratch = int(max(64, rng.uniform(4, 8) * math.sqrt(n * max(1.0, math.log2(n)))))
                if hooks:
                    blk = int(rng.choice([16, 32, 64]))
            vm.test_set_minrun(minrun)
            vm.test_set_tiles(fz, mt, blk)
            vm.test_set_mode(mode)
            case = dict(case=c, seed=seed, n=n, kt=kt, pat=pat, hv=hv, minrun=minrun, fuse_z=fz, tile=mt,
                        mode=mode, scratch=scratch, blk=blk)
            try:
                k0 = gen(rng, n, kt, pat)
                perm = np.argsort(order_image(k0, kt), kind="stable")
                kd = to_dev(k0, kt)
                vd = torch.arange(n, dtype=torch.int32, device="cuda").view(torch.uint32) if hv else None
                vm.sort_(kd, vd, scratch=scratch)
                torch.cuda.synchronize()
                kb = to_host_bits(kd, kt)
                want = (k0.view(np.uint64) if kt == "u64" else k0.view(np.uint32))[perm]
                ok = np.array_equal(kb, want)
                if hv:
                    ok = ok and np.array_equal(vd.view(torch.int32).cpu().numpy().astype(np.int64), perm)
            except vm.VmpsError as e:  # a library error fails the case, except a scratch
                if "budget" in str(e).lower():  # below the minimum working set (refused by contract)
                    skipped += 1
                    continue
                ok = False
                case["error"] = repr(e)[:200]
            tot += n
            if not ok:
                failed.append(case)
    finally:
        vm.test_set_minrun(0)
        vm.test_set_tiles(0, 0, 0)
        vm.test_set_mode(2)
    return failed, skipped, tot


def main():
    cases = int(sys.argv[1]) if len(sys.argv) > 1 else 300
    seed = int(sys.argv[2]) if len(sys.argv) > 2 else 2026
    maxlog = int(sys.argv[3]) if len(sys.argv) > 3 else 23
    t0 = time.time()
    failed, skipped, tot = run(cases, seed, maxlog)
    for f in failed:
        print(json.dumps({"fail": f}), flush=True)
    print(json.dumps({"cases": cases, "seed": seed, "maxlog": maxlog, "failures": len(failed), "skipped_budget": skipped,
                      "elements": tot, "seconds": round(time.time() - t0, 1)}), flush=True)
    sys.exit(1 if failed else 0)


if __name__ == "__main__":
    main()
