"""Pipe-throughput microbenchmarks on the GPU box (lib/libplubench.so)."""
import ctypes as C
import json
import os

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
L = C.CDLL(os.path.join(ROOT, "paper_1407_2343_b200", "lib", "libplubench.so"))
for fn in (L.plub_rate, L.plub_pair_rate):
    fn.restype = C.c_double
    fn.argtypes = [C.c_int, C.c_int, C.c_int, C.c_int, C.POINTER(C.c_double)]
import torch  # noqa: E402  (initialises the device)
torch.cuda.init()
ms = C.c_double(0)
res = {}
for name, w in (("ex2", 0), ("ffma", 1), ("ffma2", 2)):
    res[name + "_per_s"] = L.plub_rate(w, 8, 256, 4096, C.byref(ms))
for form in (0, 1, 2):
    for bps, thr in ((2, 64), (4, 64), (6, 64), (8, 64), (4, 128), (8, 128), (16, 64)):
        r = L.plub_pair_rate(form, bps, thr, 2000, C.byref(ms))
        res[f"pair_form{form}_b{bps}_t{thr}"] = r
res["ex2_frac"] = {k: v / res["ex2_per_s"] for k, v in res.items() if k.startswith("pair")}
print(json.dumps(res, indent=1))
L.plub_pk_rate.restype = C.c_double
L.plub_pk_rate.argtypes = [C.c_int, C.c_int, C.c_int, C.c_int]
clk = 1.965e9
pk = {}
for op, name in enumerate(["ffma2_3pair", "fadd2_2pair", "fmul2_2pair", "ffma2_fadd2_mix", "ffma_3reg", "fadd_2reg", "imad_3reg", "iadd3"]):
    for bps, thr in ((4, 128), (8, 128)):
        r = L.plub_pk_rate(op, bps, thr, 4000)
        pk[f"{name}_w{bps*thr//32}"] = {"warp_instr_per_clk_per_sm": r / clk, "cycles_per_instr_per_smsp": 4 * clk / r}
print(json.dumps(pk, indent=1))

# Mixed-pipe dispatch test (cycles per warp-iteration per SMSP).
L.plub_mix_cycles.restype = C.c_double
L.plub_mix_cycles.argtypes = [C.c_int, C.c_int, C.c_int, C.c_int, C.c_double]
names = ["8xFFMA2", "2xMUFU", "8xFFMA2+2xMUFU", "16xFFMA", "16xFFMA+2xMUFU", "8xFFMA2+8xIADD",
         "8xIADD", "12xFFMA2+2xMUFU", "6xFFMA2+2xMUFU"]
mix = {}
for w, nm in enumerate(names):
    for bps, thr in ((1, 128), (2, 128), (4, 128)):
        mix[f"{nm}_warps{bps * thr // 128}"] = round(L.plub_mix_cycles(w, bps, thr, 20000, 1965.0), 2)
print(json.dumps(mix, indent=1))
