"""Write profiles/<round>_profile_latest.md (+ copies of the bench JSON lines,
launch lists and the traffic table) from a tools/gpu_profiles.sh run in
gpurun_out/.  usage: python tools/write_profile_md.py [round, default r2]"""
import json
import shutil
import subprocess
import sys

G = "gpurun_out"
P = "profiles"
R = sys.argv[1] if len(sys.argv) > 1 else "r2"


def last_json(path):
    return json.loads(open(path).read().strip().splitlines()[-1])


def main():
    b, t, f = last_json(f"{G}/bench.json"), last_json(f"{G}/train.json"), last_json(f"{G}/fine.json")
    r = last_json(f"{G}/ref.json")
    for name, obj in ((f"{R}_bench_default.json", b), (f"{R}_train_bench.json", t), (f"{R}_fine_bench.json", f),
                      (f"{R}_reference_arm.json", r)):
        with open(f"{P}/{name}", "w") as fh:
            fh.write(json.dumps(obj) + "\n")
    shutil.copy(f"{G}/launches.csv", f"{P}/{R}_launches_default.csv")
    shutil.copy(f"{G}/train_launches.csv", f"{P}/{R}_launches_train.csv")
    kernels = ["k_blend", "k_mlp_tc_2s", "k_hexplane_latent_c32t", "k_preprocess", "k_tile_sort", "k_emit_partition"]
    subprocess.run([sys.executable, "tools/ncu_traffic.py", f"{P}/{R}_traffic.json"] +
                   [f"{G}/full_{k}.ncu-rep" for k in kernels], check=True, capture_output=True)
    run = lambda *a: subprocess.run([sys.executable, "tools/ncu_summary.py", *a], capture_output=True,  # noqa: E731
                                    text=True).stdout
    l1, l2 = run("launches", f"{P}/{R}_launches_default.csv"), run("launches", f"{P}/{R}_launches_train.csv")
    full = "\n".join(run("full", f"{G}/full_{k}.ncu-rep") for k in kernels)
    train_kernels = ["k_blend_bwd2", "k_mlp_bwd_tc", "k_hexplane_bwd_c32", "k_preprocess_bwd"]
    full_train = "\n".join(run("full", f"{G}/full_{k}.ncu-rep") for k in train_kernels)
    rf = b["roofline"]
    txt = f"""# Round {R[1:].lstrip("0")} — committed-build profile (latest)

Bench (no profiler, `python bench.py`): **{b['value']:.1f} frames/s** whole-job (configs[2] sequence,
{b['config']['parallelism']}, {b.get('setup', {}).get('frames_in_flight', '')}; {b.get('setup', b['config']).get('l2', '')}); one frame at a time with an L2 flush between
frames: {b['value_serial']['value']:.1f} frames/s ({b['value_serial']['ms_per_frame']:.3f} ms/frame).
End to end through pinned PCIe copies (H2D {b['e2e']['h2d_bytes_per_step']/1e6:.1f} MB + D2H
{b['e2e']['d2h_bytes_per_step']/1e6:.1f} MB per frame): {b['e2e']['value']:.1f} frames/s.  CPU reference arm:
{r['value']:.3f} frames/s on {r['cpu_baseline']['cores']} cores.  Clocks: {json.dumps(b['clocks'])}.

Roofline (dominant kernel `{rf['kernel']}`): {rf['achieved']:.0f} GB/s algorithmic of {rf['peak']:.0f} GB/s
(frac {rf['frac']:.3f}); DRAM traffic {rf['traffic']/1e6:.1f} MB per launch (ncu) vs
{rf['algorithmic_bytes_per_launch']/1e6:.1f} MB algorithmic — the projected records it gathers are
L2-resident from `k_preprocess`.  Serial stage times (ms): {json.dumps(b['stage_ms'])}.
Per-kernel algorithmic GB/s: {json.dumps({k: round(v['achieved_gbs'], 1) for k, v in b['kernels'].items()})}.
MLP: {b['mlp']['tflops']:.1f} TFLOP/s useful (x3 issued as the bf16 split:
{b['mlp']['frac_of_bf16_peak_issued']:.3f} of the bf16 peak).

Training (configs[4], 8 pairs, fwd+bwd+all-reduce, {t['config'].get('pairs_in_flight', 1)} pairs in flight): {t['value']:.1f} steps/s ({t['ms_per_step']:.2f} ms/step);
stage ms/step (one serial step) {json.dumps(t['stage_ms_per_step'])}.
Fine-stage iteration (decoder + depth + TV + Adam): {f['value']:.1f} steps/s ({f['ms_per_step']:.2f} ms/step).

## Render launch list (`ncu --metrics gpu__time_duration.sum --clock-control none`; serialised, cold cache: compare shares)

{l1}
## Training-step launch list

{l2}
## `ncu --set full` of the top render kernels (one launch each, `-s 3 -c 1`)

{full}

## `ncu --set full` of the top training-step kernels (one launch each, `-s 2 -c 1`)

{full_train}
"""
    open(f"{P}/{R}_profile_latest.md", "w").write(txt)
    print(txt[:1800])


if __name__ == "__main__":
    main()
