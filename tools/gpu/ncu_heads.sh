# ncu --set full captures of every default kernel at HEAD (one GPU; W > 1
# groups emulated in one process by tools/ncu_targets.py), plus the raw C-ABI
# kernels. Each capture follows a plain run of the same command.
set -x
mkdir -p gpurun_out/ncu
NCU="ncu --set full --clock-control none --import-source on"
ONLY=${1:-}   # optional substring filter on the capture names
run() {  # name, regex, skip, command... (ALGKEY: the plain-run key of the bytes)
  local name=$1 re=$2 skip=$3; shift 3
  case "$name" in *"$ONLY"*) ;; *) return ;; esac
  timeout 600 "$@" > gpurun_out/ncu/$name.plain.log 2>&1 &&
  timeout 900 $NCU -k regex:$re -s $skip -c 1 -o gpurun_out/ncu/$name "$@" > gpurun_out/ncu/$name.ncu.log 2>&1
  echo "$name rc=$?"
  # summary on the box (the .ncu-rep files exceed gpurun's 64 MiB return)
  alg=$(python tools/ncu_summary.py alg gpurun_out/ncu/$name.plain.log $ALGKEY)
  python tools/ncu_summary.py full gpurun_out/ncu/$name.ncu-rep $alg > gpurun_out/ncu/$name.json 2>&1
  [ "$name" = fused_w1_7b ] || rm -f gpurun_out/ncu/$name.ncu-rep
}
run fused_w1_7b fused_step 0 python tools/ncu_targets.py fused --world 1 --model llama-7b --steps 2
run fused_w2_1b fused_step 0 python tools/ncu_targets.py fused --world 2 --steps 2
run fused_w4_1b fused_step 0 python tools/ncu_targets.py fused --world 4 --steps 2
run fused_w8_1b fused_step 0 python tools/ncu_targets.py fused --world 8 --steps 2
run gather_tma_w4_1b gather_tma 2 python tools/ncu_targets.py gather --world 4 --steps 2 --unit 2
run raw_adamw adamw_flat 1 python tools/bench_raw.py --only adamw_flat_kernel\<bf16 --iters 1 --warmup 1
run raw_rs4 rs_upcast 1 python tools/bench_raw.py --only rs_upcast_scale_kernel\<4 --iters 1 --warmup 1
run raw_ag4 ag_downcast 1 python tools/bench_raw.py --only ag_downcast_kernel\<4 --iters 1 --warmup 1
# M > 1 with s_g > 1 (ZeRO-2, W=2 / 4 emulated): the accumulation kernel and
# the fused update with accumulator sources in its TMA ring
ALGKEY=algorithmic_bytes_accumulate run staged_accumulate_w2_1b accumulate_kernel 0 python tools/ncu_targets.py staged --world 2 --steps 2
run staged_fused_w2_1b fused_step 0 python tools/ncu_targets.py staged --world 2 --steps 2
run staged_fused_w4_1b fused_step 0 python tools/ncu_targets.py staged --world 4 --steps 2
ls -la gpurun_out/ncu
# the step's push all-gather (s_p > 1 default), ZeRO-3 W=4 emulated
run push_w4_1b push_tma 0 python tools/ncu_targets.py push --world 4 --steps 2
ls -la gpurun_out/ncu
