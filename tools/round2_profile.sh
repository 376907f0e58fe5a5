# round-2 evidence for profiles/: launch list of one config-2 request
# (cold, serialised: shares), --set full of the step's hand-written kernels
# (layer 0: blend, rmsnorm, QKV epilogue, attention, rmsnorm, SwiGLU)
set -x
timeout 900 ncu --profile-from-start off --metrics gpu__time_duration.sum --clock-control none \
  --csv --log-file gpurun_out/r2_step_launches.csv python tools/profile_step.py --what step > /dev/null 2>&1
timeout 1200 ncu --profile-from-start off --set full --import-source on --clock-control none \
  -k regex:"attention_pp|blend_bf16|qkv_bf16|swiglu|rmsnorm" -c 6 -o gpurun_out/r2_step_full \
  python tools/profile_step.py --what step > /dev/null 2>&1
ls -la gpurun_out
