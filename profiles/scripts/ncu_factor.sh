for C in 2 3; do
  timeout 900 ncu --set full --import-source on --clock-control none --profile-from-start off -k regex:k_factor_dag -o gpurun_out/r01_fdag_c$C python profiles/profile_factor.py --config $C > gpurun_out/ncu_fdag_c$C.log 2>&1
done
