# ncu --set full of one k_solve_dag launch (config 2) and one k_vertex_assemble launch (config 5)
timeout 900 ncu --set full --import-source on --clock-control none --profile-from-start off -k regex:k_vertex_assemble -c 1 -o gpurun_out/r01_vertex_c5 python profiles/profile_assembly.py --config 5 --reps 1 > gpurun_out/ncu_vertex.log 2>&1
SGN_BICG_GRAPH=0 timeout 900 ncu --set full --import-source on --clock-control none -k regex:k_solve_dag -s 40 -c 1 -o gpurun_out/r01_solve_c2 python profiles/solve_timing.py --reps 3 > gpurun_out/ncu_solve.log 2>&1
