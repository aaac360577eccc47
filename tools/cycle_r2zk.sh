# k_sweep_rows variants (g: ns>0 guard, ng: no guard, ng2: no guard + lean staging) and the static_init profile
bash tools/ring_cycle.sh r2zk g ng ng2 2>&1 | grep -v "^ab base\|^base"
bash tools/init_profile.sh r2zk
