#!/bin/bash
# Committed SASS listings (north star: "plus a committed SASS listing") of the
# hot kernels, from the in-tree objects, with a mnemonic histogram per kernel.
set -eu
B=paper_2102_11089_b200/csrc/build
O=profiles/sass
mkdir -p $O
dump() {  # object mangled-name outfile
  cuobjdump -sass -fun "$2" $B/$1 | grep -E '^\s+/\*[0-9a-f]{4,}\*/' | sed -E 's@^\s+/\*([0-9a-f]+)\*/\s+@\1 @; s@\s*/\*.*\*/\s*;?\s*$@@' > $O/$3.sass
  awk '{op=$2; if (op ~ /^@/) op=$3; sub(/\..*/, "", op); c[op]++} END {for (k in c) print c[k], k}' $O/$3.sass | sort -rn > $O/$3.hist
  echo "$3: $(wc -l < $O/$3.sass) instructions; $(grep -cE 'UBLKCP|UTMALDG' $O/$3.sass || true) bulk-copy, $(grep -c 'SYNCS' $O/$3.sass || true) SYNCS"
}
dump fixed_phase_f32.o _ZN4ldpc22phase_check_tma_kernelIfLi0ELb0ELi8ELb0EEEvNS_11PhaseParamsEiiii check_tma_f32_exact_flooding
dump fixed_phase_f32.o _ZN4ldpc22phase_check_tma_kernelIfLi0ELb1ELi8ELb0EEEvNS_11PhaseParamsEiiii check_tma_f32_exact_layered
dump fixed_phase_f32.o _ZN4ldpc19phase_vn_tma_kernelIfLi8EEEvNS_11PhaseParamsE vn_tma_f32
dump dyn_f64_exact_b.o _ZN4ldpc17dyn_decode_kernelIdLi0ELi2ELi2ELi32ELb0ELb0EEEvNS_9DynParamsE dyn_f64_exact_cirbp_mode2
dump dyn_f64_exact_a.o _ZN4ldpc17dyn_decode_kernelIdLi0ELi2ELi1ELi32ELb0ELb0EEEvNS_9DynParamsE dyn_f64_exact_rbp_mode2
dump dyn_f64_exact_a.o _ZN4ldpc17dyn_decode_kernelIdLi0ELi3ELi1ELi32ELb0ELb0EEEvNS_9DynParamsE dyn_f64_exact_rbp_mode3
dump dyn_f64_exact_b.o _ZN4ldpc17dyn_decode_kernelIdLi0ELi3ELi2ELi32ELb0ELb0EEEvNS_9DynParamsE dyn_f64_exact_cirbp_mode3
dump dyn_f64_exact_d.o _ZN4ldpc17dyn_decode_kernelIdLi0ELi2ELi6ELi32ELb0ELb0EEEvNS_9DynParamsE dyn_f64_exact_me_cirbp_mode2
dump dyn_f64_exact_d.o _ZN4ldpc17dyn_decode_kernelIdLi0ELi3ELi6ELi32ELb0ELb0EEEvNS_9DynParamsE dyn_f64_exact_me_cirbp_mode3
dump dyn_f32_exact_k.o _ZN4ldpc17dyn_decode_kernelIfLi0ELi3ELi1ELi32ELb0ELb0EEEvNS_9DynParamsE dyn_f32_exact_rbp_mode3
