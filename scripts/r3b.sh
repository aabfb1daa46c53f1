#!/bin/bash
bash scripts/ab_iround.sh r3b "ZKDL_IR_PREFETCH=0" "" "ZKDL_IR_MULW=1" "ZKDL_IR_MULW=1 ZKDL_IR_LB_B=3" "ZKDL_IR_LB_B=3" "ZKDL_IR_MULW=1 ZKDL_IR_PREFETCH=0"
