// Scheduling knobs of libpolykv.so (host side). Read from the environment
// once per process -- not on every launch -- and re-read only when the caller
// asks for it with pkv_reload_tuning() (include/polykv.h). None of them
// changes a result: they move work between SMs (role splits, absmax lag,
// attention split count) or select the warp-granular codec for A/B tests;
// tests/test_gpu_parity.py::test_role_splits_and_schedules_do_not_change_results
// checks that every setting gives bit-identical pools.
#pragma once

namespace pkv {

struct Tuning {
  bool codec_warp = false;         // PKV_CODEC_PATH=warp: warp-granular codec (codec.cu) only
  int dbg_enc = 0;                 // PKV_DBG_ENC: encode timing experiments (skip math)
  int key_lag = 0;                 // PKV_KEY_LAG (0 = default): absmax layers ahead of the key encode
  bool enc_co = false;             // PKV_ENC_ROLES=co: co-resident encode roles (enc_co_kernel) instead of SM role split
  bool abs_on_values = false;      // PKV_ABSMAX_ROLE=values: per-tensor key absmax items run on the value CTAs
  double key_sm_fraction = -1.0;   // PKV_KEY_SM_FRACTION (<0 = default): encode SMs for the key role
  double dec_key_fraction = -1.0;  // PKV_DEC_KEY_FRACTION (<0 = default): decode SMs for key items
  int attn_ctas_per_sm = 0;        // PKV_ATTN_CTAS_PER_SM (0 = default): attention prefix splits
  bool attn_simt = false;          // PKV_ATTN_PATH=simt: fp32 CUDA-core prefix kernel instead of mma.sync
  int attn_min_tiles = 0;          // PKV_ATTN_MIN_TILES (0 = default 4): 64-token tiles per attention split
};

// The current knobs (an immutable snapshot; cheap to call per launch).
const Tuning& tuning();
// Re-read the environment (pkv_reload_tuning).
void reload_tuning();

}  // namespace pkv
