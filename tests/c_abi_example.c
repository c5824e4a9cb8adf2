/* Plain-C use of the library through include/dsi_sim.h (README "Using it").
 * Build: gcc -std=c11 -Iinclude tests/c_abi_example.c -Lpaper_2405_14105_b200 -ldsi_sim
 * Exit status: 0 with a GPU (prints the means), 3 when no sm_100 device is present
 * (create stops with DSI_E_DEVICE after validating the config), 1 on any other error. */
#include <stdio.h>
#include <string.h>

#include "dsi_sim.h"

int main(void) {
  dsi_options opt;
  memset(&opt, 0, sizeof opt);
  opt.abi_version = DSI_ABI_VERSION;
  opt.tick = 0.01;
  opt.seed = 2405141050u;
  opt.n_devices = 1;
  opt.world = 1;
  /* t_target, t_drafter, accept_rate, lookahead, sp_degree, n_tokens, stream_id, n_trials, TTFTs */
  dsi_config cfg = {1.0, 0.1, 0.8, 5, 2, 50, 0, 1000, 0.0, 0.0};
  dsi_sim *h = NULL;
  dsi_status s = dsi_sim_create(&opt, &cfg, 1, &h);
  if (s == DSI_E_DEVICE) {
    printf("no device: %s\n", dsi_last_create_error());
    return 3;
  }
  if (s != DSI_OK) {
    printf("create: %s (%s)\n", dsi_status_str(s), dsi_last_create_error());
    return 1;
  }
  dsi_result r;
  s = dsi_sim_run(h);
  if (s == DSI_OK) s = dsi_sim_reduce(h, &r, 1);
  if (s != DSI_OK) {
    printf("run/reduce: %s (%s)\n", dsi_status_str(s), dsi_sim_last_error(h));
    dsi_sim_destroy(h);
    return 1;
  }
  printf("mean non-SI %.6f SI %.6f DSI %.6f over %llu trials\n", r.mean_nonsi, r.mean_si, r.mean_dsi,
         (unsigned long long)r.trials);
  dsi_sim_destroy(h);
  return 0;
}
