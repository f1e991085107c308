// tt_ws_w2.cu -- instantiation of the warp-specialised contraction kernel, tile ws80x80x16_2cta.
#include "tt_contract_ws.cuh"

namespace tt { namespace ws { using Cfg_w2 = WCfg<80, 80, 16, 2, 2, 6, 2>; } }
TT_WS_DEFINE(w2, ws::Cfg_w2, "ws80x80x16_2cta")
