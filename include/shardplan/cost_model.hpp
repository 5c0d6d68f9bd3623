// Drop-in forwarding header: the reference path shardplan/cost_model.hpp maps onto
// the single AMSP planner header.
#pragma once
#include "amsp/plan.hpp"
